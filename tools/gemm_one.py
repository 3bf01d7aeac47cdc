"""One prefill GEMM launch (4096x4096, M=512, p=4) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import gemm
from paper_2410_13461_b200.quant import quantize_tensor
N = K = 4096; M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pk = quantize_tensor(torch.randn((K, N), device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
x = torch.randn((M, K), device="cuda").half()
pd = torch.tensor([4], dtype=torch.int32, device="cuda")
for _ in range(3):
    y = gemm(pk, x, pd)
torch.cuda.synchronize()
print("ok")
