"""One prefill GEMM launch for ncu: gemm_one.py [M] [K] [N] (KN tensor, p=4, f32 output)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import gemm
from paper_2410_13461_b200.quant import quantize_tensor
M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
N = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
pk = quantize_tensor(torch.randn((K, N), device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
x = torch.randn((M, K), device="cuda").half()
pd = torch.tensor([4], dtype=torch.int32, device="cuda")
for _ in range(3):
    y = gemm(pk, x, pd)
torch.cuda.synchronize()
print("ok")
