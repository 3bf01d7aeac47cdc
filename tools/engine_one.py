"""Run one engine program (single big op, or a chain) a few times: target for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.engine import OpSpec, Program
from paper_2410_13461_b200.quant import quantize_tensor
K, N = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x32000").split("x"))
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.manual_seed(0)
pk = quantize_tensor(torch.randn(K, N, device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
prog = Program([OpSpec(pk)])
x = torch.randn(1, K, device="cuda").half()
y = torch.zeros(N, device="cuda")
pd = torch.tensor([p], dtype=torch.int32, device="cuda")
for _ in range(4):
    prog.run(x, pd, y)
torch.cuda.synchronize()
print("ok")
