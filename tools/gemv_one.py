"""One pmpd_gemv shape at batch m, a few launches (for ncu captures): gemv_one.py K N m p"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.linear import Workspace, gemv, workspace_bytes
from paper_2410_13461_b200.quant import quantize_tensor

K, N, m, p = (int(v) for v in sys.argv[1:5])
torch.manual_seed(0)
pk = quantize_tensor(torch.randn(K, N, device="cuda") * 0.02, 4, 64).packed()
ws = Workspace(workspace_bytes(pk, m))
x = torch.randn(m, K, device="cuda").half()
pd = torch.tensor([p], dtype=torch.int32, device="cuda")
for _ in range(6):
    y = gemv(pk, x, pd, ws)
torch.cuda.synchronize()
print("ok", float(y.float().norm()))
