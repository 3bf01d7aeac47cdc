"""n-group grid vs split-K grid for the decode GEMV across batch sizes (CUDA-graph timing, L2-resident
weights are avoided by rotating 8 copies).  python tools/gemv_grid_sweep.py; set PMPD_GEMV_SPLITK=1
in the environment to force the split-K grid."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.linear import Workspace, gemv, workspace_bytes
from paper_2410_13461_b200.quant import quantize_tensor

shapes = [(2048, 2048), (5632, 2048), (2048, 6144), (4096, 4096), (11008, 4096), (4096, 1536), (1376, 4096)]
torch.manual_seed(0)
out = {}
for K, N in shapes:
    pks = [quantize_tensor(torch.randn(K, N, device="cuda") * 0.02, 4, 64).packed() for _ in range(8)]
    for m in (1, 4, 8):
        ws = Workspace(max(workspace_bytes(pk, m) for pk in pks))
        x = torch.randn(m, K, device="cuda").half()
        y = torch.empty(m, N, device="cuda")
        pd = torch.tensor([2], dtype=torch.int32, device="cuda")
        for pk in pks:
            gemv(pk, x, pd, ws, out=y)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(4):
                for pk in pks:
                    gemv(pk, x, pd, ws, out=y)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[f"{K}x{N} m{m}"] = round(e0.elapsed_time(e1) * 1e3 / (5 * 32), 2)
    del pks
print(json.dumps(out))
