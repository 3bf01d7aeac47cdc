"""Per-shape GEMV timing probe (CUDA events, rotating weight copies > L2)."""
import argparse
import math
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import Workspace, gemv, workspace_bytes
from paper_2410_13461_b200.quant import quantize_tensor

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="4096x4096,4096x22016,11008x4096,4096x32000")  # KxN
ap.add_argument("--copies", type=int, default=0)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--layout", default="kn")
ap.add_argument("--graph", action="store_true")
ap.add_argument("--p", default="4,3,2")
args = ap.parse_args()
lay = _capi.LAYOUT_KN if args.layout == "kn" else _capi.LAYOUT_NK
torch.manual_seed(0)
for spec in args.shapes.split(","):
    K, N = (int(v) for v in spec.split("x"))
    per = K * N * 0.625  # bytes at p=4 incl scales
    copies = args.copies or max(2, int(math.ceil(400e6 / per)))
    pks = []
    for c in range(copies):
        w = torch.randn(K, N, device="cuda") * 0.02
        if lay == _capi.LAYOUT_NK:
            w = w.t().contiguous()
        qt = quantize_tensor(w, 4, 64)
        pks.append(qt.packed(lay))
        qt.drop_reference_copy()
        del w
    ws = Workspace(workspace_bytes(pks[0], args.m))
    x = torch.randn(args.m, K, device="cuda").half()
    y = torch.empty(args.m, N, device="cuda")
    for p in [int(v) for v in args.p.split(",")]:
        pd = torch.tensor([p], dtype=torch.int32, device="cuda")
        for i in range(3):
            gemv(pks[i % copies], x, pd, ws, out=y)
        torch.cuda.synchronize()
        if args.graph:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                gemv(pks[0], x, pd, ws, out=y)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                for i in range(copies):
                    gemv(pks[i], x, pd, ws, out=y)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            g.replay(); torch.cuda.synchronize()
            e0.record()
            for _ in range(max(1, args.iters // copies)):
                g.replay()
            e1.record(); torch.cuda.synchronize()
            n = max(1, args.iters // copies) * copies
        else:
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for i in range(args.iters):
                gemv(pks[i % copies], x, pd, ws, out=y)
            e1.record(); torch.cuda.synchronize()
            n = args.iters
        us = e0.elapsed_time(e1) * 1e3 / n
        byt = pks[0].stream_bytes(p)
        print(f"K={K} N={N} p={p} m={args.m} copies={copies} graph={args.graph}: {us:8.2f} us  {byt/us/1e3:8.1f} GB/s",
              flush=True)
