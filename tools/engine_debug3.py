import os, sys, math, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.engine import OpSpec, Program
from paper_2410_13461_b200.linear import Workspace, gemv
from paper_2410_13461_b200.quant import quantize_tensor

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
pd = torch.tensor([2], dtype=torch.int32, device="cuda")
def mk(K, N):
    w = torch.randn(K, N, device="cuda") * 0.02
    return quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
torch.manual_seed(0)
d, f, V = 4096, 11008, 32000
qkv, o, up, dn, hd = mk(d, 3 * d), mk(d, d), mk(d, 2 * f), mk(f, d), mk(d, V)
x = torch.randn(1, d, device="cuda").half()
ws = Workspace(1 << 24)
def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
chains = {
    "o": [(o, -1, 0)], "up": [(up, -1, 0)], "down": [(dn, -1, 0)], "head": [(hd, -1, 0)],
    "qkv>o": [(qkv, -1, 0), (o, 0, 2 * d)], "o>up": [(o, -1, 0), (up, 0, 0)], "up>down": [(up, -1, 0), (dn, 0, 0)],
    "down>head": [(dn, -1, 0), (hd, 0, 0)], "o>o>o>o": [(o, -1, 0), (o, 0, 0), (o, 1, 0), (o, 2, 0)],
}
for name, ch in chains.items():
    xin = x if ch[0][0].desc.k == d else torch.randn(1, ch[0][0].desc.k, device="cuda").half()
    # reference chain with per-op gemv (f16 between ops)
    h = xin
    for i, (pk, src, col) in enumerate(ch):
        if i > 0:
            h = h[:, col:col + pk.desc.k].contiguous()
        h = gemv(pk, h, pd, ws, out_dtype=torch.float16 if i + 1 < len(ch) else torch.float32)
    ref = h[0].float().cpu().numpy()
    prog = Program([OpSpec(pk, src=src, src_col=col) for pk, src, col in ch])
    y = torch.zeros(ch[-1][0].desc.n, device="cuda")
    prog.run(xin, pd, y)
    torch.cuda.synchronize()
    r1 = rel(y.cpu().numpy(), ref)
    us = timeit(lambda: prog.run(xin, pd, y))
    print(f"{name:10s} rel-first {r1:.2e} rel-after {rel(y.cpu().numpy(), ref):.2e}  engine {us:8.1f} us  bar {prog.bar.tolist()} st {prog.status.tolist()}", flush=True)
