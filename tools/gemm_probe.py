"""Prefill GEMM probe: time pmpd_gemm per forced tile configuration.

usage: gemm_probe.py M K N [ng,mb,sk ...]   (default: the library's own choice, then every config)
PMPD_LIB selects a library variant (tools/build_variant.sh gemm <tag> -D...).  f32 output, p = 4.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import gemm
from paper_2410_13461_b200.quant import quantize_tensor


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


M, K, N = (int(v) for v in sys.argv[1:4])
cfgs = sys.argv[4:] or ["default"] + [f"{a},{b},{s}" for a, b in ((1, 1), (1, 2), (1, 4), (2, 1), (2, 2), (2, 4),
                                                                  (4, 1), (4, 2)) for s in (1, 2, 4)]
P = int(os.environ.get("PROBE_P", "4"))
pk = quantize_tensor(torch.randn((K, N), device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
x = torch.randn((M, K), device="cuda").half()
y = torch.empty((M, N), device="cuda", dtype=torch.float32)
pd = torch.tensor([P], dtype=torch.int32, device="cuda")
ref = None
for c in cfgs:
    os.environ.pop("PMPD_GEMM_CFG", None)
    os.environ.pop("PMPD_GEMM_SPLITK", None)
    if c != "default":
        a, b, s = c.split(",")
        os.environ["PMPD_GEMM_CFG"] = f"{a},{b}"
        os.environ["PMPD_GEMM_SPLITK"] = s
    us = timeit(lambda: gemm(pk, x, pd, out=y))
    if ref is None:
        ref = y.clone()
    err = float((y - ref).norm() / ref.norm())
    print(json.dumps(dict(M=M, K=K, N=N, p=P, cfg=c, us=round(us, 2), tflops=round(2 * M * N * K / us / 1e6, 1),
                          dev=f"{err:.1e}")), flush=True)
