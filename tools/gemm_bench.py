"""Prefill GEMM throughput on the BASELINE config-4 shapes (M = 512, 2048): pmpd_gemm vs cuBLAS fp16."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import gemm
from paper_2410_13461_b200.quant import quantize_tensor

def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps  # us

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["bf16_tflops"]
rows = []
shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (2048, 5632), (5632, 2048), (32000, 4096)]
if len(sys.argv) > 1:
    shapes = shapes[:int(sys.argv[1])]
for N, K in shapes:
    w = torch.randn((K, N), device="cuda") * 0.02
    pk = quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
    wt = w.t().contiguous().half()
    for M in (512, 2048):
        x = torch.randn((M, K), device="cuda").half()
        y = torch.empty((M, N), device="cuda", dtype=torch.float32)  # f32 as the model runner uses
        y16 = torch.empty((M, N), device="cuda", dtype=torch.float16)
        for p in (4, 2):
            pd = torch.tensor([p], dtype=torch.int32, device="cuda")
            us = timeit(lambda: gemm(pk, x, pd, out=y))
            tf = 2 * M * N * K / us / 1e6
            rows.append(dict(N=N, K=K, M=M, p=p, us=round(us, 2), tflops=round(tf, 1), frac=round(tf / peak, 3)))
            print(json.dumps(rows[-1]), flush=True)
        us = timeit(lambda: torch.matmul(x, wt.t(), out=y16))
        tf = 2 * M * N * K / us / 1e6
        rows.append(dict(N=N, K=K, M=M, p="cublas_fp16", us=round(us, 2), tflops=round(tf, 1), frac=round(tf / peak, 3)))
        print(json.dumps(rows[-1]), flush=True)
    del w, pk, wt
