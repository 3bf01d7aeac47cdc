"""Run one prefill GEMM configuration back to back for a few seconds while sampling SM clocks,
power and throttle reasons (nvidia-smi): does the dequant + tcgen05 mix run at full clock?"""
import os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.linear import gemm
from paper_2410_13461_b200.quant import quantize_tensor

M, K, N = (int(v) for v in sys.argv[1:4])
pk = quantize_tensor(torch.randn((K, N), device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
x = torch.randn((M, K), device="cuda").half()
y = torch.empty((M, N), device="cuda", dtype=torch.float32)
pd = torch.tensor([4], dtype=torch.int32, device="cuda")
samples, stop = [], False
def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.2)
for _ in range(10):
    gemm(pk, x, pd, out=y)
torch.cuda.synchronize()
th = threading.Thread(target=sampler); th.start()
t0 = time.time(); n = 0
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(200):
        gemm(pk, x, pd, out=y)
    n += 200
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
stop = True; th.join()
print(f"{os.environ.get('PMPD_LIB','main')}: {e0.elapsed_time(e1) * 1e3 / n:.2f} us/launch over {n}")
for s in samples[2:-1]: print("  ", s)
