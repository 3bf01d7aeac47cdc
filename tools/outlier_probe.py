import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from oracle import quant as oq
from paper_2410_13461_b200 import _capi, quant
from paper_2410_13461_b200.linear import Workspace, gemv
from paper_2410_13461_b200.engine import OpSpec, Program
from pmpd_testutil import rel_l2
rng = np.random.default_rng(17)
K, N = 4096, 4096
w = (0.02 * rng.standard_normal((K, N))).astype(np.float32)
ref = oq.quantize(w, 4, 64)
pk = quant.quantize_tensor(w, 4, 64).packed(_capi.LAYOUT_KN)
ws = Workspace()
prog = Program([OpSpec(pk)])
for scale in (1.0, 10.0, 100.0, 1000.0):
    for M in (1, 2, 4, 8):
        x = rng.standard_normal((M, K))
        x[:, rng.choice(K, 6, replace=False)] *= scale
        x = x.astype(np.float16)
        for p in (4, 2):
            y = gemv(pk, torch.from_numpy(x).cuda(), torch.tensor([p], dtype=torch.int32, device="cuda"), ws)
            want = x.astype(np.float64) @ oq.dequantize(ref, p)
            e = rel_l2(y.cpu().numpy(), want)
            s = ""
            if M == 1:
                yy = torch.zeros(N, device="cuda")
                prog.run(torch.from_numpy(x).cuda(), torch.tensor([p], dtype=torch.int32, device="cuda"), yy)
                s = f" engine {rel_l2(yy.cpu().numpy(), want[0]):.2e}"
            print(f"scale {scale:6.0f} M {M} p {p}: gemv {e:.2e}{s}", flush=True)
