import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_13461_b200 import _capi
from paper_2410_13461_b200.engine import OpSpec, Program
from paper_2410_13461_b200.quant import quantize_tensor
torch.manual_seed(0)
def mk(K, N):
    return quantize_tensor(torch.randn(K, N, device="cuda") * 0.02, 4, 64).packed(_capi.LAYOUT_KN)
o = mk(4096, 4096); up = mk(4096, 22016)
x = torch.randn(1, 4096, device="cuda").half()
pd = torch.tensor([2], dtype=torch.int32, device="cuda")
for name, ops in (("o x4", [OpSpec(o)] + [OpSpec(o, src=i) for i in range(3)]), ("up,o", [OpSpec(up), OpSpec(o, src=0)])):
    prog = Program(ops)
    y = torch.zeros(ops[-1].packed.desc.n, device="cuda")
    for _ in range(3):
        tr = prog.run_traced(x, pd, y)
    cyc = tr[:, :, 4:7].clone()
    tt = tr[:, :, :4]
    t0 = tt[tt > 0].min()
    tr = (tt - t0).float() / 1000.0  # us
    print(f"== {name}")
    for oi in range(len(ops)):
        col = tr[:, oi, :]
        valid = col[:, 3] > 0
        print(f" op{oi}: ready med {col[:,0].median():6.2f} max {col[:,0].max():6.2f} | staged med {col[:,1].median():6.2f} max {col[:,1].max():6.2f}"
              f" | tiles med {col[:,2].median():6.2f} max {col[:,2].max():6.2f} | publish med {col[valid,3].median():6.2f} max {col[:,3].max():6.2f}")
        cc = cyc[:, oi, :].float()
        m = cc[:, 1] > 0
        if m.any():
            print(f"       warp0: tile calls {cc[m,1].median():.0f}, cycles/call {float((cc[m,0]/cc[m,1]).median()):.0f}, "
                  f"tile share of loop {float((cc[m,0]/cc[m,2]).median()):.2f}")
