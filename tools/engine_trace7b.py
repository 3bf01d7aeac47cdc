"""Per-op timeline of one 7B-shape token through the persistent engine (globaltimer per CTA).
Saves gpurun_out/trace7b_p{p}.npz with int64 [grid, n_ops, 8]; prints a critical-path summary."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st = LinearStack(LLAMA2_7B, seed=1)
prog = st.build_engine()
st.set_schedule({p: 0})
pd = torch.tensor([p], dtype=torch.int32, device="cuda")
for _ in range(4):
    tr = prog.run_traced(st.x0, pd, st.logits)
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/trace7b_p{p}{os.environ.get('TAG', '')}.npz", tr=tr.numpy())
t = tr[:, :, :4].numpy().astype(np.float64)
t0 = t[t > 0].min()
t = (t - t0) / 1e3
print("total us", t[:, -1, 3].max())
