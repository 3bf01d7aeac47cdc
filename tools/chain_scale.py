"""RMS of the synthetic 7B linear chain's activations per layer at p = 4, 3, 2 (per-op GEMVs),
and the engine status word after one token."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import torch
from paper_2410_13461_b200.linear import gemv
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1234
st = LinearStack(LLAMA2_7B, seed=seed)
d, f = st.shape.d_model, st.shape.d_ff
a_d = 1.0 / (st.std * math.sqrt(d))
a_f = 1.0 / (st.std * math.sqrt(f))
for p in (4, 3, 2):
    st.p_dev.fill_(p)
    inp = st.x0
    rms = []
    for (_, wqkv), (_, wo), (_, wup), (_, wdn) in st.layers:
        gemv(wqkv, inp, st.p_dev, st.ws, out=st.qkv, alpha=a_d)
        gemv(wo, st.qkv[:, 2 * d:], st.p_dev, st.ws, out=st.o, alpha=a_d)
        gemv(wup, st.o, st.p_dev, st.ws, out=st.u, alpha=a_d)
        gemv(wdn, st.u[:, :f], st.p_dev, st.ws, out=st.h, alpha=a_f)
        inp = st.h
        rms.append(st.h.float().pow(2).mean().sqrt().item())
    print(f"p={p}: rms per layer " + " ".join(f"{r:.3g}" for r in rms[::4]) + f" ... last {rms[-1]:.3g}", flush=True)
st.build_engine(paired=False)
for p in (4, 3, 2):
    st.set_schedule({p: 0})
    st.program.status.zero_()
    st.token_engine()
    torch.cuda.synchronize()
    print(f"engine p={p}: status {int(st.program.status.item())}, logits rms {st.logits.pow(2).mean().sqrt().item():.3g}")
