"""Time the 7B linear stack per token through the persistent engine (graph replays); with
``--per-op`` also the per-op GEMV chain.  PMPD_LIB selects a library variant."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack, algorithmic_bytes

st = LinearStack(LLAMA2_7B, seed=1)
st.build_engine()
fns = (("per-op", st.token), ("engine", st.token_engine)) if "--per-op" in sys.argv else (("engine", st.token_engine),)
for name, fn in fns:
    g = st.capture(fn)
    for p in (4, 3, 2):
        st.set_schedule({p: 0})
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        print(f"{name:7s} p={p}: {us:8.1f} us/token  {algorithmic_bytes(LLAMA2_7B, p) / us / 1e3:7.1f} GB/s", flush=True)
