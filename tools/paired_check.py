"""Paired (k-sliced row-parallel ops) vs plain engine program on the 7B linear stack: logits
agreement and µs/token at p = 4, 3, 2."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack

st = LinearStack(LLAMA2_7B, seed=1)
res = {}
for paired in (False, True):
    st.build_engine(paired=paired)
    g = st.capture(st.token_engine)
    for p in (4, 3, 2):
        st.set_schedule({p: 0})
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        lg = st.logits.clone()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        again = torch.equal(lg, st.logits)
        res[(paired, p)] = lg
        print(f"paired={paired} p={p}: {us:8.1f} us/token  reproducible={again}  status={int(st.program.status.item())}",
              flush=True)
for p in (4, 3, 2):
    a, b = res[(False, p)].double(), res[(True, p)].double()
    print(f"p={p}: rel-L2(paired vs plain) = {((a - b).norm() / a.norm()).item():.3e}")
