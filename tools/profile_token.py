"""One-token workloads for ncu: the 7B linear stack through the engine and the per-op chain."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "engine"
st = LinearStack(LLAMA2_7B, seed=1)
st.build_engine()
st.set_schedule({p: 0})
fn = st.token_engine if mode == "engine" else st.token
for _ in range(4):
    fn()
torch.cuda.synchronize()
print("ok")
