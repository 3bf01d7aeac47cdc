"""Tiny linear-stack engine launch (sanitizer / debugging target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.stack import LinearStack, StackShape

dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,256,512,1000").split(",")]
st = LinearStack(StackShape(*dims), seed=3)
st.build_engine()
for p in (4, 2):
    st.set_schedule({p: 0})
    for _ in range(3):
        st.token_engine()
    torch.cuda.synchronize()
print("ok", st.logits[:4].tolist())
