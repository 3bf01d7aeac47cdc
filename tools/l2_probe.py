"""Per-layer engine time with the weights L2-resident (a 1-layer 7B-width stack, small head) vs
streamed from HBM (32 layers): how much of a layer is memory, how much the op chain + compute."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.stack import LinearStack, StackShape
for L, V in ((1, 4096), (2, 4096), (32, 4096)):
    st = LinearStack(StackShape(L, 4096, 11008, V), seed=1)
    st.build_engine()
    g = st.capture(st.token_engine)
    for p in (4, 2):
        st.set_schedule({p: 0})
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 50
        print(f"L={L} p={p}: {us:8.1f} us/token, {us / L:6.2f} us/layer (incl. head)", flush=True)
    del st, g
    torch.cuda.empty_cache()
