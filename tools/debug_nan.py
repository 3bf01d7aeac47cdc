import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, math
from paper_2410_13461_b200.stack import LinearStack, StackShape
st = LinearStack(StackShape(2, 1024, 2816, 4000), seed=4)
st.build_engine()
for p in (4, 2):
    st.set_schedule({p: 0})
    outs = []
    for _ in range(5):
        st.token_engine()
        outs.append(st.logits.clone())
    torch.cuda.synchronize()
    print(p, [bool(o.isnan().any()) for o in outs], [bool(torch.equal(o, outs[0])) for o in outs], float(outs[0].abs().max()))
    st.token(); torch.cuda.synchronize()
    print("per-op", bool(st.logits.isnan().any()), float(st.logits.abs().max()), "status", int(st.program.status.item()))
    print("p_dev", int(st.p_dev.item()), "step", int(st.step.item()))
