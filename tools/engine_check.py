"""Engine determinism + accuracy check on small stacks (run on the GPU box)."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_13461_b200.stack import LinearStack, StackShape
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_engine import _chain_f64
from pmpd_testutil import rel_l2
for shape in (StackShape(1, 512, 1408, 2048), StackShape(2, 256, 512, 1000), StackShape(1, 4096, 11008, 32000)):
    st = LinearStack(shape, seed=3)
    st.build_engine()
    for p in (4, 3, 2):
        ref = _chain_f64(st, p).cpu().numpy() if shape.d_model < 4096 else None
        st.set_schedule({p: 0}); st.token(); per_op = st.logits.clone().cpu().numpy()
        outs = []
        for r in range(5):
            st.set_schedule({p: 0}); st.logits.zero_(); st.token_engine(); torch.cuda.synchronize()
            outs.append(st.logits.clone().cpu().numpy())
        det = all(np.array_equal(outs[0], o) for o in outs[1:])
        msg = f"{shape} p={p} deterministic={det} eng-vs-perop {rel_l2(outs[0], per_op):.2e}"
        if ref is not None:
            msg += f" eng-vs-f64 {rel_l2(outs[0], ref):.2e} perop-vs-f64 {rel_l2(per_op, ref):.2e}"
        print(msg, flush=True)
