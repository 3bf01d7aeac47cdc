import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2410_13461_b200.stack import LinearStack, StackShape
from test_gpu_engine import _chain_f64
from pmpd_testutil import rel_l2
for trial in range(6):
    for shape in (StackShape(2, 256, 512, 1000), StackShape(1, 512, 1408, 2048)):
        st = LinearStack(shape, seed=3)
        st.build_engine()
        for p in (4, 2):
            ref = _chain_f64(st, p).cpu().numpy()
            ref2 = _chain_f64(st, p).cpu().numpy()
            st.set_schedule({p: 0}); st.token(); per_op = st.logits.clone().cpu().numpy()
            st.set_schedule({p: 0}); st.token_engine(); torch.cuda.synchronize(); eng = st.logits.cpu().numpy()
            bad = rel_l2(per_op, ref) > 5e-3 or rel_l2(eng, ref) > 5e-3
            import hashlib
            h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
            print(f"hash ref {h(ref)} perop {h(per_op)} eng {h(eng)} x0 {h(st.x0.cpu().numpy())}", end=" ")
            print(f"t{trial} {shape.d_model}/{shape.d_ff} p={p} ref-det {np.array_equal(ref, ref2)} perop {rel_l2(per_op, ref):.2e} eng {rel_l2(eng, ref):.2e} eng-perop {rel_l2(eng, per_op):.2e} {'BAD' if bad else ''}", flush=True)
