"""Calibrated partition probe: plain engine program vs the same program re-partitioned with per-CTA
budget reductions measured from traced tokens (engine.calibrate_deltas)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13461_b200.engine import calibrate_deltas
from paper_2410_13461_b200.stack import LLAMA2_7B, LinearStack


def timeit(st):
    g = st.capture(st.token_engine)
    out = {}
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
        out[p] = e0.elapsed_time(e1) * 1e3 / 20
    return out


st = LinearStack(LLAMA2_7B, seed=1)
st.build_engine()
print("plain", {p: round(v, 1) for p, v in timeit(st).items()}, flush=True)
for unit in (0.25, 0.15):
    st.build_engine()
    st.set_schedule({2: 0})
    pd = torch.tensor([2], dtype=torch.int32, device="cuda")
    delta = calibrate_deltas(st.program, st.x0, pd, st.logits, unit_us=unit)
    print("unit", unit, "deltas: nonzero", sum(1 for v in delta if v), "max", max(delta), "sum", sum(delta), flush=True)
    st.build_engine(cta_delta=delta)
    print("calibrated", {p: round(v, 1) for p, v in timeit(st).items()}, flush=True)
    # second pass: refine on top of the calibrated partition
    d2 = calibrate_deltas(st.program, st.x0, pd, st.logits, unit_us=unit)
    delta2 = [min(8, a + b) for a, b in zip(delta, d2)]
    st.build_engine(cta_delta=delta2)
    print("calibrated x2", {p: round(v, 1) for p, v in timeit(st).items()}, "sum", sum(delta2), flush=True)
