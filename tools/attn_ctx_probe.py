"""Probe: decode-engine attention vs per-op attention kernel vs the oracle across context lengths.

Generates greedily with ``generate`` (persistent decoder engine) and ``generate_batch`` (per-op
GEMVs + pmpd_attention_rope) and prints, per decode row, the logits difference between the two
and each one's rel-L2 against the float64 oracle fed the same tokens."""
import sys
sys.path.insert(0, "tests")
import numpy as np
from oracle import model as om
from oracle import schedule as osched
from paper_2410_13461_b200 import quant, tinylm
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler
from pmpd_testutil import rel_l2

nh, d = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (4, 512)
P0 = int(sys.argv[3]) if len(sys.argv) > 3 else 128
N = int(sys.argv[4]) if len(sys.argv) > 4 else 96
ARGS = dict(n_layers=2, n_heads=nh, d_model=d, d_ff=2 * d, vocab_size=512, max_context=P0 + N + 8)
mv = tinylm.ModelVariants.from_random(tinylm.ModelConfig(**ARGS), quant.PrecisionSet((4, 3, 2)), seed=3)
prompt = [int(t) for t in np.random.default_rng(1).integers(0, 512, P0)]
sch = StaticScheduler(PrecisionSchedule((4,), 4, {4: 0}, N))
a = tinylm.generate(mv, prompt, sch, eos_id=-1, max_new=N, record_logits=True)
b = tinylm.generate_batch(mv, [prompt], sch, eos_id=-1, max_new=N, record_logits=True)[0]
om_ = om.Model.from_random(om.Config(**ARGS), (4, 3, 2), seed=3)
toks = a.output_tokens
la, lb = a.logits.double().cpu().numpy(), b.logits.double().cpu().numpy()
ref, cache = om.prefill(om_, 4, prompt)
_, c1 = tinylm.prefill(mv, 4, prompt)
shown = 0
for i in range(1, N):
    ref, cache = om.decode_step(om_, 4, toks[i - 1], cache)
    lc, c1 = tinylm.decode_step(mv, 4, toks[i - 1], c1)
    ea, eb, ec = rel_l2(la[i], ref), rel_l2(lb[i], ref), rel_l2(lc.double().cpu().numpy(), ref)
    if (max(ea, eb, ec) > 3e-3 and shown < 6) or i % 16 == 0:
        shown += max(ea, eb, ec) > 3e-3
        print(f"row {i} T={P0 + i - 1} engine {ea:.1e} batch {eb:.1e} eager-decode {ec:.1e}")
print("tokens identical", a.output_tokens == b.output_tokens)
