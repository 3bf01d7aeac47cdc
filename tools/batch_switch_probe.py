"""Probe: generate (engine) vs generate_batch (per-op) logits per row around a precision switch."""
import sys
sys.path.insert(0, "tests")
import numpy as np
import torch
from paper_2410_13461_b200 import quant, tinylm
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler
from pmpd_testutil import rel_l2

nh, d, P0, S, N = (int(a) for a in sys.argv[1:6])
L, FF, V = (int(a) for a in sys.argv[6:9]) if len(sys.argv) > 8 else (2, 2 * d, 2048)
SEED, PSEED = (int(a) for a in sys.argv[9:11]) if len(sys.argv) > 10 else (3, 1)
ARGS = dict(n_layers=L, n_heads=nh, d_model=d, d_ff=FF, vocab_size=V, max_context=P0 + N + 8)
mv = tinylm.ModelVariants.from_random(tinylm.ModelConfig(**ARGS), quant.PrecisionSet((4, 3, 2)), seed=SEED, std=0.02)
prompt = [int(t) for t in np.random.default_rng(PSEED).integers(0, V, P0)]
sch = StaticScheduler(PrecisionSchedule((3, 2), 4, {3: 0, 2: S}, N))
a = tinylm.generate(mv, prompt, sch, eos_id=-1, max_new=N, record_logits=True)
b = tinylm.generate_batch(mv, [prompt], sch, eos_id=-1, max_new=N, record_logits=True)[0]
la, lb = a.logits.double().cpu().numpy(), b.logits.double().cpu().numpy()
ta, tb = a.output_tokens, b.output_tokens
first = next((k for k in range(N) if ta[k] != tb[k]), N)
for i in range(min(first + 1, N)):
    if abs(i - S) <= 2 or i == first or rel_l2(la[i], lb[i]) > 1e-2:
        top = np.sort(la[i])[-2:]
        print(f"row {i} p_at(row-1)={sch.resolve(None).precision_at(max(i - 1, 0))} diff {rel_l2(la[i], lb[i]):.1e} "
              f"margin {top[1] - top[0]:.3f} tok {ta[i]} {tb[i]}")
print("first token difference", first)
# third path: eager per-op decode_step with the precision passed from the host, fed a's tokens
sc = sch.resolve(None)
lc, c = tinylm.prefill(mv, sc.p_prefill, prompt)
for i in range(1, min(S + 3, N)):
    lc, c = tinylm.decode_step(mv, sc.precision_at(i - 1), ta[i - 1], c)
    if i >= S - 2:
        l3 = lc.double().cpu().numpy()
        print(f"row {i} eager vs engine {rel_l2(l3, la[i]):.1e} eager vs batch {rel_l2(l3, lb[i]):.1e}")
