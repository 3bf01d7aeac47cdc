"""Debug: progressive decode vs oracle with the prompt run through the GEMM (f16 weights) or token by token (GEMV)."""
import sys; sys.path.insert(0, "tests")
import numpy as np
from oracle import model as om
from paper_2410_13461_b200 import quant, tinylm
from pmpd_testutil import rel_l2
ARGS = dict(n_layers=2, n_heads=4, d_model=256, d_ff=512, max_context=160)
PROMPT = list(b"Old maps mark the mountain")
mv = tinylm.ModelVariants.from_random(tinylm.ModelConfig(**ARGS), quant.PrecisionSet((4, 3, 2)), seed=5)
om_ = om.Model.from_random(om.Config(**ARGS), (4, 3, 2), seed=5)
h = lambda t: t.double().cpu().numpy()
for mode in ("gemm", "gemv"):
    ref, cache = om.prefill(om_, 4, PROMPT)
    if mode == "gemm":
        one, c1 = tinylm.prefill(mv, 4, PROMPT)
    else:
        one, c1 = tinylm.prefill(mv, 4, PROMPT[:1])
        for t in PROMPT[1:]:
            one, c1 = tinylm.decode_step(mv, 4, t, c1)
    out = [f"{rel_l2(h(one), ref):.1e}"]
    tok = om.greedy(ref)
    for i, pd in enumerate((4, 4, 4, 3, 3, 2)):
        ref, cache = om.decode_step(om_, pd, tok, cache); one, c1 = tinylm.decode_step(mv, pd, tok, c1)
        out.append(f"{pd}/{tok}:{rel_l2(h(one), ref):.1e}")
        tok = om.greedy(ref)
    print(mode, " ".join(out))
