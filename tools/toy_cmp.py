"""Diagnostics: toy-model incremental-vs-full and vs-golden rel-L2 per precision (run with and
without PMPD_ATTN_GENERIC=1 to compare the split and generic attention kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from pmpd_testutil import rel_l2, load_golden
from paper_2410_13461_b200 import quant, tinylm

g = load_golden("model.npz")
cfg = tinylm.ModelConfig(n_layers=4, n_heads=4, d_model=128, d_ff=256, max_context=256)
toy = tinylm.ModelVariants.from_random(cfg, quant.PrecisionSet((4, 3, 2)), seed=11)
toks = [int(t) for t in g["toy/tokens"]]
host = lambda t: t.double().cpu().numpy()
for p in (2, 3, 4, 16):
    full = host(tinylm.forward_full(toy, p, toks))
    _, cache = tinylm.prefill(toy, p, toks[:1])
    got = [host(tinylm.forward_full(toy, p, toks[:1])[0])]
    for t in toks[1:]:
        lg, cache = tinylm.decode_step(toy, p, t, cache)
        got.append(host(lg))
    got = np.array(got)
    print(f"p={p} generic={os.environ.get('PMPD_ATTN_GENERIC')} full_vs_gold={rel_l2(full, g[f'toy/full{p}']):.2e} "
          f"inc_vs_full={rel_l2(got, full):.2e} inc_vs_gold={rel_l2(got, g[f'toy/full{p}']):.2e}")
