"""Prefill wall time (CUDA events) of the BASELINE config-2 model at several prompt lengths."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000, max_context=1032)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
res = {}
for n in (32, 64, 128, 256, 512):
    prompt = np.random.default_rng(7).integers(0, 32000, size=n).tolist()
    ts = []
    for _ in range(3):
        c = tinylm.KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        tinylm._forward(model, 4, prompt, c)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[n] = round(min(ts), 3)
print(json.dumps({"sdpa_min_rows": os.environ.get("PMPD_SDPA_MIN_ROWS", "256"), "prefill_ms": res}))
