"""One BASELINE config-2 prefill (1.4B shape, 128 prompt ids, 4-bit) after warm-up (graph capture),
for an ncu launch list: prefill_profile2.py [p]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000, max_context=400)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
prompt = np.random.default_rng(7).integers(0, 32000, size=128).tolist()
for _ in range(3):
    c = tinylm.KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    tinylm._forward(model, p, prompt, c)
    e1.record()
    torch.cuda.synchronize()
    print(f"prefill p={p}: {e0.elapsed_time(e1):.3f} ms", flush=True)
