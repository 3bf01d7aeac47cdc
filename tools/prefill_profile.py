"""One BASELINE config-3 prefill (7B shape, 512 prompt ids, 4-bit) after a warm-up, for an ncu launch list."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet

cfg = tinylm.ModelConfig(n_layers=32, n_heads=32, d_model=4096, d_ff=11008, vocab_size=32000, max_context=1032)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
prompt = np.random.default_rng(7).integers(0, 32000, size=512).tolist()
for _ in range(2):
    c = tinylm.KVCache(cfg.n_layers, cfg.d_model, cfg.max_context)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    tinylm._forward(model, 4, prompt, c)
    e1.record()
    torch.cuda.synchronize()
    print("prefill ms", e0.elapsed_time(e1), flush=True)
