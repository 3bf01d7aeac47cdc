"""One config-2 batched decode run (B prompts, few tokens) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000, max_context=200)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
rng = np.random.default_rng(7)
prompts = [rng.integers(0, 32000, size=128).tolist() for _ in range(B)]
sch = StaticScheduler(PrecisionSchedule((3, 2), 4, {3: 0, 2: 64}, 256))
tr = tinylm.generate_batch(model, prompts, sch, eos_id=-1, max_new=6)
torch.cuda.synchronize()
print("ok", [t.output_tokens[:3] for t in tr][:2])
