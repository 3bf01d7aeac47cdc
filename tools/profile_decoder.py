"""A few decode steps of the BASELINE config-2 decoder through the decoder engine (for ncu:
`ncu -k regex:engine_kernel -s 2 -c 1 ... python tools/profile_decoder.py`)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler

cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000, max_context=400)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
prompt = np.random.default_rng(7).integers(0, 32000, size=128).tolist()
sch = StaticScheduler(PrecisionSchedule((3, 2), 4, {3: 0, 2: 1}, 256))
tr = tinylm.generate(model, prompt, sch, eos_id=-1, max_new=int(sys.argv[1]) if len(sys.argv) > 1 else 8,
                     check_every=1)
torch.cuda.synchronize()
print("ok", tr.output_tokens[:4])
