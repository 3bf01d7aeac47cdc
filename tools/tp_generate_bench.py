"""Greedy generation through the tensor-parallel decoder on ONE GPU (LocalComm: every rank in one
process, lockstep), BASELINE config-2 model, 64 tokens: eager vs one CUDA graph per decode step,
and the 1-GPU DecodeEngine for reference.  Wall-clock from the host."""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.schedule import PrecisionSchedule, StaticScheduler
from paper_2410_13461_b200.tpmodel import LocalComm, TPModel

cfg = tinylm.ModelConfig(n_layers=24, n_heads=16, d_model=2048, d_ff=5632, vocab_size=32000, max_context=400)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
prompt = np.random.default_rng(7).integers(0, 32000, size=128).tolist()
N = 64
sch = StaticScheduler(PrecisionSchedule((3, 2), 4, {3: 0, 2: 16}, N))


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t) * 1e3


ref, t1 = timed(lambda: tinylm.generate(model, prompt, sch, eos_id=-1, max_new=N))
res = {"1-GPU engine ms": round(t1, 1)}
for tp in (1, 2):
    m = TPModel(model, tp, LocalComm(tp))
    for graph in (False, True):
        tr, t = timed(lambda: m.generate(prompt, sch, eos_id=-1, max_new=N, graph=graph))
        res[f"tp{tp} {'graph' if graph else 'eager'} ms"] = round(t, 1)
        res[f"tp{tp} {'graph' if graph else 'eager'} same tokens"] = tr.output_tokens == ref.output_tokens
print(json.dumps({"tokens": N, "prompt": len(prompt), **res}))
