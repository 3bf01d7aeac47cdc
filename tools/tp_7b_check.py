"""Full-size check of the tensor-parallel decoder: Llama-2-7B shape (random init N(0, 0.02^2)),
tp = 2 / 4 / 8 on ONE GPU (LocalComm), prefill 32 ids at 4 bits + 8 progressive decode steps,
logits vs the 1-GPU model (rel-L2) and greedy tokens."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import tinylm
from paper_2410_13461_b200.quant import PrecisionSet
from paper_2410_13461_b200.tpmodel import LocalComm, TPModel

cfg = tinylm.ModelConfig(n_layers=32, n_heads=32, d_model=4096, d_ff=11008, vocab_size=32000, max_context=64)
model = tinylm.ModelVariants.from_random(cfg, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
prompt = np.random.default_rng(7).integers(0, 32000, size=32).tolist()
ps = [4, 4, 3, 3, 3, 2, 2, 2]
one, c1 = tinylm.prefill(model, 4, prompt)
ref = [one.double().cpu().numpy()]
tok = int(torch.argmax(one))
toks = [tok]
for p in ps:
    one, c1 = tinylm.decode_step(model, p, tok, c1)
    ref.append(one.double().cpu().numpy())
    tok = int(torch.argmax(one))
    toks.append(tok)
res = {}
for tp in (2, 4, 8):
    m = TPModel(model, tp, LocalComm(tp))
    got = [m.prefill(4, prompt).double().cpu().numpy()]
    for p, t in zip(ps, toks):
        got.append(m.decode_step(p, t).double().cpu().numpy())
    err = [float(np.linalg.norm(g - r) / np.linalg.norm(r)) for g, r in zip(got, ref)]
    res[f"tp{tp}"] = {"max_rel_l2": max(err), "argmax_same": all(int(np.argmax(g)) == int(np.argmax(r))
                                                                 for g, r in zip(got, ref))}
    del m
    torch.cuda.empty_cache()
print(json.dumps(res))
