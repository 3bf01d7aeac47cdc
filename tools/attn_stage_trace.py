"""o-op staging after attention, sub-steps (library built with -DPMPD_ENGINE_TRACE_ATTNSTAGE):
median over o CTAs of ready / records read / (m, l) read / staged, relative to the last attention
unit's end, per layer (config 2 or 3 decoder)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import _capi, tinylm
from paper_2410_13461_b200.quant import PrecisionSet

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
shape = dict(n_layers=24, n_heads=16, d_model=2048, d_ff=5632) if cfgn == 2 else \
    dict(n_layers=32, n_heads=32, d_model=4096, d_ff=11008)
ctx = 384 if cfgn == 2 else 1024
mc = tinylm.ModelConfig(vocab_size=32000, max_context=ctx + 8, **shape)
model = tinylm.ModelVariants.from_random(mc, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
eng = tinylm.DecodeEngine(model, 8)
prompt = list(np.random.default_rng(7).integers(0, 32000, size=ctx // 2))
tinylm._forward(model, 4, prompt, eng.cache)
eng.buf.p.fill_(2)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _capi.call("pmpd_gather_rows", eng.dw.embed.ref(), eng.buf.ids.data_ptr(), 1, eng.buf.p.data_ptr(),
               eng.buf.x.data_ptr(), s)
    tr = eng.program.run_traced(eng.buf.x, eng.buf.p, eng.buf.logits).numpy().astype(np.float64)
n_ops = tr.shape[1]
rows = []
for i in range(1, n_ops - 1):
    if i % 5 != 1:
        continue  # attention ops
    att_end = np.nanmax(np.where(tr[:, i, 2] > 0, tr[:, i, 2], np.nan))
    o = i + 1
    busy = tr[:, o, 1] > 0
    r0 = np.median(tr[busy, o, 0]) - att_end
    r4 = np.median(tr[busy, o, 4]) - att_end
    r5 = np.median(tr[busy, o, 5]) - att_end
    r1 = np.median(tr[busy, o, 1]) - att_end
    last_rec = np.max(tr[busy, o, 4]) - att_end
    rows.append((r0, r4, r5, r1, last_rec))
r = np.array(rows) / 1e3
print(f"config {cfgn}: relative to the last unit's end (us), mean over layers:")
print(f"  o ready {r[:,0].mean():6.2f}  records read {r[:,1].mean():6.2f} (last CTA {r[:,4].mean():6.2f})  "
      f"(m,l) read {r[:,2].mean():6.2f}  staged {r[:,3].mean():6.2f}")
