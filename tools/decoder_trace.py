"""Per-op timeline of one decode step through the decoder engine program (BASELINE config 2 or 3
shape, random weights): prints median phase times per op kind (ticket, staging, tiles, publish)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13461_b200 import _capi, tinylm
from paper_2410_13461_b200.quant import PrecisionSet

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape = dict(n_layers=24, n_heads=16, d_model=2048, d_ff=5632) if cfgn == 2 else \
    dict(n_layers=32, n_heads=32, d_model=4096, d_ff=11008)
ctx = 384 if cfgn == 2 else 1024
mc = tinylm.ModelConfig(vocab_size=32000, max_context=ctx + 8, **shape)
model = tinylm.ModelVariants.from_random(mc, PrecisionSet((4, 3, 2)), seed=1234, std=0.02)
eng = tinylm.DecodeEngine(model, 8)
assert eng.program is not None
prompt = list(np.random.default_rng(7).integers(0, 32000, size=ctx // 2))
tinylm._forward(model, 4, prompt, eng.cache)
eng.buf.p.fill_(p)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _capi.call("pmpd_gather_rows", eng.dw.embed.ref(), eng.buf.ids.data_ptr(), 1, eng.buf.p.data_ptr(),
               eng.buf.x.data_ptr(), s)
    tr = eng.program.run_traced(eng.buf.x, eng.buf.p, eng.buf.logits)
t = tr[:, :, :4].numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
n_ops = t.shape[1]
pub = np.nanmax(t[:, :, 3], axis=0)
print(f"ops {n_ops}, last publish {np.nanmax(pub):.1f} us")
kinds = ["qkv", "attn", "o", "up", "down"]
for k, nm in enumerate(kinds):
    idx = [i for i in range(n_ops - 1) if i % 5 == k]
    if nm == "attn":
        # attention ops stamp [0] unit start and [2] units done on the CTAs that hold units
        st0 = [np.nanmedian(t[:, i, 0]) - pub[i - 1] for i in idx]
        dur = [np.nanmax(t[:, i, 2]) - np.nanmedian(t[:, i, 0]) for i in idx]
        o_st = [np.nanmedian(t[:, i + 1, 1]) - np.nanmax(t[:, i, 2]) for i in idx]
        qin = [np.nanmedian(t[:, i, 1] - t[:, i, 0]) for i in idx]
        lp = [np.nanmedian(t[:, i, 3] - t[:, i, 1]) for i in idx]
        cmb = [np.nanmedian(t[:, i, 2] - t[:, i, 3]) for i in idx]
        print(f"  {nm:5s} qkv publish -> unit start {np.mean(st0):5.2f}, start -> last unit done {np.mean(dur):5.2f}, "
              f"last unit -> o staged (median) {np.mean(o_st):5.2f} us")
        print(f"        per unit (median): start -> q ready {np.mean(qin):5.2f}, rows loop {np.mean(lp):5.2f}, "
              f"combine + records {np.mean(cmb):5.2f} us")
        continue
    tk = [np.nanmedian(t[:, i, 0]) - (pub[i - 1] if i > 0 else 0) for i in idx if i > 0]
    st = [np.nanmedian(t[:, i, 1] - t[:, i, 0]) for i in idx]
    ti = [np.nanmedian(t[:, i, 2] - t[:, i, 1]) for i in idx]
    pb = [pub[i] - np.nanmax(t[:, i, 2]) for i in idx]
    print(f"  {nm:5s} ticket {np.mean(tk):5.2f} staging {np.mean(st):5.2f} tiles {np.mean(ti):5.2f} publish {np.mean(pb):5.2f}")
