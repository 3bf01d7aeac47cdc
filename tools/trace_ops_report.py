"""Per-op summary of an engine trace (tools/engine_trace7b.py) for any program layout: ops are
grouped by their index modulo the layer period (argv[2], default 4); per group, over the CTAs
with tiles: median input-ready -> staged, staged -> tiles done, done spread (max - median) and
the op's end (last publish) relative to the previous op's end."""
import sys
import numpy as np

tr = np.load(sys.argv[1])["tr"].astype(np.float64)
per = int(sys.argv[2]) if len(sys.argv) > 2 else 4
t = tr[:, :, :4]
t0 = t[t > 0].min()
N = t.shape[1]
pub = np.where(t[:, :, 3] > 0, t[:, :, 3], np.nan)
pubmax = np.nanmax(pub, 0)
print(f"== {sys.argv[1]}: {(pubmax[-2] - t0) / 1e3:.1f} us to the head, {N} ops, period {per}")
for k in range(per):
    idx = [i for i in range(1, N - 1) if (i - 1) % per == k]
    st, ph, sp, en, nb = [], [], [], [], []
    for i in idx:
        busy = t[:, i, 2] - t[:, i, 1] > 0
        if not busy.any():
            continue
        r, s_, d = t[busy, i, 0], t[busy, i, 1], t[busy, i, 2]
        st.append(np.median(s_ - r))
        ph.append(np.median(d - s_))
        sp.append(d.max() - np.median(d))
        en.append(pubmax[i] - pubmax[i - 1])
        nb.append(busy.sum())
    print(f"  op {k:2d}: ctas {np.mean(nb):5.1f}  stage {np.mean(st) / 1e3:5.2f}  tiles {np.mean(ph) / 1e3:5.2f}  "
          f"spread {np.mean(sp) / 1e3:5.2f}  | op end +{np.mean(en) / 1e3:5.2f} us")
