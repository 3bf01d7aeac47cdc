"""Per-warp loop ends (PMPD_ENGINE_TRACE_WSET probes): median (end - staged) per consumer warp per op kind."""
import sys
import numpy as np
res = {}
for f in sys.argv[1:]:
    w0 = int(f.split("ws")[-1][0]) * 4
    tr = np.load(f)["tr"].astype(np.float64)
    N = tr.shape[1]
    for k, nm in enumerate(("qkv", "o", "up", "down")):
        idx = [i for i in range(1, N - 1) if i % 4 == k]
        t = tr[:, idx]
        busy = (t[:, :, 2] - t[:, :, 1]) > 300
        for j in range(4):
            e = np.where(busy, (t[:, :, 4 + j] - t[:, :, 1]) / 1e3, np.nan)
            res.setdefault(nm, {})[w0 + j] = np.nanmedian(e)
for nm, d in res.items():
    print(f"  {nm:5s} " + " ".join(f"w{w}:{d[w]:5.2f}" for w in sorted(d)))
