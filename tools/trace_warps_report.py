"""Summarise a PMPD_ENGINE_TRACE_WARPS trace (tools/engine_trace7b.py on a library built with
-DPMPD_ENGINE_TRACE_WARPS): per op kind, the tile phase of warp 0, the spread of the consumer
warps' loop ends, and the mean per-warp call / full-stage wait time."""
import sys
import numpy as np

GHZ = 1.965e3
tr = np.load(sys.argv[1])["tr"].astype(np.float64)
N = tr.shape[1]
for k, nm in enumerate(("qkv", "o", "up", "down")):
    idx = [i for i in range(1, N - 1) if i % 4 == k]
    t = tr[:, idx]
    busy = (t[:, :, 2] - t[:, :, 1]) > 300
    ph = np.where(busy, (t[:, :, 2] - t[:, :, 1]) / 1e3, np.nan)
    spread = np.where(busy, (t[:, :, 6] - t[:, :, 7]) / 1e3, np.nan)
    last = np.where(busy, (t[:, :, 6] - t[:, :, 1]) / 1e3, np.nan)
    call = np.where(busy, t[:, :, 4] / 12 / GHZ, np.nan)
    wait = np.where(busy, t[:, :, 5] / 12 / GHZ, np.nan)
    print(f"  {nm:5s} warp0 phase {np.nanmedian(ph):5.2f}  last warp {np.nanmedian(last):5.2f}  spread {np.nanmedian(spread):5.2f} "
          f"| per warp: calls {np.nanmedian(call):5.2f}  full-wait {np.nanmedian(wait):5.2f}  rest {np.nanmedian(last - call - wait):5.2f} us")
