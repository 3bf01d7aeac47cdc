"""Summarise gpurun_out/engine_trace.npz (tools/engine_trace.py): per op, med/max over CTAs of each event (µs)."""
import sys
import numpy as np
d = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/engine_trace.npz")
EV = [(0, "stage0"), (1, "staged"), (12, "s0.data"), (13, "s0.done"), (14, "s1.data"), (15, "s1.done"), (8, "loopend"),
      (2, "cons.done"), (10, "rowN"), (11, "fin.start"), (7, "fin.done")]
for k in d.files:
    tr = d[k].astype(np.float64)
    G, n_ops, nf = tr.shape
    ts = tr[:, :, [e for e, _ in EV]]
    t0 = ts[ts > 0].min()
    print("==", k, "  (µs; med/max over CTAs)")
    print("      " + " ".join(f"{n:>13s}" for _, n in EV) + "   tile-cyc  wait-cyc calls")
    for oi in range(n_ops):
        row = []
        for e, _ in EV:
            v = tr[:, oi, e]
            v = np.where(v > 0, (v - t0) / 1000.0, np.nan)
            row.append(f"{np.nanmedian(v):6.2f}/{np.nanmax(v):6.2f}" if np.isfinite(v).any() else f"{'-':>13s}")
        m = tr[:, oi, 5] > 0
        print(f" op{oi:<3d} " + " ".join(row) + f"  {np.median(tr[m, oi, 4]):8.0f} {np.median(tr[m, oi, 6]):8.0f} {np.median(tr[m, oi, 5]):4.0f}")
        if len(sys.argv) > 2:
            fm = tr[:, oi, 14] > 0
            if fm.any():
                print(f"        finalize (warp0): sweeps med {np.median(tr[fm, oi, 12]):.0f} max {tr[fm, oi, 12].max():.0f} | cycles med {np.median(tr[fm, oi, 13]):.0f} max {tr[fm, oi, 13].max():.0f} | rows med {np.median(tr[fm, oi, 14]):.0f} max {tr[fm, oi, 14].max():.0f}")
