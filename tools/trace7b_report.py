"""Summarise gpurun_out/trace7b_*.npz (tools/engine_trace7b.py): per-op-kind critical path phases."""
import glob
import sys
import numpy as np

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace7b_*.npz")):
    tr = np.load(f)["tr"]
    t = tr[:, :, :4].astype(np.float64)
    t0 = t[t > 0].min()
    t = (t - t0) / 1e3
    N = t.shape[1]
    pub = t[:, :, 3].max(0)
    rm, sm, tm, tx = (np.median(t[:, :, 0], 0), np.median(t[:, :, 1], 0), np.median(t[:, :, 2], 0), t[:, :, 2].max(0))
    r = np.array([(rm[i] - pub[i - 1], sm[i] - rm[i], tm[i] - sm[i], tx[i] - tm[i], pub[i] - tx[i], pub[i] - pub[i - 1])
                  for i in range(1, N)])
    print(f"== {f}: {pub[-1]:.1f} us, {N} ops")
    for k, nm in enumerate(("qkv", "o", "up", "down")):
        idx = [i - 1 for i in range(1, N - 1) if i % 4 == k]
        print(f"  {nm:5s} ticket {r[idx,0].mean():5.2f} stage {r[idx,1].mean():5.2f} tiles {r[idx,2].mean():6.2f} "
              f"imbal {r[idx,3].mean():5.2f} publish {r[idx,4].mean():5.2f} | op {r[idx,5].mean():6.2f}")

    # inside the tile phase (consumer warp 0, SM clock cycles -> us at the 1965 MHz boost clock):
    # tile calls, n-group flushes (of which waiting for the epilogue's buffer), the rest (ring waits)
    GHZ = 1.965e3
    cyc = tr[:, :, 4:8].astype(np.float64)
    for k, nm in enumerate(("qkv", "o", "up", "down")):
        idx = [i for i in range(1, N - 1) if i % 4 == k]
        tc, ncall, tot = cyc[:, idx, 0], cyc[:, idx, 1], cyc[:, idx, 2]
        fw = (tr[:, idx, 7] >> 32).astype(np.float64)
        fc = (tr[:, idx, 7] & 0xffffffff).astype(np.float64)
        print(f"  {nm:5s} phase {np.median(tot) / GHZ:5.2f} us: calls {np.median(ncall):4.1f} x "
              f"{np.median(tc / np.maximum(ncall, 1)):5.0f} cyc = {np.median(tc) / GHZ:5.2f} us, flush "
              f"{np.median(fc) / GHZ:5.2f} (wait {np.median(fw) / GHZ:5.2f}), other {np.median(tot - tc - fc) / GHZ:5.2f}")
