"""Summarise an ncu report: key metrics + per-opcode instruction counts + top stalls."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
d = dict(zip(hdr, vals))
for k in keys:
    print(f"{k:75s} {d.get(k)}")
for h, v in zip(hdr, vals):
    if "average_warps_issue_stalled" in h and "per_issue_active.ratio" in h:
        try:
            if float(v) > 0.1:
                print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rs = list(csv.reader(io.StringIO(src)))[2:]
ops = collections.Counter()
for r in rs:
    if len(r) > 5 and r[5]:
        s = r[1].strip()
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        ops[op.split(".")[0]] += int(r[5])
tot = sum(ops.values())
print(f"instructions per tile: {tot / tiles:.1f}")
print("  " + ", ".join(f"{k}:{v / tiles:.1f}" for k, v in ops.most_common(18)))
