"""gpurun_out/traffic_p*.csv (ncu --csv) -> profiles/engine_traffic.json (bytes per engine launch by precision)."""
import csv, io, json, os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {"bytes_per_launch": {}, "duration_ms": {}, "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
       "--clock-control none -k regex:engine_kernel (tools/capture_traffic.sh), one launch = one 7B token"}
for p in (4, 3, 2):
    path = os.path.join(root, "gpurun_out", f"traffic_p{p}.csv")
    if not os.path.exists(path):
        continue
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    h = rows[0]
    vals = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        unit, v = d["Metric Unit"], float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}.get(unit, 1)
        vals[d["Metric Name"]] = v * scale
    out["bytes_per_launch"][str(p)] = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    out["duration_ms"][str(p)] = vals.get("gpu__time_duration.sum")
json.dump(out, open(os.path.join(root, "profiles", "engine_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
