"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*)
into per-kernel share of the step, mean duration and DRAM bytes per launch.

    python tools/ncu_summary.py gpurun_out/launches_c2.csv WORKLOAD_NAME [out.json]

Also merges the dominant kernel's DRAM bytes/launch into profiles/ncu_traffic.json
(read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import sys
from collections import defaultdict

path, workload = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else None
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = defaultdict(dict)
for r in rows[1:]:
    per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
    per[int(r[ii])]["name"] = r[ki]
agg = defaultdict(lambda: {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
for d in per.values():
    name = d["name"].split("(")[0]
    a = agg[name]
    a["launches"] += 1
    a["time_ns"] += d.get("gpu__time_duration.sum", 0.0)
    a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
total = sum(a["time_ns"] for a in agg.values())
summary = {"workload": workload, "source": os.path.basename(path), "kernels": []}
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_ns"]):
    summary["kernels"].append({
        "kernel": name, "launches": a["launches"], "share_of_time": a["time_ns"] / total,
        "mean_us": a["time_ns"] / a["launches"] / 1e3,
        "dram_bytes_per_launch": a["dram_bytes"] / a["launches"]})
for k in summary["kernels"]:
    print(f"{k['share_of_time']*100:6.2f}%  {k['launches']:5d}x  {k['mean_us']:10.2f} us  "
          f"{k['dram_bytes_per_launch']/1e9:8.4f} GB/launch  {k['kernel']}")
if out:
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
top = summary["kernels"][0]
tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
traffic[workload] = top["dram_bytes_per_launch"]
json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
