"""Summarise an ncu --set full capture (one kernel launch) + the launch list into profiles/.

usage: python profiles/summarize.py <report.ncu-rep> <launches.csv> <tag> <config>
writes profiles/<tag>_ncu_summary.txt, profiles/<tag>_launches.csv and profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

rep, launches, tag, config = sys.argv[1:5]
here = os.path.dirname(os.path.abspath(__file__))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
info = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        info[w] = (vals[i], units[i])
lines = [f"ncu --set full summary: {os.path.basename(rep)} (config {config})"]
for k, (v, u) in info.items():
    lines.append(f"  {k:62s} {v} {u}")


def num(k):
    v, u = info[k]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(u, 1)
    return x * scale


traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
lines.append(f"  dram traffic per launch (read + write): {traffic:.4g} bytes")
# stall reasons (source view)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot = defaultdict(int)
h = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Line No":
        h = r
        continue
    if not h or len(r) != len(h) or not r[0].isdigit() or r[2] != "-":
        continue
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                tot[name[6:]] += int(r[i])
            except ValueError:
                pass
T = sum(tot.values()) or 1
lines.append("  warp-stall samples: " + ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in
                                                sorted(tot.items(), key=lambda kv: -kv[1]) if v))
# launch list shares
lrows = list(csv.reader(open(launches)))
start = next(i for i, r in enumerate(lrows) if r and r[0] == "ID")
hh = lrows[start]
kn, mv = hh.index("Kernel Name"), hh.index("Metric Value")
agg = defaultdict(list)
for r in lrows[start + 1:]:
    if len(r) > mv:
        agg[r[kn].split("(")[0][:60]].append(float(r[mv].replace(",", "")))
tt = sum(sum(v) for v in agg.values())
lines.append("  launch list (gpu__time_duration, cold-cache, serialised) shares:")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"    {100 * sum(v) / tt:5.1f}%  n={len(v):3d}  avg {sum(v) / len(v) / 1e3:9.1f} us  {k}")
open(os.path.join(here, f"{tag}_ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(launches, os.path.join(here, f"{tag}_launches.csv"))
json.dump({"config": config, "kernel": info.get("Kernel Name", ("", ""))[0][:80], "dram_bytes_per_launch": traffic,
           "source": f"profiles/{tag}_ncu_summary.txt"}, open(os.path.join(here, "ncu_traffic.json"), "w"), indent=1)
print("\n".join(lines))
