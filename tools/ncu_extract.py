"""Box-side reduction of an ncu --set full report to a small text summary (the .ncu-rep files are ~15 MB
each and gpurun copies back at most 64 MiB): key metrics per captured launch + warp-stall shares.
usage: python tools/ncu_extract.py <report.ncu-rep> [--keep]   -> <report>.txt"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
out = []
if len(rows) >= 3:
    hdr, units = rows[0], rows[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
    for vals in rows[2:]:
        out.append("launch:")
        for k in keys:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k:66s} {vals[i]} {units[i]}")
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
out.append("  warp-stall samples: " + ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in
                                               sorted(tot.items(), key=lambda kv: -kv[1]) if v))
open(os.path.splitext(rep)[0] + ".txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
if "--keep" not in sys.argv:
    os.remove(rep)
