"""Stall-reason totals (warp-stall samples) of an ncu --set full report, overall and for the
top source lines.  usage: python profiles/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
tot = defaultdict(int)
per_line = defaultdict(lambda: defaultdict(int))
src = {}
path = ""
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i])
            except ValueError:
                continue
            tot[h] += v
            per_line[(path, int(r[0]))][h] += v
    src[(path, int(r[0]))] = r[1].strip()[:80]
T = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for key, d in sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(d.values())
    parts = ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{100*s/T:5.1f}% {key[0]}:{key[1]} [{parts}] {src[key]}")
