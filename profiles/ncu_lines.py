"""Summarise an ncu --set full report per CUDA source line (warp-stall samples).
usage: python profiles/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: [0, 0, ""])
path = ""
total = 0
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) < 7 or not r[0].isdigit():
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    if r[2] != "-":
        continue  # sass rows repeat; cuda rows carry the line aggregate
    key = (path, int(r[0]))
    agg[key][0] += s
    agg[key][1] += int(r[7] or 0)
    agg[key][2] = r[1].strip()[:90]
    total += s
print(f"total stall samples {total}")
for (f, ln), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * s / max(total, 1):5.1f}%  {f}:{ln:<5d} {src}")

if len(sys.argv) > 3 and sys.argv[3] == "inst":
    agg2 = defaultdict(lambda: [0, ""])
    for r in rows:
        if r and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0].isdigit() or r[2] != "-":
            continue
        try:
            agg2[(path, int(r[0]))][0] += int(r[7] or 0)
            agg2[(path, int(r[0]))][1] = r[1].strip()[:90]
        except ValueError:
            pass
    tot = sum(v[0] for v in agg2.values())
    print(f"\ntotal warp instructions executed {tot}")
    for (f, ln), (c, src) in sorted(agg2.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100.0 * c / max(tot, 1):5.1f}%  {f}:{ln:<5d} {src}")
