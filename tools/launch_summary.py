"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch): total per kernel name and the
per-launch sequence of the bl_* kernels (level structure)."""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    unit = r.get("Metric Unit", "ns")
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
    rows.append((int(r["ID"]), name, us))
tot = defaultdict(float)
cnt = defaultdict(int)
for _, n, us in rows:
    tot[n] += us
    cnt[n] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {len(rows)} launches")
for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {100 * v / T:5.1f}%  n={cnt[n]:5d}  avg {v / cnt[n]:9.2f} us  {n}")
if len(sys.argv) > 2:
    for i, n, us in rows[: int(sys.argv[2])]:
        print(i, n, f"{us:.1f}")
