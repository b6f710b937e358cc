"""DRAM traffic and device time of ONE factorisation of the batch-interleaved path from an ncu launch list
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`, cold-cache and serialised)
of `tools/bl_once.py <config> <K>`: the factorisation kernels' sums divided by the number of factorisations
(2 forwards x (K + 1)).  Writes/updates profiles/ncu_traffic.json[config] for bench.py's roofline.traffic.

usage: python tools/factor_traffic.py <launches.csv> <config> <batch> <factorisations> [<source tag>]"""
import csv
import json
import os
import sys
from collections import defaultdict

FACTOR_KERNELS = ("bl_update_rb", "bl_update", "bl_factor", "bl_persist", "bl_subtree", "bl_update_items",
                  "bl_factor_red")

path, config, batch, nfac = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
tag = sys.argv[5] if len(sys.argv) > 5 else os.path.basename(path)
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
per = defaultdict(lambda: defaultdict(float))
names = {}
for r in csv.DictReader(lines):
    name = r["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
    per[int(r["ID"])][r["Metric Name"]] += v * scale
    names[int(r["ID"])] = name
tot = defaultdict(float)
for i, m in per.items():
    if names[i] in FACTOR_KERNELS:
        for k, v in m.items():
            tot[k] += v
rd = tot["dram__bytes_read.sum"] / nfac
wr = tot["dram__bytes_write.sum"] / nfac
t = tot["gpu__time_duration.sum"] / nfac
out = {"batch": batch, "kernel": "factorisation (" + " + ".join(FACTOR_KERNELS) + ")",
       "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_time_s": t,
       "source": f"profiles/{tag}"}
tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
try:
    allj = json.load(open(tp))
    if "config" in allj:   # the round-1 single-entry format
        allj = {allj["config"]: allj}
except Exception:
    allj = {}
allj[config] = out
json.dump(allj, open(tp, "w"), indent=1)
print(json.dumps(out))
