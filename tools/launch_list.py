"""Print an ncu --csv launch list (gpu__time_duration / dram bytes per launch) in launch order:
  python tools/launch_list.py gpurun_out/x_launches.csv [first] [count]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
hdr = None
k = OrderedDict()
for r in rows:
    if len(r) > 10 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = k.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = 0.0
for i, e in enumerate(list(k.values())[first:first + count]):
    name = e["name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    t = e.get("gpu__time_duration.sum", 0.0) / 1e3
    rd = e.get("dram__bytes_read.sum", 0.0) / 1e6
    wr = e.get("dram__bytes_write.sum", 0.0) / 1e6
    tot += t
    print(f"{first + i:4d} {name[:28]:28s} {e['grid']:>14s} {t:9.1f} us  rd {rd:8.1f} MB  wr {wr:8.1f} MB  {(rd + wr) / max(t, 1e-9):5.2f} TB/s")
print(f"total {tot:.1f} us")
