"""Summarise an ncu launch-list CSV (tools/sweep.sh): per kernel time, el/s, DRAM bytes."""
import csv
import sys
from collections import OrderedDict

E = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = (int(d["ID"]), d["Kernel Name"].split("(")[0])
        agg.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, name), m in agg.items():
    t = m.get("gpu__time_duration.sum", 0) * 1e-9
    print(f"{i:3d} {name:40s} {t*1e3:9.3f} ms  {E/t:10.3e} el/s  rd {m.get('dram__bytes_read.sum',0)/1e6:9.1f} MB  wr {m.get('dram__bytes_write.sum',0)/1e6:9.1f} MB")
