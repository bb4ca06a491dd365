"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv; python tools/ncu_lines.py s.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
res = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            inst = float(r[hdr.index("Instructions Executed")] or 0)
            stall = float(r[4] or 0)
        except (ValueError, IndexError):
            continue
        res.append((inst, stall, cur_file, r[0], r[1][:90]))
tot = sum(x[0] for x in res) or 1
tst = sum(x[1] for x in res) or 1
for inst, stall, f, ln, src in sorted(res, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{inst/tot*100:6.2f}% inst {stall/tst*100:6.2f}% stall  {f}:{ln}  {src}")
