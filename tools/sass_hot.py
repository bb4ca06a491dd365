"""Top stall lines of an ncu report's SASS source page, with per-opcode totals.
usage: python tools/sass_hot.py <report.ncu-rep> [n]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
tot = sum(int(r[iall] or 0) for r in data)
print(f"total samples {tot}")
byop = Counter()
for r in data:
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    byop[op.split(".")[0]] += int(r[iall] or 0)
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(12)))
for r in sorted(data, key=lambda r: -int(r[iall] or 0))[:n]:
    print(f"{100*int(r[iall])/tot:5.1f}% {r[ia][-5:]} {r[isrc][:90]}")
