"""Split an ncu SASS source page into producer / consumer regions (the
consumer region spans the DMMA instructions) and list stall reasons per region.
usage: python tools/sass_regions.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys
from collections import Counter

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, d = rows[1], rows[2:]
isrc, iall = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall = [(i, c) for i, c in enumerate(h) if c.startswith("stall_")]
dm = [k for k, r in enumerate(d) if "DMMA" in r[isrc]]
lo, hi = (min(dm), max(dm)) if dm else (0, -1)
# widen to the enclosing barrier syncs
while lo > 0 and "BAR.SYNC" not in d[lo][isrc]:
    lo -= 1
regions = {"before-consumer": d[:lo], "consumer-mainloop": d[lo:hi + 1], "after": d[hi + 1:]}
tot = sum(int(r[iall] or 0) for r in d)
for name, rs in regions.items():
    s = sum(int(r[iall] or 0) for r in rs)
    c = Counter()
    for r in rs:
        for i, col in stall:
            try:
                c[col] += float(r[i] or 0)
            except ValueError:
                pass
    top = ", ".join(f"{k.replace('stall_', '')} {v / max(1, s) * 100:.0f}%" for k, v in c.most_common(6))
    print(f"{name:18s} {100 * s / tot:5.1f}% of samples | {top}")
