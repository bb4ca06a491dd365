"""Top source lines per stall reason of an ncu report (needs --import-source on captures).
usage: python tools/ncu_stalls.py X.ncu-rep [n]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True).stdout.decode("latin-1")
rows = list(csv.reader(io.StringIO(txt)))
hdr = cur = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
REASONS = ("stall_barrier", "stall_wait", "stall_math", "stall_short_sb", "stall_mio", "stall_long_sb")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur, hdr = r[1].split("/")[-1], None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and r[0].isdigit():
        key = (cur, int(r[0]))
        src[key] = r[1].strip()[:90]
        for c in REASONS + ("Instructions Executed", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared"):
            agg[key][c] += num(r[hdr.index(c)])
allst = sum(agg[k][c] for k in agg for c in REASONS)
print(f"total stall samples {allst:.0f}")
for c in REASONS + ("Instructions Executed", "L1 Wavefronts Shared Excessive"):
    tot = sum(v[c] for v in agg.values())
    print(f"== {c}: {tot:.3g} ({100 * tot / allst:.1f}% of stalls)" if c in REASONS else f"== {c}: {tot:.3g}")
    for k in sorted(agg, key=lambda k: -agg[k][c])[:n]:
        print(f"  {100 * agg[k][c] / max(tot, 1):5.1f}%  {k[0]}:{k[1]}  {src[k]}")
