"""Summarise the ncu launch list of the bench command against the bench line.
usage: python tools/launch_summary.py <tag> [launches.csv] [bench.json]
  (defaults gpurun_out/bench_launches_<tag>.csv, profiles/bench_r01_final.json)
writes profiles/bench_launches_<tag>.md and copies the csv next to it."""
import csv
import json
import shutil
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / f"bench_launches_{tag}.csv"
bench_json = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "profiles" / "bench_r01_final.json"
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
t, n, by = defaultdict(float), defaultdict(int), defaultdict(float)
for r in data:
    k = r[ki].split("(")[0].replace("void pib::", "")
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    if r[mi] == "gpu__time_duration.sum":
        t[k] += v
        n[k] += 1
    else:
        by[k] += v
b = json.load(open(bench_json))
step = b["ms_per_step"]
keys = [k for k in t if "peak" not in k]
tot = sum(t[k] for k in keys)
pp = {"p2_lane_kernel<0, 1, double>": "2", "p2_lane_kernel<0, 1, double, 0>": "2", "sumfact_kernel<3, 1, 0, 1>": "3",
      "sumfact_kernel<4, 1, 0, 1>": "4"}
out = [f"# ncu launch list of the bench command ({tag})", "",
       "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv",
       "python bench.py --steps 2 --warmup 1 --sweep '' --no-e2e --no-cpu --no-parity --no-load` (1 B200; cold-cache, serialised launches;",
       f"e2e / CPU legs skipped to keep the capture to the device step).  Raw list: `bench_launches_{tag}.csv`.", "",
       f"| kernel | launches | total ms | share of the step (ncu) | share from bench.py events (`{bench_json.name}`) | DRAM bytes / launch | algorithmic bytes / launch |",
       "|---|---|---|---|---|---|---|"]
for k in sorted(keys, key=lambda k: t[k]):
    per = b["per_p"][pp[k]]
    alg = per["bytes_per_element"] * (1 << 20)
    out.append(f"| `{k}` | {n[k]} | {t[k]:.1f} | {100 * t[k] / tot:.1f} % | {100 * per['ms'] / step:.1f} % "
               f"({per['ms']:.3f} ms) | {by[k] / n[k] / 1e9:.2f} GB | {alg / 1e9:.2f} GB |")
out += ["", "(`dmma_peak_kernel` / `dfma_peak_kernel` are the in-run FP64 peak probes, outside the timed step.)",
        "The dominant kernel's DRAM traffic equals its algorithmic bytes (K written once, geometry read once)."]
(ROOT / "profiles" / f"bench_launches_{tag}.md").write_text("\n".join(out) + "\n")
shutil.copy(src, ROOT / "profiles" / f"bench_launches_{tag}.csv")
print("\n".join(out))
