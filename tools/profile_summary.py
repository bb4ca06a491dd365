"""Turn a gpurun sweep (ncu launch list CSV) + one full ncu capture into a
committed summary under profiles/.

  python tools/profile_summary.py <tag> [--full gpurun_out/prof_<tag>_pN.ncu-rep ...]

Writes profiles/<tag>_launches.csv (copy), profiles/<tag>.md and updates
profiles/traffic.json (DRAM bytes per launch per (p, coeff), read by bench.py).
"""
import argparse
import csv
import json
import shutil
import subprocess
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
E_SWEEP = 2 * 128 * 64 * 16  # tools/sweep.sh uses --nz 16
LAPLACE = {1: 3390, 2: 48402, 3: 531408, 4: 2910080, 5: 14934750, 6: 54773565, 7: 170459184}
CDR = {1: 4326, 2: 64602, 3: 711888, 4: 3894080, 5: 19962150, 6: 73155621, 7: 227552304}
NSH = {p: (p + 1) ** 2 * (p + 2) // 2 for p in range(1, 8)}
FP64_PEAK = 37.0e12  # measured DMMA peak (pi_measure_fp64_peak), TFLOP/s
HBM_PEAK = 6549.8e9


def parse_launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = (int(d["ID"]), d["Kernel Name"].split("(")[0])
            agg.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return agg


def kernel_key(name):
    """Kernel name -> (p, weak form): sumfact_kernel<P, NE, FORM, SYM>,
    p1_thread_kernel<GENERAL>, p2_lane_kernel<GENERAL, SYM>."""
    n_eq3 = {"p1_elastic_lane_kernel": 1, "p2_elastic_warp_kernel": 2, "p3_elastic_cta_kernel": 3}
    for k, p in n_eq3.items():
        if k in name:
            return p, "elasticity"
    inside = name.split("<")[1].rstrip(">").replace(" ", "").replace("(int)", "").replace("(bool)", "").split(",")
    general = lambda v: v in ("1", "true")  # noqa: E731
    if "p1_thread" in name:
        return 1, "cdr" if general(inside[0]) else "laplace"
    if "p2_lane" in name:
        if not general(inside[0]):
            return 2, "laplace"
        return 2, "uniform-sym" if general(inside[1]) else "cdr"
    p, ne, form = int(inside[0]), int(inside[1]), int(inside[2])
    if ne == 3:
        return p, "elasticity" if form == 2 else "system"
    return p, "cdr" if form == 1 else "laplace"


NQ = {1: 6, 2: 18, 3: 48, 4: 80, 5: 150, 6: 231, 7: 336}


def dense_flops(p, form):
    if form == "elasticity":  # the reference's 63-flop block model (flop_costs.hpp)
        return NQ[p] * (63 * NSH[p] ** 2 + 15 * NSH[p] + 154)
    return (LAPLACE if form == "laplace" else CDR)[p]


def dims(p, form):
    return (3 if form in ("elasticity", "system") else 1) * NSH[p]


def launch_elements(p, form):
    """tools/prof_run.py caps K at 60 GB per launch."""
    return min(E_SWEEP, int(60e9 / 8) // dims(p, form) ** 2)


def full_counters(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    if len(r) < 3:
        return {}
    d = dict(zip(r[0], r[2]))
    keep = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum"]
    return {k: d.get(k) for k in keep}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--full", action="append", default=[])
    a = ap.parse_args()
    src = ROOT / "gpurun_out" / f"sweep_{a.tag}.csv"
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    shutil.copy(src, prof / f"{a.tag}_launches.csv")
    agg = parse_launches(src)
    seen = {}
    for (i, name), m in agg.items():
        key = kernel_key(name)
        seen.setdefault(key, []).append((name, m))
    lines = [f"# Kernel sweep `{a.tag}` (1 B200, ncu launch list, up to {E_SWEEP} prisms per launch, cold/serialised)", "",
             "Dense roofline = min(FP64 peak 37.0 TF/s / FLOP_alg, HBM 6549.8 GB/s / bytes) per SURVEY.md 8(d) (elasticity: the reference's 63-flop block model).", "",
             "| p | weak form | kernel | elements | ms | elements/s | vs dense roofline | DRAM read MB | DRAM write MB | K bytes ideal MB |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    tf = prof / "traffic.json"
    if tf.exists():
        traffic = json.load(open(tf))
    for (p, form), lst in sorted(seen.items()):
        name, m = lst[-1]
        t = m["gpu__time_duration.sum"] * 1e-9
        flops = dense_flops(p, form)
        n = launch_elements(p, form)
        byts = 8 * dims(p, form) ** 2 + 144 + {"cdr": 128, "elasticity": 16}.get(form, 0)
        bound = min(FP64_PEAK / flops, HBM_PEAK / byts)
        rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        lines.append(f"| {p} | {form} | `{name.replace('void ', '')}` | {n} | {t*1e3:.3f} | {n/t:.3e} | "
                     f"{n/t/bound:.2f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {8*dims(p, form)**2*n/1e6:.1f} |")
        traffic[f"p{p}_{form}"] = (rd + wr) / n  # DRAM bytes per element (per launch / elements)
    json.dump(traffic, open(tf, "w"), indent=1)
    for full in a.full:
        c = full_counters(full)
        lines += ["", f"## Full capture `{Path(full).name}`", "", "| counter | value |", "|---|---|"]
        lines += [f"| {k} | {v} |" for k, v in c.items()]
    (prof / f"{a.tag}.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
