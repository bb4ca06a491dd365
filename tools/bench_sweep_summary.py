"""Summarise tools/bench_sweep.sh output: one row per (weak form, p)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
print("| p | weak form | elements | el/s | ms | dense-roofline frac | executed FP64 frac | HBM frac | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows:
    for p, v in r["per_p"].items():
        print(f"| {p} | {r['config']['coeff']} | {r['config']['elements_per_gpu']} | {v['elements_per_s']:.3e} | "
              f"{v['ms']:.3f} | {v['frac_of_dense_roofline']:.2f} | {v.get('frac_executed_fp64', v.get('frac_executed_fp32', 0)):.2f} | "
              f"{v['frac_hbm']:.2f} | {r['clocks'].get('sm_mhz')} |")
