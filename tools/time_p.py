"""Warm, event-timed kernel throughput of one (p, weak form) on cuda:0 -- for
A/B runs of library variants (PRISM_B200_LIB=<so> python tools/time_p.py ...).
Prints one JSON line: p, coeff, elements, median ms per launch, el/s."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_1191_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--coeff", default="laplace", choices=["laplace", "cdr", "elasticity"])
ap.add_argument("--nz", type=int, default=32)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--variant", type=int, default=0, help="0 auto, 1 dense, 2 sumfact")
a = ap.parse_args()
E = 2 * 128 * 64 * a.nz
n_eq = 3 if a.coeff == "elasticity" else 1
mode = {"laplace": pb.LAPLACE, "cdr": pb.PER_ELEMENT, "elasticity": pb.ELASTICITY}[a.coeff]
geom = torch.from_numpy(pb.generate_box_mesh(128, 64, a.nz, 0.1, 42, soa=True)).cuda()
coeff = None
if mode == pb.PER_ELEMENT:
    coeff = torch.from_numpy(pb.generate_cdr_coefficients(42, 0, E, soa=True)).cuda()
elif mode == pb.ELASTICITY:
    coeff = torch.from_numpy(pb.generate_materials(0, E, soa=True)).cuda()
dim = n_eq * pb.shape_count(a.p)
chunk = min(E, int(100e9 / 8) // (dim * dim))
out = torch.empty(chunk * dim * dim, dtype=torch.float64, device="cuda")
it = pb.Integrator(a.p, n_eq=n_eq, variant=a.variant)
s = torch.cuda.Stream()


def run():
    for lo in range(0, E, chunk):
        n = min(chunk, E - lo)
        it.integrate_device(n, geom.data_ptr() + 8 * lo, out, mode, None if coeff is None else coeff.data_ptr() + 8 * lo,
                            geom_ld=E, coeff_ld=E, element_id_base=lo, stream=s.cuda_stream)


for _ in range(2):
    run()
it.check()
times = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    run()
    e1.record(s)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
it.check()
ms = float(np.median(times))
print(json.dumps({"lib": str(pb.LIB_PATH if not __import__("os").environ.get("PRISM_B200_LIB") else
                             __import__("os").environ["PRISM_B200_LIB"]),
                  "p": a.p, "coeff": a.coeff, "variant": a.variant, "elements": E, "ms": ms,
                  "el_per_s": E / ms * 1e3}))
