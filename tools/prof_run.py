"""Minimal driver for ncu captures: integrates E prisms at one p a few times.

  python tools/prof_run.py --p 4 [--coeff laplace|cdr] [--nz 64] [--launches 4]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_1191_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--coeff", default="laplace")
ap.add_argument("--nz", type=int, default=64)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--variant", type=int, default=0)
a = ap.parse_args()
E = 2 * 128 * 64 * a.nz
geom = torch.from_numpy(pb.generate_box_mesh(128, 64, a.nz, 0.1, 42, soa=True)).cuda()
mode = {"laplace": pb.LAPLACE, "cdr": pb.PER_ELEMENT, "elasticity": pb.ELASTICITY}[a.coeff]
n_eq = 3 if mode == pb.ELASTICITY else 1
coeff = None
if mode == pb.PER_ELEMENT:
    coeff = torch.from_numpy(pb.generate_cdr_coefficients(42, 0, E, soa=True)).cuda()
elif mode == pb.ELASTICITY:
    coeff = torch.from_numpy(pb.generate_materials(0, E, soa=True)).cuda()
nsh = n_eq * pb.shape_count(a.p)
E_out = min(E, int(60e9 / 8) // (nsh * nsh))  # launches beyond 60 GB of K integrate the first E_out prisms
out = torch.empty(E_out * nsh * nsh, dtype=torch.float64, device="cuda")
E = E_out
it = pb.Integrator(a.p, n_eq=n_eq, variant=a.variant)
s = None  # the context's own stream
for _ in range(a.launches):
    it.integrate_device(E, geom, out, mode, coeff, stream=s)
it.check()
torch.cuda.synchronize()
print("ok", a.p, E)
