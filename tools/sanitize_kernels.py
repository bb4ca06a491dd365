"""Drive every kernel family once at a small size, for compute-sanitizer.

Usage (on the GPU box):
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_kernels.py [--only FAMILY]

Families (the launch each one reaches, pi_context.cu dispatch):
  p1       p1_thread_kernel (Laplace, per-element CDR), FP64 and FP32 output
  p2       p2_lane_kernel (symmetric 9-warp / general 18-warp), FP32 compute variant
  sumfact  sumfact_kernel<P, 1> p = 3..7 row split (CDR) and symmetric shapes (Laplace p = 3, 4)
  pairs    sumfact_pairs_kernel p = 5..7 (symmetric scalar forms)
  dense    the non-default strategies: sumfact_kernel<2, 1>, sumfact_kernel<3, 3>
  elastic  p1_elastic_lane / p2_elastic_warp / p3_elastic_cta, sumfact_kernel<P, 3> p = 4..7
  load     load_vector_kernel p = 1..7
  fused    pi_integrate_load: the scalar kernels with the fused load vector
  tc32     sumfact_tc32_kernel (tcgen05, TMEM, mbarrier ring), VARIANT_TC32
  initprobe  initcheck and TMA bulk stores (see fam_initprobe)
  host     pi_integrate_host: aos_to_soa_kernel + chunked two-stream path
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1310_1191_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)


def mesh_of(n):
    m = pb.generate_box_mesh(16, 8, 4, 0.2, seed=7)[:n]
    return m, torch.from_numpy(np.ascontiguousarray(m.reshape(len(m), 18).T)).to(dev)


def run(p, n, mode, n_eq=1, variant=pb.VARIANT_AUTO, f32=False, layout=pb.OUT_CANONICAL, load=False):
    m, geom = mesh_of(n)
    coeff = None
    if mode == pb.PER_ELEMENT:
        c = pb.generate_cdr_coefficients(42, 0, n) if n_eq == 1 else np.random.default_rng(1).standard_normal((n, 144))
        coeff = torch.from_numpy(np.ascontiguousarray(c.T)).to(dev)
    elif mode == pb.ELASTICITY:
        coeff = torch.from_numpy(np.ascontiguousarray(pb.generate_materials(0, n).T)).to(dev)
    with pb.Integrator(p, n_eq=n_eq, variant=variant) as it:
        dim = it.dim
        out = torch.full((n, dim, dim), float("nan"), dtype=torch.float32 if f32 else torch.float64, device=dev)
        kw = {}
        if layout == pb.OUT_SOA:
            out = out.reshape(dim * dim, n)
            kw["ld_out"] = n
        if load:
            kw["load_out"] = torch.full((n, it.n_shape), float("nan"), dtype=torch.float64, device=dev)
            kw["f"] = torch.rand(n, dtype=torch.float64, device=dev)
        it.integrate_device(n, geom, out, mode, coeff, out_layout=layout, **kw)
        it.check()
        torch.cuda.synchronize()
    assert torch.isfinite(out).all(), f"p={p} mode={mode} n_eq={n_eq}: unwritten / non-finite output"
    if load:
        assert torch.isfinite(kw["load_out"]).all(), f"p={p}: unwritten load vector"
    print(f"ok p={p} mode={mode} n_eq={n_eq} variant={variant} f32={f32} layout={layout} n={n}", flush=True)


def fam_p1():
    for mode in (pb.LAPLACE, pb.PER_ELEMENT):
        run(1, 300, mode)
        run(1, 300, mode, f32=True)
    run(1, 37, pb.LAPLACE, layout=pb.OUT_SOA)


def fam_p2():
    for mode in (pb.LAPLACE, pb.PER_ELEMENT):
        run(2, 70, mode)
        run(2, 70, mode, f32=True)
    run(2, 33, pb.PER_ELEMENT, layout=pb.OUT_SOA)


def fam_sumfact():
    for p in (3, 4, 5, 6, 7):
        run(p, 5 if p < 6 else 2, pb.PER_ELEMENT)
    for p in (3, 4):
        run(p, 5, pb.LAPLACE)
        run(p, 3, pb.LAPLACE, layout=pb.OUT_SOA)


def fam_pairs():
    for p in (5, 6, 7):
        run(p, 3 if p < 7 else 2, pb.LAPLACE)


def fam_dense():  # the non-default strategies: sum factorisation at p = 2, dense elasticity is the default
    run(2, 40, pb.LAPLACE, variant=pb.VARIANT_SUMFACT)
    run(2, 40, pb.PER_ELEMENT, variant=pb.VARIANT_SUMFACT)
    run(3, 4, pb.PER_ELEMENT, n_eq=3, variant=pb.VARIANT_SUMFACT)


def fam_elastic():
    run(1, 100, pb.ELASTICITY, n_eq=3)
    run(2, 20, pb.ELASTICITY, n_eq=3)
    run(3, 4, pb.ELASTICITY, n_eq=3)
    for p in (4, 5, 6, 7):
        run(p, 2, pb.ELASTICITY, n_eq=3)
    run(4, 2, pb.PER_ELEMENT, n_eq=3)


def fam_load():
    for p in range(1, 8):
        n = 40
        _, geom = mesh_of(n)
        with pb.Integrator(p) as it:
            out = torch.full((n, it.n_shape), float("nan"), dtype=torch.float64, device=dev)
            f = torch.rand(n, dtype=torch.float64, device=dev)
            it.load_vectors_device(n, geom, out, f=f)
            it.check()
        assert torch.isfinite(out).all()
        print(f"ok load p={p}", flush=True)


def fam_fused():  # pi_integrate_load: every scalar kernel family with the load vector
    for p in range(1, 8):
        n = {1: 300, 2: 70, 3: 5, 4: 5, 5: 3}.get(p, 2)
        run(p, n, pb.LAPLACE, load=True)
        run(p, n, pb.PER_ELEMENT, load=True)
    run(2, 40, pb.LAPLACE, variant=pb.VARIANT_SUMFACT, load=True)


def fam_tc32():  # sumfact_tc32_kernel (tcgen05 FP32, opt-in VARIANT_TC32)
    for p in (3, 4, 5):
        run(p, 5, pb.LAPLACE, variant=pb.VARIANT_TC32, f32=True)
        run(p, 5, pb.PER_ELEMENT, variant=pb.VARIANT_TC32, f32=True)


def fam_initprobe():
    """initcheck does not see writes of the TMA bulk-copy engine: the same
    p = 1 launch into a fresh (uninitialised) buffer, 16-byte aligned (TMA bulk
    stores) and 8-byte aligned (ordinary stores), then read by a torch kernel."""
    n, kk = 300, 36
    m, geom = mesh_of(n)
    with pb.Integrator(1) as it:
        for shift, tag in ((1, "st.global (8-byte aligned base)"), (0, "cp.async.bulk (16-byte aligned base)")):
            buf = torch.empty(n * kk + 2 + shift * 1000, dtype=torch.float64, device=dev)  # fresh allocation
            out = buf[shift:shift + n * kk]
            it.integrate_device(n, geom, out, pb.LAPLACE)
            it.check()
            print(f"initprobe {tag}: reading the output now", flush=True)
            assert torch.isfinite(out).all()
            torch.cuda.synchronize()
            print(f"initprobe {tag}: done; now a D2H copy of the same output", flush=True)
            host = out.cpu()
            assert torch.isfinite(host).all()
            print(f"initprobe {tag}: D2H done", flush=True)


def fam_host():
    m, _ = mesh_of(64)
    for p in (1, 2, 3, 4):
        with pb.Integrator(p) as it:
            k = it.integrate_host(m, pb.LAPLACE, chunk_elems=24)
            assert np.isfinite(k).all()
        print(f"ok host p={p}", flush=True)


FAMS = {k[4:]: v for k, v in globals().items() if k.startswith("fam_")}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    names = a.only.split(",") if a.only else list(FAMS)
    for name in names:
        FAMS[name]()
    print("sanitize driver done", flush=True)
