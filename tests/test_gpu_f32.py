"""FP32 variant: K in float32.  Stated bound: per-element
relative Frobenius <= 5e-5 against the FP64 reference -- the reference's own
f32 tolerance (test_kernels.cpp:41-61).  The p = 1 thread and p = 2 lane
kernels compute in FP32; at p >= 3 the default FP32 output is the FP64 DMMA
result rounded at the store (exactly the FP64 matrices rounded), and
VARIANT_TC32 runs the contraction on the tcgen05 tensor cores (3xTF32,
kernels_tc32.cuh) -- measured <= 5e-7."""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import REF_SO, Oracle, Reference, laplace_tensor, rel_frobenius

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BOUND = 5e-5


def run(p, mesh, mode, coeff, dtype, n_eq=1, layout=pb.OUT_CANONICAL, variant=pb.VARIANT_AUTO):
    n = len(mesh)
    dim = n_eq * pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    c = coeff
    if mode in (pb.PER_ELEMENT, pb.ELASTICITY):
        c = torch.from_numpy(np.ascontiguousarray(np.asarray(coeff).reshape(n, -1).T)).cuda()
    with pb.Integrator(p, n_eq=n_eq, variant=variant) as it:
        if layout == pb.OUT_CANONICAL:
            out = torch.full((n, dim, dim), float("nan"), dtype=dtype, device="cuda")
            it.integrate_device(n, g, out, mode, c)
        else:
            out = torch.full((dim * dim, n + 1), float("nan"), dtype=dtype, device="cuda")
            it.integrate_device(n, g, out, mode, c, out_layout=pb.OUT_SOA, ld_out=n + 1)
        it.check()
    res = out.double().cpu().numpy()
    if layout == pb.OUT_SOA:
        res = res[:, :n].T.reshape(n, dim, dim)
    return res


@pytest.mark.parametrize("p", range(1, 8))
@pytest.mark.parametrize("form", ["laplace", "cdr", "elasticity"])
def test_f32_output_bound(p, form):
    mesh = pb.generate_box_mesh(2, 2, 1, 0.2, seed=p)
    n = len(mesh)
    n_eq, mode, coeff = 1, pb.LAPLACE, None
    if form == "cdr":
        mode, coeff = pb.PER_ELEMENT, pb.generate_cdr_coefficients(7, 0, n)
    elif form == "elasticity":
        n_eq, mode, coeff = 3, pb.ELASTICITY, pb.generate_materials(0, n)
    k32 = run(p, mesh, mode, coeff, torch.float32, n_eq)
    k64 = run(p, mesh, mode, coeff, torch.float64, n_eq)
    assert np.isfinite(k32).all()
    err = rel_frobenius(k64, k32, axis=(1, 2))
    assert err.max() <= BOUND, err.max()
    if n_eq == 1 and p <= 2:  # FP32 arithmetic
        assert err.max() <= 1e-5, err.max()
    else:  # FP64 arithmetic: the FP32 matrices are exactly the FP64 ones rounded
        assert err.max() <= 1e-6, err.max()
        assert np.array_equal(k32, k64.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
def test_f32_soa_layout(p):
    mesh = pb.generate_box_mesh(3, 2, 1, 0.1, seed=3)
    a = run(p, mesh, pb.LAPLACE, None, torch.float32, layout=pb.OUT_SOA)
    b = run(p, mesh, pb.LAPLACE, None, torch.float32)
    assert np.array_equal(a, b)


def test_f32_against_reference():
    p = 3
    mesh = pb.generate_box_mesh(2, 2, 2, 0.2, seed=11)
    k32 = run(p, mesh, pb.LAPLACE, None, torch.float32)
    idx = [0, len(mesh) - 1]
    if REF_SO.exists():
        ref, err = Reference().integrate_batch(p, mesh[idx], laplace_tensor(), threads=0)
        assert err is None
    else:
        ref = Oracle().integrate_batch(p, mesh[idx], laplace_tensor())
    assert rel_frobenius(ref, k32[idx], axis=(1, 2)).max() <= BOUND


@pytest.mark.parametrize("p", [3, 4, 5, 6, 7])
@pytest.mark.parametrize("form", ["laplace", "cdr", "symmetric"])
def test_f32_tensor_core_path_against_reference(p, form):
    """VARIANT_TC32 (tcgen05 3xTF32, p >= 3) against the reference's
    integrate_generic, ragged element counts (partial persistent waves), and the
    SoA layout against the canonical one."""
    mesh = pb.generate_box_mesh(3, 3, 2, 0.2, seed=p + 20)[: 7 + p]
    n = len(mesh)
    coeff = None
    mode = pb.LAPLACE
    ref_c = laplace_tensor()
    if form == "cdr":
        mode = pb.PER_ELEMENT
        coeff = pb.generate_cdr_coefficients(3, 0, n)
        ref_c = coeff
    elif form == "symmetric":
        rng = np.random.default_rng(p)
        a = rng.standard_normal((4, 4))
        coeff = (a @ a.T + 4 * np.eye(4)).reshape(16)
        mode = pb.UNIFORM
        ref_c = coeff
    k32 = run(p, mesh, mode, coeff, torch.float32, variant=pb.VARIANT_TC32)
    assert np.isfinite(k32).all()
    soa = run(p, mesh, mode, coeff, torch.float32, variant=pb.VARIANT_TC32, layout=pb.OUT_SOA)
    assert np.array_equal(soa, k32)
    idx = [0, n // 2, n - 1]
    rc = np.asarray(ref_c).reshape(-1, 16)
    rc = rc if len(rc) == 1 else rc[idx]
    if REF_SO.exists():
        ref, err = Reference().integrate_batch(p, mesh[idx], rc, threads=0)
        assert err is None
    else:
        ref = Oracle().integrate_batch(p, mesh[idx], rc)
    e = rel_frobenius(ref, k32[idx], axis=(1, 2)).max()
    assert e <= 1e-5, e
