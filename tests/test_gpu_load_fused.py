"""Load vectors with the stiffness pass (pi_integrate_load),
fused into every scalar stiffness kernel family (LOAD_FUSED) and as the
separate sum-factorised launch (LOAD_SEPARATE).

F_i = sum_q det w_q f phi_i(x_q) has no reference entry point;
it equals f times column 0 of the mass matrix integrate_generic returns for
c[0][0][0][0] = 1 (phi_0 = 1), which is the checker here -- the reference's
own integrate_generic (oracle/_ref) when built, else the C restatement's
load_vector (pinned to that column and to exact Poly3 integrals in
tests/test_oracle.py).  Bars: F within 1e-12 relative Frobenius per element;
K from the fused call bitwise equal to K from pi_integrate (the fused kernels
must not perturb the stiffness arithmetic).
"""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import REF_SO, Oracle, Reference, rel_frobenius, sample_indices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


def mass_column_checker(p, geoms, f):
    """f * column 0 of the c[0][0][0][0] = 1 mass matrix (integrate_generic)."""
    if REF_SO.exists():
        c = np.zeros(16)
        c[0] = 1.0
        k, err = Reference().integrate_batch(p, geoms, c, threads=0)
        assert err is None
        return k[:, :, 0] * f[:, None]
    o = Oracle()
    return np.stack([o.load_vector(p, g, fe) for g, fe in zip(geoms, f)])


def sym_tensor():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((4, 4))
    c = a @ a.T + 4 * np.eye(4)  # symmetric, non-zero value/derivative couplings c[0][k]
    return c.reshape(16)


FORMS = ["laplace", "cdr", "symmetric"]


@pytest.mark.parametrize("fusion", [pb.LOAD_FUSED, pb.LOAD_SEPARATE])
@pytest.mark.parametrize("p", range(1, 8))
@pytest.mark.parametrize("form", FORMS)
def test_fused_load_vectors(p, form, fusion):
    mesh = pb.generate_box_mesh(5, 3, 3, 0.2, seed=17)
    n = len(mesh) if p <= 4 else (13 if p == 5 else 5)  # ragged: partial CTAs / element groups
    mesh = mesh[:n]
    nsh = pb.shape_count(p)
    geom = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    mode, coeff = pb.LAPLACE, None
    if form == "cdr":
        mode = pb.PER_ELEMENT
        coeff = torch.from_numpy(np.ascontiguousarray(pb.generate_cdr_coefficients(42, 0, n).T)).cuda()
    elif form == "symmetric":
        mode, coeff = pb.UNIFORM, sym_tensor()
    f = np.linspace(0.5, 2.0, n)
    fd = torch.from_numpy(f).cuda()
    with pb.Integrator(p) as it:
        it.set_load_fusion(fusion)
        k_plain = torch.full((n, nsh, nsh), float("nan"), dtype=torch.float64, device="cuda")
        it.integrate_device(n, geom, k_plain, mode, coeff)
        k_fused = torch.full_like(k_plain, float("nan"))
        load = torch.full((n, nsh), float("nan"), dtype=torch.float64, device="cuda")
        it.integrate_device(n, geom, k_fused, mode, coeff, load_out=load, f=fd)
        load_c = torch.full_like(load, float("nan"))
        it.integrate_device(n, geom, torch.empty_like(k_plain), mode, coeff, load_out=load_c, f_const=1.5)
        it.check()
    kp, kf = k_plain.cpu().numpy(), k_fused.cpu().numpy()
    assert np.array_equal(kp.view(np.uint64), kf.view(np.uint64)), "fused load vectors changed K"
    got, got_c = load.cpu().numpy(), load_c.cpu().numpy()
    assert np.isfinite(got).all() and np.isfinite(got_c).all(), "unwritten load-vector entries"
    idx = sample_indices(n, min(n, 6))
    ref = mass_column_checker(p, mesh[idx], f[idx])
    err = rel_frobenius(ref, got[idx], axis=1)
    assert err.max() <= TOL, f"p={p} {form}: load vector error {err.max():.3e}"
    ref_c = mass_column_checker(p, mesh[idx], np.full(len(idx), 1.5))
    assert rel_frobenius(ref_c, got_c[idx], axis=1).max() <= TOL


@pytest.mark.parametrize("p", [2, 3])
def test_fused_load_vectors_sumfact_variant_and_standalone(p):
    """p = 2 through the sum-factorised kernel, and the standalone pi_load_vectors
    (sum-factorised for p >= 2) against the fused result."""
    mesh = pb.generate_box_mesh(4, 4, 2, 0.2, seed=3)
    n = len(mesh)
    nsh = pb.shape_count(p)
    geom = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    f = torch.linspace(1.0, 3.0, n, dtype=torch.float64, device="cuda")
    with pb.Integrator(p, variant=pb.VARIANT_SUMFACT) as it:
        it.set_load_fusion(pb.LOAD_FUSED)
        load = torch.full((n, nsh), float("nan"), dtype=torch.float64, device="cuda")
        it.integrate_device(n, geom, torch.empty((n, nsh, nsh), dtype=torch.float64, device="cuda"), pb.LAPLACE,
                            load_out=load, f=f)
        alone = torch.full_like(load, float("nan"))
        it.load_vectors_device(n, geom, alone, f=f)
        it.check()
    a, b = load.cpu().numpy(), alone.cpu().numpy()
    assert rel_frobenius(a, b, axis=1).max() <= TOL
    idx = sample_indices(n, 5)
    ref = mass_column_checker(p, mesh[idx], f.cpu().numpy()[idx])
    assert rel_frobenius(ref, a[idx], axis=1).max() <= TOL


def test_fused_load_vectors_contract():
    mesh = pb.generate_box_mesh(2, 2, 1, 0.1, seed=1)
    n = len(mesh)
    geom = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    with pb.Integrator(2, n_eq=3) as it:
        mats = torch.from_numpy(np.ascontiguousarray(pb.generate_materials(0, n).T)).cuda()
        out = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        with pytest.raises(pb.ConfigError):
            it.integrate_device(n, geom, out, pb.ELASTICITY, mats,
                                load_out=torch.empty((n, it.n_shape), dtype=torch.float64, device="cuda"))
    with pb.Integrator(2) as it:
        with pytest.raises(pb.ConfigError):
            it.set_load_fusion(7)
        out32 = torch.empty((n, 18, 18), dtype=torch.float32, device="cuda")
        with pytest.raises(pb.ContractViolation):
            it.integrate_device(n, geom, out32, pb.LAPLACE, load_out=torch.empty((n, 18), dtype=torch.float64,
                                                                                  device="cuda"))
        with pytest.raises(pb.ContractViolation):  # load buffer too small
            it.integrate_device(n, geom, torch.empty((n, 18, 18), dtype=torch.float64, device="cuda"), pb.LAPLACE,
                                load_out=torch.empty((n - 1, 18), dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_host_path_load_vectors(p):
    """pi_integrate_host_load (the run_batch-style host path, chunked through
    device memory) equals the device path bit for bit, K and F."""
    mesh = pb.generate_box_mesh(5, 3, 2, 0.2, seed=23)
    n = len(mesh)
    f = np.linspace(0.25, 1.75, n)
    with pb.Integrator(p) as it:
        k_h, f_h = it.integrate_host_load(mesh, pb.LAPLACE, f=f, chunk_elems=7)
        geom = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
        k_d = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        f_d = torch.empty((n, it.n_shape), dtype=torch.float64, device="cuda")
        it.integrate_device(n, geom, k_d, pb.LAPLACE, load_out=f_d, f=torch.from_numpy(f).cuda())
        it.check()
        k_c, f_c = it.integrate_host_load(mesh, pb.LAPLACE, f_const=2.0)
    assert np.array_equal(k_h, k_d.cpu().numpy()) and np.array_equal(f_h, f_d.cpu().numpy())
    idx = sample_indices(n, 4)
    assert rel_frobenius(mass_column_checker(p, mesh[idx], np.full(len(idx), 2.0)), f_c[idx], axis=1).max() <= TOL
    assert np.array_equal(k_c, k_h)
