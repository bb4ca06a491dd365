"""GPU parity for systems (n_eq = 3): isotropic linear elasticity -- the
reference's own model problem (integrate_optimized, integrate_ref.cpp:93-130;
elasticity_tensor, coefficients.cpp:40-59; the material input of its batch
API, MaterialData per element, kernels.hpp:47-50) -- and general n_eq = 3
coefficient tensors, against the reference's integrate_generic /
integrate_optimized (oracle/_ref) or the C restatement.

Bar: per-element relative Frobenius <= 1e-12, like the reference's own
optimized == generic check (test_integrate_ref.cpp:117-129).
"""
from pathlib import Path

import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import REF_SO, Oracle, Reference, rel_frobenius

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12
GOLD = np.load(Path(__file__).parent / "golden" / "reference_golden.npz")
SAMPLE = {1: 6, 2: 5, 3: 4, 4: 3, 5: 2, 6: 1, 7: 1}


def elasticity_tensor(young, nu):
    if REF_SO.exists():
        out = np.zeros(144)
        import ctypes as C
        assert Reference().lib.ref_elasticity_tensor(young, nu, out.ctypes.data_as(C.POINTER(C.c_double)), None) == 0
        return out.reshape(3, 3, 4, 4)
    return Oracle().elasticity_tensor(young, nu)


def checker(p, geoms, coeffs):
    """integrate_generic with n_eq = 3 on the given elements."""
    if REF_SO.exists():
        out, err = Reference().integrate_batch(p, geoms, coeffs, n_eq=3, threads=0)
        assert err is None
        return out
    return Oracle().integrate_batch(p, geoms, coeffs, n_eq=3)


def materials(n, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(0.5, 2.0, n), rng.uniform(0.0, 0.45, n)], axis=1)  # (E, nu)


def run(p, geoms, mode, coeff=None, base=0):
    n = len(geoms)
    dim = 3 * pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(geoms.reshape(n, 18).T)).cuda()
    out = torch.full((n, dim, dim), float("nan"), dtype=torch.float64, device="cuda")
    c = coeff
    if mode in (pb.ELASTICITY, pb.PER_ELEMENT):
        c = torch.from_numpy(np.ascontiguousarray(np.asarray(coeff).reshape(n, -1).T)).cuda()
    with pb.Integrator(p, n_eq=3) as it:
        it.integrate_device(n, g, out, mode, c, element_id_base=base)
        it.check()
    return out.cpu().numpy()


@pytest.mark.parametrize("p", range(1, 8))
def test_elasticity_per_element_materials(p):
    mesh = pb.generate_box_mesh(3, 2, 2, 0.2, seed=40 + p)
    mats = materials(len(mesh), p)
    got = run(p, mesh, pb.ELASTICITY, mats)
    assert np.isfinite(got).all()
    idx = np.linspace(0, len(mesh) - 1, SAMPLE[p]).astype(int)
    ref = checker(p, mesh[idx], np.stack([elasticity_tensor(*mats[i]) for i in idx]))
    err = rel_frobenius(ref, got[idx], axis=(1, 2))
    assert err.max() <= TOL, err
    # K is symmetric (major symmetry of the tensor)
    k = got[idx]
    assert np.abs(k - np.transpose(k, (0, 2, 1))).max() <= 1e-13 * np.abs(k).max()


@pytest.mark.parametrize("p", [1, 2])
def test_elasticity_golden(p):
    """Committed reference outputs (generic and optimized) for E=3, nu=0.25."""
    geom = GOLD["K_laplace_geoms_p1"][1]  # the reference's distorted prism
    got = run(p, geom[None], pb.ELASTICITY_UNIFORM, np.array([3.0, 0.25]))[0]
    assert rel_frobenius(GOLD[f"K_elasticity_generic_p{p}"], got) <= TOL
    assert rel_frobenius(GOLD[f"K_elasticity_optimized_p{p}"], got) <= TOL


@pytest.mark.parametrize("p", [2, 4, 7])
def test_elasticity_matches_integrate_optimized(p):
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    mesh = pb.generate_box_mesh(2, 2, 1, 0.15, seed=p)
    got = run(p, mesh, pb.ELASTICITY_UNIFORM, np.array([2.0, 0.3]))
    for e in (0, len(mesh) - 1):
        ref = Reference().integrate_optimized(p, mesh[e], 2.0, 0.3)
        assert rel_frobenius(ref, got[e]) <= TOL


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_general_system_tensor(p):
    """Any n_eq = 3 tensor (value and derivative slots, nonsymmetric), uniform and per element."""
    rng = np.random.default_rng(100 + p)
    mesh = pb.generate_box_mesh(2, 2, 1, 0.2, seed=p)
    n = len(mesh)
    base = elasticity_tensor(1.0, 0.3)
    cs = base[None] + 0.1 * rng.normal(size=(n, 3, 3, 4, 4))
    got = run(p, mesh, pb.PER_ELEMENT, cs.reshape(n, 144))
    idx = [0, n // 2, n - 1]
    ref = checker(p, mesh[idx], cs[idx])
    assert rel_frobenius(ref, got[idx], axis=(1, 2)).max() <= TOL
    got_u = run(p, mesh[:2], pb.UNIFORM, cs[0])
    ref_u = checker(p, mesh[:2], cs[0][None])
    assert rel_frobenius(ref_u, got_u, axis=(1, 2)).max() <= TOL


def test_symmetric_system_tensor_path():
    """The elasticity tensor passed as a UNIFORM tensor takes the symmetric path."""
    p = 2
    mesh = pb.generate_box_mesh(2, 2, 2, 0.2, seed=9)
    c = elasticity_tensor(1.5, 0.2)
    got = run(p, mesh, pb.UNIFORM, c)
    ref = run(p, mesh, pb.ELASTICITY_UNIFORM, np.array([1.5, 0.2]))
    assert rel_frobenius(ref, got, axis=(1, 2)).max() <= TOL


@pytest.mark.parametrize("p", [1, 3])
def test_rigid_translations_annihilated(p):
    """K u = 0 for rigid translations (test_integrate_ref.cpp:53-68)."""
    mesh = pb.generate_box_mesh(2, 1, 1, 0.2, seed=3)
    k = run(p, mesh, pb.ELASTICITY_UNIFORM, np.array([1.0, 0.25]))
    nsh = pb.shape_count(p)
    # constant function = dof of (t=0, a=0) with value 1 (m_0 = P_0 = 1)
    for d in range(3):
        u = np.zeros(3 * nsh)
        u[0 * 3 + d] = 1.0
        r = k @ u
        assert np.abs(r).max() <= 1e-12 * np.abs(k).max()


def test_elasticity_host_path_and_run_batch():
    p = 3
    mesh = pb.generate_box_mesh(3, 3, 2, 0.1, seed=5)
    mats = materials(len(mesh), 7)
    dev = run(p, mesh, pb.ELASTICITY, mats)
    with pb.Integrator(p, n_eq=3) as it:
        host = it.integrate_host(mesh, pb.ELASTICITY, mats, chunk_elems=7)
    assert np.array_equal(dev, host)
    rb = pb.run_batch(p, mesh, pb.ELASTICITY_UNIFORM, np.array([1.0, 0.3]), n_eq=3)
    assert rb.shape == (len(mesh), 3 * pb.shape_count(p), 3 * pb.shape_count(p))


def test_elasticity_inverted_element_and_errors():
    p = 2
    mesh = pb.generate_box_mesh(2, 2, 1, 0.1, seed=1).copy()
    mesh[5, [0, 1]] = mesh[5, [1, 0]]  # fault injection (verify.cpp:315-336)
    with pytest.raises(pb.InvertedElementError) as ei:
        run(p, mesh, pb.ELASTICITY_UNIFORM, np.array([1.0, 0.3]), base=1000)
    assert ei.value.element == 1005
    with pb.Integrator(p, n_eq=3) as it:
        g = torch.zeros((18, 4), dtype=torch.float64, device="cuda")
        out = torch.zeros(4 * 54 * 54, dtype=torch.float64, device="cuda")
        with pytest.raises(pb.ConfigError):
            it.integrate_device(4, g, out, pb.LAPLACE)
        with pytest.raises(pb.DomainError):
            it.integrate_device(4, g, out, pb.ELASTICITY_UNIFORM, np.array([1.0, 0.5]))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_elasticity_soa_layout(p):
    """PI_OUT_SOA ([dim^2][ld]) carries the same matrices as the canonical layout."""
    mesh = pb.generate_box_mesh(2, 2, 1, 0.1, seed=21)
    n = len(mesh)
    dim = 3 * pb.shape_count(p)
    mats = materials(n, p)
    canon = run(p, mesh, pb.ELASTICITY, mats)
    g = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    c = torch.from_numpy(np.ascontiguousarray(mats.T)).cuda()
    out = torch.full((dim * dim, n + 5), float("nan"), dtype=torch.float64, device="cuda")
    with pb.Integrator(p, n_eq=3) as it:
        it.integrate_device(n, g, out, pb.ELASTICITY, c, out_layout=pb.OUT_SOA, ld_out=n + 5)
        it.check()
    soa = out.cpu().numpy()[:, :n].T.reshape(n, dim, dim)
    assert np.array_equal(soa, canon)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_sumfact_variant_at_low_p(p):
    """The DMMA sum-factorisation strategy (pi_context_set_variant SUMFACT) for
    n_eq = 3 at p <= 3, where the default is the dense lane / warp / CTA kernels."""
    mesh = pb.generate_box_mesh(2, 2, 1, 0.2, seed=60 + p)
    n = len(mesh)
    mats = materials(n, 60 + p)
    dim = 3 * pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    c = torch.from_numpy(np.ascontiguousarray(mats.T)).cuda()
    res = {}
    for v in (pb.VARIANT_DENSE, pb.VARIANT_SUMFACT):
        out = torch.full((n, dim, dim), float("nan"), dtype=torch.float64, device="cuda")
        with pb.Integrator(p, n_eq=3, variant=v) as it:
            it.integrate_device(n, g, out, pb.ELASTICITY, c)
            it.check()
        res[v] = out.cpu().numpy()
    assert rel_frobenius(res[pb.VARIANT_DENSE], res[pb.VARIANT_SUMFACT], axis=(1, 2)).max() <= TOL
