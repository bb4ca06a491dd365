"""GPU parity: the sm_100a kernels (through the C ABI) against the checker.

The checker is the reference's own integrate_generic (oracle/_ref, compiled
from the unmodified sources) when present, else the plain-C restatement
(oracle/liboracle.so), which is bitwise equal to it (tests/test_oracle.py).
Bar: per-element relative Frobenius <= 1e-12 (north star; comparator
verify.cpp:461-469).
"""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import Oracle, Reference, REF_SO, laplace_tensor, rel_frobenius, sample_indices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12
# Oracle samples per p, sized so the CPU checker finishes in seconds.
SAMPLE = {1: 64, 2: 48, 3: 24, 4: 12, 5: 6, 6: 3, 7: 2}


def checker_batch(p, geoms, coeffs):
    """Reference integrate_generic on the sampled elements (threads), else the C oracle."""
    if REF_SO.exists():
        out, err = Reference().integrate_batch(p, geoms, coeffs, threads=0)
        assert err is None
        return out
    return Oracle().integrate_batch(p, geoms, coeffs)


def device_soa(aos, extra_ld=0):
    """AoS [n][w] host -> device SoA [w][n + extra_ld] (ld padding exercises geom_ld)."""
    aos = np.asarray(aos, dtype=np.float64).reshape(len(aos), -1)
    n, w = aos.shape
    buf = np.zeros((w, n + extra_ld))
    buf[:, :n] = aos.T
    return torch.from_numpy(buf).cuda()


def run_gpu(p, mesh, mode, coeff=None, layout=pb.OUT_CANONICAL, base=0, extra_ld=0, **kw):
    n = len(mesh)
    nsh = pb.shape_count(p)
    g = device_soa(mesh.reshape(n, 18), extra_ld)
    it = pb.Integrator(p, **kw)
    c = None
    if mode == pb.PER_ELEMENT:
        c = device_soa(coeff.reshape(n, 16), extra_ld)
    elif mode == pb.UNIFORM:
        c = coeff
    if layout == pb.OUT_CANONICAL:
        out = torch.full((n, nsh, nsh), float("nan"), dtype=torch.float64, device="cuda")
        it.integrate_device(n, g, out, mode, c, element_id_base=base)
    else:
        out = torch.full((nsh * nsh, n + 3), float("nan"), dtype=torch.float64, device="cuda")
        it.integrate_device(n, g, out, mode, c, element_id_base=base, out_layout=pb.OUT_SOA, ld_out=n + 3)
    it.check()
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    it.close()
    if layout == pb.OUT_SOA:
        res = res[:, :n].T.reshape(n, nsh, nsh)
    return res


@pytest.mark.parametrize("p", range(1, 8))
def test_laplace_matches_reference(p):
    mesh = pb.generate_box_mesh(4, 4, 3, 0.2, seed=42)  # 96 distorted prisms
    got = run_gpu(p, mesh, pb.LAPLACE)
    assert np.isfinite(got).all(), "unwritten output entries"
    idx = sample_indices(len(mesh), SAMPLE[p])
    ref = checker_batch(p, mesh[idx], laplace_tensor())
    err = rel_frobenius(ref, got[idx], axis=(1, 2))
    assert err.max() <= TOL, f"p={p} worst rel-Frobenius {err.max():.3e}"


@pytest.mark.parametrize("p", range(1, 8))
def test_cdr_per_element_matches_reference(p):
    mesh = pb.generate_box_mesh(4, 3, 3, 0.15, seed=7)  # 72 prisms
    coeff = pb.generate_cdr_coefficients(42, 0, len(mesh))
    got = run_gpu(p, mesh, pb.PER_ELEMENT, coeff, extra_ld=5)
    assert np.isfinite(got).all()
    idx = sample_indices(len(mesh), SAMPLE[p])
    ref = checker_batch(p, mesh[idx], coeff[idx])
    err = rel_frobenius(ref, got[idx], axis=(1, 2))
    assert err.max() <= TOL, f"p={p} worst rel-Frobenius {err.max():.3e}"


@pytest.mark.parametrize("p", [1, 2, 4, 7])
def test_uniform_tensor_and_layouts(p):
    mesh = pb.generate_box_mesh(3, 2, 2, 0.1, seed=3)  # 24 prisms (ragged vs CTA batching)
    lap = run_gpu(p, mesh, pb.LAPLACE)
    uni = run_gpu(p, mesh, pb.UNIFORM, laplace_tensor())
    assert rel_frobenius(lap, uni) <= 1e-13
    soa = run_gpu(p, mesh, pb.LAPLACE, layout=pb.OUT_SOA)
    assert np.array_equal(lap, soa)
    again = run_gpu(p, mesh, pb.LAPLACE)
    assert np.array_equal(lap, again), "not bitwise deterministic"


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_ragged_counts_and_twins(p):
    base = pb.generate_box_mesh(2, 2, 2, 0.2, seed=5)
    for n in (1, 2, 3, 5, 9, 33, 47):
        mesh = np.concatenate([base] * 2)[:n]
        got = run_gpu(p, mesh, pb.LAPLACE)
        assert np.isfinite(got).all()
        ref = checker_batch(p, mesh[:1], laplace_tensor())
        assert rel_frobenius(ref[0], got[0]) <= TOL
    twins = np.stack([base[3]] * 4)
    out = run_gpu(p, twins, pb.LAPLACE)
    for k in range(1, 4):
        assert np.array_equal(out[0], out[k])


@pytest.mark.parametrize("p", [1, 2, 6])
def test_inverted_element_reports_global_id(p):
    mesh = pb.generate_box_mesh(2, 2, 1, 0.0)
    mesh[6, [0, 1]] = mesh[6, [1, 0]]  # kernels.cpp test: swap two vertices of element 6
    with pytest.raises(pb.InvertedElementError) as ei:
        run_gpu(p, mesh, pb.LAPLACE, base=100)
    assert ei.value.element == 106
    assert ei.value.det <= 0.0
    # the context stays usable afterwards
    ok = pb.generate_box_mesh(2, 2, 1, 0.0)
    assert np.isfinite(run_gpu(p, ok, pb.LAPLACE)).all()


@pytest.mark.parametrize("p", [1, 3, 7])
def test_reference_tables_drop_in(p):
    """The context accepts the reference's own rule + shape table (run_batch path)."""
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    r = Reference()
    pts, w = r.quadrature(p)
    tab = r.shape_table(p)
    mesh = pb.generate_box_mesh(2, 2, 2, 0.2, seed=9)
    a = run_gpu(p, mesh, pb.LAPLACE)
    b = run_gpu(p, mesh, pb.LAPLACE, points=pts, weights=w, shape_table=tab)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_host_buffer_path_equals_device_path(p):
    mesh = pb.generate_box_mesh(4, 4, 2, 0.2, seed=11)
    coeff = pb.generate_cdr_coefficients(5, 0, len(mesh))
    dev = run_gpu(p, mesh, pb.PER_ELEMENT, coeff)
    with pb.Integrator(p) as it:
        host = it.integrate_host(mesh, pb.PER_ELEMENT, coeff, chunk_elems=7)  # many ragged chunks
    assert np.array_equal(dev, host)
    lap = pb.run_batch(p, mesh)
    assert np.array_equal(lap, run_gpu(p, mesh, pb.LAPLACE))


@pytest.mark.parametrize("p", range(1, 8))
def test_load_vectors(p):
    mesh = pb.generate_box_mesh(3, 3, 2, 0.2, seed=13)
    n = len(mesh)
    f = np.linspace(0.5, 2.0, n)
    g = device_soa(mesh.reshape(n, 18))
    out = torch.zeros((n, pb.shape_count(p)), dtype=torch.float64, device="cuda")
    fd = torch.from_numpy(f).cuda()
    with pb.Integrator(p) as it:
        it.load_vectors_device(n, g, out, f=fd)
        it.check()
    got = out.cpu().numpy()
    o = Oracle()
    for e in sample_indices(n, 4):
        ref = o.load_vector(p, mesh[e], f[e])
        assert rel_frobenius(ref, got[e]) <= TOL
