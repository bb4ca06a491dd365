"""The checker itself is pinned before it is trusted (CPU only).

1. The C restatement (oracle/liboracle.so) reproduces the reference's golden
   vectors BITWISE (tests/golden/reference_golden.npz, produced by running the
   reference sources, tests/golden/gen_golden.py).
2. It reproduces the reference's own known-answer tests
   (test_integrate_ref.cpp, test_reference_element.cpp, test_geometry.cpp)
   restated here, including the exact-polynomial Laplace KAT.
3. When oracle/_ref is built, it agrees with the live reference too.
"""
import hashlib

import numpy as np
import pytest

from oracle_lib import Oracle, Reference, REF_SO, laplace_tensor, rel_frobenius, shape_count, QUAD_COUNTS
from poly3 import basis_polynomial

GOLD = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "reference_golden.npz")


@pytest.fixture(scope="module")
def o():
    return Oracle()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("p", range(1, 8))
def test_quadrature_and_shapes_bitwise(o, p):
    pts, w = o.quadrature(p)
    assert np.array_equal(pts, GOLD[f"quad_points_p{p}"])
    assert np.array_equal(w, GOLD[f"quad_weights_p{p}"])
    tab = o.shape_table(p)
    assert sha(tab) == str(GOLD[f"shape_sha_p{p}"])


def test_table_sizes(o):
    # test_reference_element.cpp:20-28 and :298-312
    assert [shape_count(p) for p in range(1, 8)] == [6, 18, 40, 75, 126, 196, 288]
    assert [QUAD_COUNTS[p] for p in range(1, 8)] == [6, 18, 48, 80, 150, 231, 336]
    for deg, n in zip((2, 4, 6, 8, 10, 12, 14), (3, 6, 12, 16, 25, 33, 42)):
        pts, w = o.triangle_rule(deg)
        assert len(pts) == n
        assert abs(w.sum() - 0.5) < 1e-12  # weights sum to the reference area
    with pytest.raises(ValueError):
        o.triangle_rule(3)


@pytest.mark.parametrize("p", range(1, 8))
def test_prism_rule_volume_and_exactness(o, p):
    # test_reference_element.cpp:109-151: volume 1, monomials up to the rule degree
    pts, w = o.quadrature(p)
    assert abs(w.sum() - 1.0) < 1e-12
    from poly3 import Poly3
    for a, b, c in [(p, p, 0), (2 * p - 1, 1, 2 * p + 1), (0, 2 * p, 2 * p)]:
        exact = float(Poly3.monomial(a, b, c).integral_over_reference_prism())
        got = float(np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c))
        assert abs(got - exact) <= 1e-12 * max(1.0, abs(exact))


def test_meshes_bitwise(o):
    assert np.array_equal(o.box_mesh(4, 3, 2, 0.2, 5), GOLD["mesh_4_3_2_d02_s5"])
    assert np.array_equal(o.box_mesh(2, 2, 2, 0.2, 5), GOLD["mesh_2_2_2_d02_s5"])
    assert np.array_equal(o.box_mesh(1, 1, 1, 0.0, 0x5072697342657631), GOLD["mesh_1_1_1_d0_default"])
    assert sha(o.box_mesh(16, 16, 8, 0.1, 42)) == str(GOLD["mesh_sha_16_16_8_d01_s42"])


def test_mesh_volume_conserved(o):
    # test_geometry.cpp:188-199: sum over elements of sum_q w det == 1
    for d in (0.0, 0.1):
        mesh = o.box_mesh(4, 4, 4, d, 42)
        pts, w = o.quadrature(2)
        vol = 0.0
        for g in mesh:
            for q in range(len(w)):
                rc, det, _ = o.jacobian_terms(g, pts[q])
                assert rc == 0 and det > 0
                vol += w[q] * det
        assert abs(vol - 1.0) < 1e-12


@pytest.mark.parametrize("p", range(1, 8))
def test_integrate_generic_bitwise_vs_golden(o, p):
    geoms = GOLD[f"K_laplace_geoms_p{p}"]
    for kind, coeff in (("laplace", laplace_tensor()), ("cdr", GOLD["cdr_tensor"])):
        want = GOLD[f"K_{kind}_p{p}"]
        got = o.integrate_batch(p, geoms, coeff)
        assert np.array_equal(got, want), f"{kind} p={p}: max diff {np.abs(got - want).max()}"


def test_elasticity_generic_vs_golden(o):
    el = o.elasticity_tensor(3.0, 0.25)
    assert np.array_equal(el, GOLD["elasticity_tensor_3_025"])
    g = GOLD["mesh_2_2_2_d02_s5"][9]
    for p in (1, 2):
        got = o.integrate_generic(p, g, el, n_eq=3)
        assert np.array_equal(got, GOLD[f"K_elasticity_generic_p{p}"])
        # integrate_optimized == integrate_generic at 1e-12 (test_integrate_ref.cpp:117-129)
        assert rel_frobenius(GOLD[f"K_elasticity_optimized_p{p}"], got) <= 1e-12


def test_laplace_p2_identity_prism_exact(o):
    """test_integrate_ref.cpp:70-92 with the exact Poly3 integrals."""
    ident = np.array([[0, 0, -1], [1, 0, -1], [0, 1, -1], [0, 0, 1], [1, 0, 1], [0, 1, 1]], dtype=float)
    a = o.integrate_generic(2, ident, laplace_tensor())
    for r, s in [(0, 0), (3, 7), (11, 2), (17, 17), (5, 14)]:
        pr, ps = basis_polynomial(2, r), basis_polynomial(2, s)
        integrand = pr.derivative(0) * ps.derivative(0) + pr.derivative(1) * ps.derivative(1) + \
            pr.derivative(2) * ps.derivative(2)
        exact = float(integrand.integral_over_reference_prism())
        assert abs(a[r, s] - exact) <= 1e-12 * max(1.0, abs(exact))


@pytest.mark.parametrize("p", range(1, 8))
def test_load_vector_exact_on_identity(o, p):
    """F_i(f=1) = int phi_i exactly and = M[i][0]."""
    ident = np.array([[0, 0, -1], [1, 0, -1], [0, 1, -1], [0, 0, 1], [1, 0, 1], [0, 1, 1]], dtype=float)
    f = o.load_vector(p, ident, 1.0)
    for i in range(shape_count(p)):
        exact = float(basis_polynomial(p, i).integral_over_reference_prism())
        assert abs(f[i] - exact) <= 1e-12 * max(1.0, abs(exact))
    if p <= 4:
        mass = np.zeros((1, 1, 4, 4))
        mass[0, 0, 0, 0] = 1.0
        g = GOLD["mesh_2_2_2_d02_s5"][9]
        m = o.integrate_generic(p, g, mass)
        assert np.array_equal(o.load_vector(p, g, 1.0), m[:, 0])


def test_symmetry_and_rigid_modes(o):
    # test_integrate_ref.cpp:53-68 (constant mode) and :131-149 (symmetry)
    g = GOLD["mesh_2_2_2_d02_s5"][9]
    for p in (1, 2, 3):
        a = o.integrate_generic(p, g, laplace_tensor())
        assert np.sqrt(((a - a.T) ** 2).sum() / (a * a).sum()) <= 1e-12
        u = np.zeros(shape_count(p))
        u[0] = 1.0  # the constant field lies in the null space
        assert np.abs(a @ u).max() <= 1e-12 * np.abs(a).sum(axis=1).max()


def test_inverted_element_detected(o):
    g = GOLD["mesh_1_1_1_d0_default"][0].copy()
    g[[0, 1]] = g[[1, 0]]
    from oracle_lib import InvertedElement
    with pytest.raises(InvertedElement) as ei:
        o.integrate_generic(2, g, laplace_tensor())
    assert ei.value.where == 0  # first rule point already fails


@pytest.mark.skipif(not REF_SO.exists(), reason="reference library not built here")
def test_restatement_equals_live_reference(o):
    r = Reference()
    mesh = o.box_mesh(3, 2, 2, 0.25, 99)
    coeffs = np.random.default_rng(0).normal(size=(len(mesh), 16))
    for p in (1, 2, 3):
        ref, err = r.integrate_batch(p, mesh, coeffs, threads=0)
        assert err is None
        got = np.stack([o.integrate_generic(p, mesh[e], coeffs[e]) for e in range(len(mesh))])
        assert np.array_equal(ref, got)
