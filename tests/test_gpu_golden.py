"""GPU kernels against the committed golden vectors (produced by running the
reference itself, tests/golden/gen_golden.py): Laplace and a nonsymmetric
uniform CDR tensor on the reference's own "right" and "distorted" prisms
(test_integrate_ref.cpp:118-119) for p = 1..7.  Needs no reference tree."""
from pathlib import Path

import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import Oracle, laplace_tensor, rel_frobenius

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "reference_golden.npz")


def integrate(p, geoms, mode, coeff=None):
    n = len(geoms)
    nsh = pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(geoms.reshape(n, 18).T)).cuda()
    out = torch.full((n, nsh, nsh), float("nan"), dtype=torch.float64, device="cuda")
    with pb.Integrator(p) as it:
        it.integrate_device(n, g, out, mode, coeff)
        it.check()
    return out.cpu().numpy()


@pytest.mark.parametrize("p", range(1, 8))
def test_golden_laplace(p):
    geoms = GOLD[f"K_laplace_geoms_p{p}"]
    got = integrate(p, geoms, pb.LAPLACE)
    err = rel_frobenius(GOLD[f"K_laplace_p{p}"], got, axis=(1, 2))
    assert err.max() <= 1e-12, err


@pytest.mark.parametrize("p", range(1, 8))
def test_golden_cdr_uniform_nonsymmetric(p):
    geoms = GOLD[f"K_laplace_geoms_p{p}"]
    c = GOLD["cdr_tensor"]
    assert not np.array_equal(c, c.T)
    got = integrate(p, geoms, pb.UNIFORM, c)
    err = rel_frobenius(GOLD[f"K_cdr_p{p}"], got, axis=(1, 2))
    assert err.max() <= 1e-12, err


@pytest.mark.parametrize("p", range(1, 8))
def test_symmetric_uniform_tensor_path(p):
    """A symmetric anisotropic tensor with value/derivative couplings
    c[0][k] = c[k][0] != 0 takes the symmetric (mirrored) path of every launch
    shape, including the w0 terms of the pair-split kernel."""
    rng = np.random.default_rng(p)
    a = rng.normal(size=(3, 3))
    c = np.zeros((4, 4))
    c[1:, 1:] = np.eye(3) + 0.2 * (a + a.T)
    c[0, 0] = 0.7
    b = 0.3 * rng.normal(size=3)
    c[0, 1:] = b
    c[1:, 0] = b
    assert np.array_equal(c, c.T)
    geoms = pb.generate_box_mesh(3, 2, 2, 0.2, seed=p)
    got = integrate(p, geoms, pb.UNIFORM, c)
    assert np.abs(got - np.transpose(got, (0, 2, 1))).max() <= 1e-13 * np.abs(got).max()
    o = Oracle()
    for e in (0, len(geoms) // 2, len(geoms) - 1):
        ref = o.integrate_generic(p, geoms[e], c)
        assert rel_frobenius(ref, got[e]) <= 1e-12
