"""Inverted-element detection in every kernel (geometry.cpp:67-69 raises
InvertedElementError(element_id, xi, det) on det <= 0; kernels.cpp:158, 249
report the global id base + local).  With several inverted elements the
library reports the lowest global id (pi_check).  Fault injection as in the
reference's verify.cpp:315-336: swap two vertices of an element."""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FORMS = [(p, f) for f in ("laplace", "cdr", "elasticity") for p in range(1, 8)]


def run(p, mesh, form, base, dtype=torch.float64):
    n = len(mesh)
    n_eq, mode, coeff = 1, pb.LAPLACE, None
    if form == "cdr":
        mode, coeff = pb.PER_ELEMENT, pb.generate_cdr_coefficients(2, 0, n)
    elif form == "elasticity":
        n_eq, mode, coeff = 3, pb.ELASTICITY, pb.generate_materials(2, n)
    dim = n_eq * pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    c = None if coeff is None else torch.from_numpy(np.ascontiguousarray(np.asarray(coeff).reshape(n, -1).T)).cuda()
    out = torch.empty((n, dim, dim), dtype=dtype, device="cuda")
    with pb.Integrator(p, n_eq=n_eq) as it:
        it.integrate_device(n, g, out, mode, c, element_id_base=base)
        it.check()
    return out


@pytest.mark.parametrize("p,form", FORMS)
def test_lowest_inverted_global_id(p, form):
    mesh = pb.generate_box_mesh(3, 2, 1, 0.1, seed=p).copy()
    for e in (9, 4):
        mesh[e, [1, 2]] = mesh[e, [2, 1]]
    with pytest.raises(pb.InvertedElementError) as ei:
        run(p, mesh, form, base=7000)
    assert ei.value.element == 7004
    assert ei.value.det <= 0.0


@pytest.mark.parametrize("p,form", [(1, "laplace"), (2, "laplace"), (3, "laplace"), (4, "cdr"),
                                    (1, "elasticity"), (2, "elasticity"), (3, "elasticity")])
def test_inverted_late_in_persistent_loop(p, form):
    """2048 elements: every CTA of the persistent grids integrates several
    elements (p3_elastic_mma_kernel forms element e+1's Jacobians inside
    element e's iteration); inversions far from the first wave are reported,
    the lowest global id first."""
    mesh = pb.generate_box_mesh(16, 8, 8, 0.1, seed=p).copy()
    assert len(mesh) == 2048
    for e in (1999, 1501):
        mesh[e, [0, 2]] = mesh[e, [2, 0]]
    with pytest.raises(pb.InvertedElementError) as ei:
        run(p, mesh, form, base=10)
    assert ei.value.element == 1511
    assert ei.value.det <= 0.0


@pytest.mark.parametrize("p", [2, 4])
def test_inverted_detected_in_f32_variant(p):
    mesh = pb.generate_box_mesh(2, 2, 1, 0.1, seed=1).copy()
    mesh[5, [0, 1]] = mesh[5, [1, 0]]
    with pytest.raises(pb.InvertedElementError) as ei:
        run(p, mesh, "laplace", base=0, dtype=torch.float32)
    assert ei.value.element == 5


@pytest.mark.parametrize("n_eq", [1, 3])
def test_empty_batch_is_a_no_op(n_eq):
    """n_elem = 0: PI_OK, nothing written (every p, both precisions)."""
    for p in range(1, 8):
        dim = n_eq * pb.shape_count(p)
        g = torch.zeros((18, 1), dtype=torch.float64, device="cuda")
        for dtype in (torch.float64, torch.float32):
            out = torch.full((dim * dim,), 7.0, dtype=dtype, device="cuda")
            with pb.Integrator(p, n_eq=n_eq) as it:
                mode = pb.LAPLACE if n_eq == 1 else pb.ELASTICITY_UNIFORM
                coeff = None if n_eq == 1 else np.array([1.0, 0.3])
                it.integrate_device(0, g, out, mode, coeff)
                it.check()
            assert bool((out == 7.0).all())


@pytest.mark.parametrize("form", ["cdr", "elasticity"])
def test_single_and_odd_counts(form):
    """1, 2 and 37 elements through every kernel of the weak form: each equals the full-batch result."""
    mesh = pb.generate_box_mesh(4, 3, 2, 0.15, seed=8)
    for p in range(1, 8):
        full = run(p, mesh[:37], form, base=0).cpu()
        for n in (1, 2):
            # coefficients / materials are pure functions of the element id
            assert torch.equal(run(p, mesh[:n], form, base=0).cpu(), full[:n])
