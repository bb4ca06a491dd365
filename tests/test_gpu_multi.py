"""Multi-GPU host path: pi_integrate_host_multi splits the mesh
into contiguous element ranges over several contexts (one per device, one
host thread each).  The box here has one GPU, so the contexts share it; the
partition, threading and error logic are the same.  Results must be bitwise
identical to one context (test_kernels.cpp:98-110: bitwise determinism
across worker-pool widths)."""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,n_ctx", [(1, 2), (3, 3), (5, 2)])
def test_multi_context_bitwise(p, n_ctx):
    mesh = pb.generate_box_mesh(5, 3, 2, 0.15, seed=p)
    coeff = pb.generate_cdr_coefficients(3, 0, len(mesh))
    with pb.Integrator(p) as one:
        ref = one.integrate_host(mesh, pb.PER_ELEMENT, coeff)
    its = [pb.Integrator(p) for _ in range(n_ctx)]
    try:
        got = pb.integrate_host_multi(its, mesh, pb.PER_ELEMENT, coeff, chunk_elems=7)
    finally:
        for it in its:
            it.close()
    assert np.array_equal(ref, got)


def test_multi_context_elasticity_and_errors():
    p = 2
    mesh = pb.generate_box_mesh(4, 2, 2, 0.1, seed=8).copy()
    mats = pb.generate_materials(0, len(mesh))
    its = [pb.Integrator(p, n_eq=3) for _ in range(2)]
    try:
        with pb.Integrator(p, n_eq=3) as one:
            ref = one.integrate_host(mesh, pb.ELASTICITY, mats)
        assert np.array_equal(ref, pb.integrate_host_multi(its, mesh, pb.ELASTICITY, mats))
        # inverted elements in both halves: the lowest global id is reported
        n = len(mesh)
        for e in (n - 3, n // 2 + 1):
            mesh[e, [0, 1]] = mesh[e, [1, 0]]
        with pytest.raises(pb.InvertedElementError) as ei:
            pb.integrate_host_multi(its, mesh, pb.ELASTICITY, mats, element_id_base=500)
        assert ei.value.element == 500 + n // 2 + 1
        with pytest.raises(pb.ContractViolation):  # the same context twice
            pb.integrate_host_multi([its[0], its[0]], mesh, pb.ELASTICITY, mats)
    finally:
        for it in its:
            it.close()
