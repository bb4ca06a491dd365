"""Host-path error handling and context isolation (the reference rethrows a
worker's exception only after every worker joined, kernels.cpp:47-57, and
checks buffers up front, kernels.cpp:423-462; lame_parameters rejects bad
materials, coefficients.cpp:23-32)."""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def soa(a):
    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a.reshape(len(a), -1).T)).cuda()


@pytest.mark.parametrize("p", [1, 2, 4])
def test_inverted_element_mid_stream(p):
    """An inverted element in a middle chunk of the streamed host path: the
    call reports it (after every chunk's copies settled) and the context
    stays usable."""
    mesh = pb.generate_box_mesh(4, 4, 2, 0.1, seed=3).copy()
    mesh[37, [0, 2]] = mesh[37, [2, 0]]
    with pb.Integrator(p) as it:
        with pytest.raises(pb.InvertedElementError) as ei:
            it.integrate_host(mesh, chunk_elems=5, element_id_base=1000)
        assert ei.value.element == 1037 and ei.value.det <= 0
        ok = pb.generate_box_mesh(4, 4, 2, 0.1, seed=3)
        assert np.isfinite(it.integrate_host(ok, chunk_elems=5)).all()


def test_stale_device_error_surfaces_on_next_host_call():
    """An unchecked asynchronous device call's inverted element surfaces on the
    next host-buffer call (header contract) with its own id -- never an
    out-of-range read of this call's buffer -- and the call after is clean."""
    p = 3
    bad = pb.generate_box_mesh(3, 3, 2, 0.1, seed=4).copy()
    bad[20, [0, 1]] = bad[20, [1, 0]]
    good = pb.generate_box_mesh(2, 2, 1, 0.1, seed=5)
    n = len(bad)
    with pb.Integrator(p) as it:
        out = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        it.integrate_device(n, soa(bad), out, element_id_base=5_000_000)
        with pytest.raises(pb.InvertedElementError) as ei:
            it.integrate_host(good, element_id_base=0)
        assert ei.value.element == 5_000_020
        ref = it.integrate_host(good)
        assert np.isfinite(ref).all()


def test_two_contexts_with_different_rules_run_concurrently():
    """Per-context tables: a context whose rule weights are doubled (exact in
    binary) gives exactly 2 K while another context runs the default rule on
    another stream at the same time (p = 2 and p = 1 elasticity kernels once
    read shared __constant__ tables)."""
    for p, n_eq, mode in ((2, 1, pb.LAPLACE), (2, 3, pb.ELASTICITY), (1, 3, pb.ELASTICITY)):
        pts, w = pb.prism_quadrature(p)
        tab = pb.tabulate_shapes(p, pts)
        mesh = pb.generate_box_mesh(8, 8, 4, 0.1, seed=p)
        n = len(mesh)
        g = soa(mesh)
        mats = soa(pb.generate_materials(0, n)) if n_eq == 3 else None
        a = pb.Integrator(p, n_eq=n_eq)
        b = pb.Integrator(p, n_eq=n_eq, points=pts, weights=2.0 * w, shape_table=tab)
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        oa = torch.empty((n, a.dim, a.dim), dtype=torch.float64, device="cuda")
        ob = torch.empty_like(oa)
        for _ in range(4):  # interleaved launches on two streams
            a.integrate_device(n, g, oa, mode, mats, stream=sa.cuda_stream)
            b.integrate_device(n, g, ob, mode, mats, stream=sb.cuda_stream)
        a.check()
        b.check()
        torch.cuda.synchronize()
        ka, kb = oa.cpu().numpy(), ob.cpu().numpy()
        a.close()
        b.close()
        assert np.array_equal(2.0 * ka, kb), (p, n_eq)


def test_material_domain_errors():
    p = 2
    mesh = pb.generate_box_mesh(2, 2, 2, 0.1, seed=6)
    n = len(mesh)
    with pb.Integrator(p, n_eq=3) as it:
        for young, nu in ((0.0, 0.3), (-1.0, 0.3), (1.0, 0.5), (1.0, -1.0), (1.0, 0.7)):
            with pytest.raises(pb.DomainError):
                it.integrate_host(mesh, pb.ELASTICITY_UNIFORM, np.array([young, nu]))
        mats = pb.generate_materials(0, n).copy()
        mats[11, 1] = 0.6
        mats[5, 0] = -2.0
        with pytest.raises(pb.DomainError) as ei:  # host buffers: checked before any launch
            it.integrate_host(mesh, pb.ELASTICITY, mats, element_id_base=100)
        assert "105" in str(ei.value)
        # device buffers: the kernels flag the lowest offending element
        out = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        it.integrate_device(n, soa(mesh), out, pb.ELASTICITY, soa(mats), element_id_base=100)
        with pytest.raises(pb.DomainError) as ei:
            it.check()
        assert "105" in str(ei.value)
        it.check()  # flags reset
    with pb.Integrator(4, n_eq=3) as it:  # sum-factorised elasticity
        mats = pb.generate_materials(0, n).copy()
        mats[3, 1] = -1.5
        out = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        it.integrate_device(n, soa(mesh), out, pb.ELASTICITY, soa(mats))
        with pytest.raises(pb.DomainError):
            it.check()


def test_device_argument_validation():
    with pb.Integrator(2) as it:
        mesh = pb.generate_box_mesh(2, 2, 1, 0.1, seed=1)
        n = len(mesh)
        g = soa(mesh)
        out = torch.empty((n, it.dim, it.dim), dtype=torch.float64, device="cuda")
        with pytest.raises(pb.ContractViolation):  # non-contiguous geometry view
            it.integrate_device(n, torch.empty((n, 18), dtype=torch.float64, device="cuda").t(), out)
        with pytest.raises(pb.ContractViolation):  # output too small
            it.integrate_device(n, g, out[:-1])
        with pytest.raises(pb.ContractViolation):  # wrong dtype
            it.integrate_device(n, g.float(), out)
        with pytest.raises(pb.ContractViolation):  # host tensor
            it.integrate_device(n, g.cpu(), out)
        with pytest.raises(pb.ContractViolation):  # coefficient width (per-element CDR needs 16 rows)
            it.integrate_device(n, g, out, pb.PER_ELEMENT, torch.zeros((15, n), dtype=torch.float64, device="cuda"))
        with pytest.raises(pb.ContractViolation):
            it.integrate_host(mesh, pb.PER_ELEMENT, np.zeros((n, 15)))
