"""Output buffers at any element-aligned address.  The kernels store whole
element matrices with TMA bulk copies (cp.async.bulk), which need 16-byte
aligned global addresses; an output base that is only 8-byte (FP64) or 4-byte
(FP32) aligned must take the per-element head/tail or plain-store paths and
give the same bits.  Covers every kernel family: p = 1 thread, p = 2 lane,
sum factorisation (row split, t'-major pairs, pair split), and the n_eq = 3
lane / warp / CTA kernels.
"""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def integrate(p, mesh, mode, coeff, n_eq, dtype, shift):
    """K computed into buf[shift : shift + n*dim*dim] of a flat buffer."""
    n = len(mesh)
    dim = n_eq * pb.shape_count(p)
    g = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
    c = coeff
    if mode in (pb.PER_ELEMENT, pb.ELASTICITY):
        c = torch.from_numpy(np.ascontiguousarray(np.asarray(coeff).reshape(n, -1).T)).cuda()
    buf = torch.full((n * dim * dim + 8,), float("nan"), dtype=dtype, device="cuda")
    out = buf[shift:shift + n * dim * dim]
    assert out.data_ptr() % 16 == (shift * buf.element_size()) % 16
    with pb.Integrator(p, n_eq=n_eq) as it:
        it.integrate_device(n, g, out, mode, c)
        it.check()
    host = buf.cpu()
    # nothing written outside the output range
    assert torch.isnan(host[:shift]).all() and torch.isnan(host[shift + n * dim * dim:]).all()
    return out.cpu().double().numpy().reshape(n, dim, dim)


CASES = [(p, "laplace") for p in range(1, 8)] + [(p, "cdr") for p in (1, 2, 3, 4)] + \
        [(p, "elasticity") for p in (1, 2, 3, 4)]


@pytest.mark.parametrize("p,form", CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32], ids=["f64", "f32"])
def test_unaligned_output_same_bits(p, form, dtype):
    mesh = pb.generate_box_mesh(3, 2, 1, 0.2, seed=11 + p)  # 12 prisms: odd/even element offsets
    n = len(mesh)
    n_eq, mode, coeff = 1, pb.LAPLACE, None
    if form == "cdr":
        mode, coeff = pb.PER_ELEMENT, pb.generate_cdr_coefficients(5, 0, n)
    elif form == "elasticity":
        n_eq, mode, coeff = 3, pb.ELASTICITY, pb.generate_materials(3, n)
    ref = integrate(p, mesh, mode, coeff, n_eq, dtype, 0)
    assert np.isfinite(ref).all()
    shifts = (1, 2, 3) if dtype == torch.float32 else (1,)
    for shift in shifts:
        got = integrate(p, mesh, mode, coeff, n_eq, dtype, shift)
        assert np.array_equal(got, ref), (p, form, shift)


def integrate_inputs(p, mesh, mode, coeff, n_eq, shift, extra):
    """Geometry / coefficients read from SoA buffers starting `shift` doubles
    into the allocation, with a row pitch of n + extra."""
    n = len(mesh)
    dim = n_eq * pb.shape_count(p)
    ld = n + extra

    def soa(aos):
        aos = np.asarray(aos, dtype=np.float64).reshape(n, -1)
        flat = np.full(shift + aos.shape[1] * ld, np.nan)
        flat[shift:].reshape(aos.shape[1], ld)[:, :n] = aos.T
        return torch.from_numpy(flat).cuda()[shift:]

    g = soa(mesh.reshape(n, 18))
    c = soa(coeff) if mode in (pb.PER_ELEMENT, pb.ELASTICITY) else None
    out = torch.full((n, dim, dim), float("nan"), dtype=torch.float64, device="cuda")
    with pb.Integrator(p, n_eq=n_eq) as it:
        it.integrate_device(n, g, out, mode, c, geom_ld=ld, coeff_ld=ld if c is not None else None)
        it.check()
    return out.cpu().numpy()


@pytest.mark.parametrize("p,form", CASES)
def test_shifted_strided_inputs_same_bits(p, form):
    mesh = pb.generate_box_mesh(3, 2, 1, 0.2, seed=31 + p)
    n = len(mesh)
    n_eq, mode, coeff = 1, pb.LAPLACE, None
    if form == "cdr":
        mode, coeff = pb.PER_ELEMENT, pb.generate_cdr_coefficients(9, 0, n)
    elif form == "elasticity":
        n_eq, mode, coeff = 3, pb.ELASTICITY, pb.generate_materials(4, n)
    ref = integrate_inputs(p, mesh, mode, coeff, n_eq, 0, 0)
    assert np.isfinite(ref).all()
    for shift, extra in ((1, 3), (3, 1)):
        assert np.array_equal(integrate_inputs(p, mesh, mode, coeff, n_eq, shift, extra), ref), (shift, extra)
