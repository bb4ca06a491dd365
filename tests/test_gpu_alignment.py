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
