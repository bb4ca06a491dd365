"""Host side of the product (CPU only): per-p constants, synthetic inputs, the
C-ABI surface and its error behaviour without a GPU."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import Oracle

ROOT = Path(__file__).resolve().parent.parent
GOLD = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def declared_symbols():
    text = (ROOT / "include" / "prism_b200.h").read_text()
    return sorted(set(re.findall(r"\b(pi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = pb.library()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", str(pb.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(pi_[a-z0-9_]+)\b", nm))
    assert set(syms) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(pb.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_dmma_in_sass():
    sass = subprocess.run(["cuobjdump", "-sass", str(pb.LIB_PATH)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass


@pytest.mark.parametrize("p", range(1, 8))
def test_rule_and_table_bitwise_equal_reference(p):
    pts, w = pb.prism_quadrature(p)
    assert np.array_equal(pts, GOLD[f"quad_points_p{p}"])
    assert np.array_equal(w, GOLD[f"quad_weights_p{p}"])
    assert sha(pb.tabulate_shapes(p)) == str(GOLD[f"shape_sha_p{p}"])


def test_counts_and_domain_errors():
    assert [pb.shape_count(p) for p in range(1, 8)] == [6, 18, 40, 75, 126, 196, 288]
    assert [pb.quadrature_point_count(p) for p in range(1, 8)] == [6, 18, 48, 80, 150, 231, 336]
    for bad in (0, 8, -1):
        with pytest.raises(pb.DomainError):
            pb.shape_count(bad)
        with pytest.raises(pb.DomainError):
            pb.prism_quadrature(bad)


def test_box_mesh_bitwise_and_ranges():
    assert np.array_equal(pb.generate_box_mesh(4, 3, 2, 0.2, 5), GOLD["mesh_4_3_2_d02_s5"])
    assert np.array_equal(pb.generate_box_mesh(1, 1, 1, 0.0), GOLD["mesh_1_1_1_d0_default"])
    assert sha(pb.generate_box_mesh(16, 16, 8, 0.1, 42)) == str(GOLD["mesh_sha_16_16_8_d01_s42"])
    full = GOLD["mesh_4_3_2_d02_s5"]
    for first, count in [(0, 1), (5, 7), (47, 1), (0, 48), (13, 0)]:
        aos = pb.generate_box_mesh(4, 3, 2, 0.2, 5, first=first, count=count)
        assert np.array_equal(aos, full[first:first + count])
        soa = pb.generate_box_mesh(4, 3, 2, 0.2, 5, first=first, count=count, soa=True, ld=count + 3)
        assert np.array_equal(soa[:, :count].T.reshape(count, 6, 3), full[first:first + count])


def test_box_mesh_errors():
    with pytest.raises(pb.DomainError):
        pb.generate_box_mesh(0, 1, 1, 0.1)
    with pytest.raises(pb.DomainError):
        pb.generate_box_mesh(1, 1, 1, 0.3)
    with pytest.raises(pb.ContractViolation):
        pb.generate_box_mesh(1, 1, 1, 0.1, first=1, count=5)


def test_box_mesh_validation_catches_nothing_on_valid_meshes():
    pb.generate_box_mesh(3, 3, 3, 0.25, seed=1, validate=True)


def test_cdr_coefficients_range_independent_and_physical():
    full = pb.generate_cdr_coefficients(42, 0, 100)
    part = pb.generate_cdr_coefficients(42, 37, 20)
    assert np.array_equal(full[37:57], part)
    soa = pb.generate_cdr_coefficients(42, 37, 20, soa=True, ld=21)
    assert np.array_equal(soa[:, :20].T, part)
    c = full.reshape(-1, 4, 4)
    d = c[:, 1:, 1:]
    assert np.allclose(d, np.transpose(d, (0, 2, 1)), atol=1e-15)  # symmetric diffusion
    eig = np.linalg.eigvalsh(d)
    assert eig.min() >= 0.5 - 1e-12 and eig.max() <= 2.0 + 1e-12
    assert np.all(np.abs(c[:, 0, 1:]) <= 1.0) and np.all((c[:, 0, 0] >= 0) & (c[:, 0, 0] <= 1))
    assert np.all(c[:, 1:, 0] == 0.0)
    assert not np.array_equal(pb.generate_cdr_coefficients(43, 0, 10), full[:10])


def test_checker_side_generators_equal_product():
    """bench.py's reference arm draws its CDR tensors and materials from the
    numpy restatements in tests/oracle_lib.py (it must not load the product
    library): they must give the product generator's values."""
    from oracle_lib import cdr_coefficients, materials

    for first, count in ((0, 257), (1048000, 1000), (16777000, 216)):
        assert np.array_equal(cdr_coefficients(42, first, count), pb.generate_cdr_coefficients(42, first, count))
        assert np.array_equal(materials(first, count), pb.generate_materials(first, count))


def test_flop_and_byte_models():
    # SURVEY.md 8(d) table
    want_lap = {1: 3390, 2: 48402, 3: 531408, 4: 2910080, 5: 14934750, 6: 54773565, 7: 170459184}
    want_cdr = {1: 4326, 2: 64602, 3: 711888, 4: 3894080, 5: 19962150, 6: 73155621, 7: 227552304}
    for p in range(1, 8):
        assert pb.flops_dense_per_element(p, pb.LAPLACE) == want_lap[p]
        assert pb.flops_dense_per_element(p, pb.PER_ELEMENT) == want_cdr[p]
    assert pb.bytes_per_element(7, pb.LAPLACE) == 663696
    assert pb.bytes_per_element(2, pb.PER_ELEMENT) == 2864


def test_context_without_gpu_fails_loudly():
    """No CPU fallback: on a box without a device, creating a context raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pb.CudaError):
        pb.Integrator(2)


def test_context_argument_errors():
    with pytest.raises(pb.DomainError):
        pb.Integrator(9)
    with pytest.raises(pb.ConfigError):
        pb.Integrator(2, n_eq=2)  # systems: n_eq = 1 or 3
    pts, w = pb.prism_quadrature(2)
    tab = pb.tabulate_shapes(2)
    with pytest.raises(pb.ConfigError):  # p mismatch (integrate_ref.cpp:36-46)
        pb.Integrator(3, points=pts, weights=w, shape_table=tab)


def test_status_names_mirror_errc():
    lib = pb.library()
    names = [lib.pi_status_name(i).decode() for i in range(10)]
    assert names == ["ok", "config", "domain", "unsupported_degree", "inverted_element", "capacity",
                     "shared_memory_exhausted", "contract_violation", "io", "cuda"]


def test_oracle_and_product_agree_on_mesh():
    o = Oracle()
    assert np.array_equal(o.box_mesh(5, 2, 3, 0.15, 77), pb.generate_box_mesh(5, 2, 3, 0.15, 77))
