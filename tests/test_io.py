"""Stiffness containers, host only: the reference's
PRISTIF1 (save_stiffness / load_stiffness, io.cpp:112-168) reproduced byte for
byte, and the FP64 batch container PRISTIF2 (exact round trip)."""
import numpy as np
import pytest

import paper_1310_1191_b200 as pb
from oracle_lib import REF_SO, Reference


def matrices(p, n_eq, count, seed):
    dim = n_eq * pb.shape_count(p)
    rng = np.random.default_rng(seed)
    return rng.normal(size=(count, dim, dim)) * 10.0 ** rng.integers(-3, 4, size=(count, 1, 1))


@pytest.mark.parametrize("p,n_eq", [(1, 1), (3, 1), (2, 3)])
def test_pristif2_roundtrip_is_exact(tmp_path, p, n_eq):
    k = matrices(p, n_eq, 5, p)
    f = tmp_path / "k.pristif2"
    pb.save_stiffness(f, k, p, n_eq, element_id_base=1000)
    got, info = pb.load_stiffness(f)
    assert info == {"format": pb.PRISTIF2, "p": p, "n_eq": n_eq, "count": 5, "element_id_base": 1000}
    assert np.array_equal(got, k)  # bit-exact FP64


@pytest.mark.skipif(not REF_SO.exists(), reason="reference library not built")
@pytest.mark.parametrize("p,n_eq", [(1, 1), (2, 1), (1, 3)])
def test_pristif1_matches_reference_bytes(tmp_path, p, n_eq):
    ref = Reference()
    if not ref.has_io:
        pytest.skip("reference io.cpp not built (no nlohmann json)")
    k = matrices(p, n_eq, 1, 10 + p)
    ours, theirs = tmp_path / "ours.bin", tmp_path / "theirs.bin"
    pb.save_stiffness(ours, k, p, n_eq, element_id_base=42, fmt=pb.PRISTIF1)
    ref.save_stiffness(theirs, p, n_eq, k[0], 42)
    assert ours.read_bytes() == theirs.read_bytes()
    # each side reads the other's file
    m, eid, rp, rn = ref.load_stiffness(ours)
    assert (eid, rp, rn) == (42, p, n_eq)
    assert np.array_equal(m, k[0].astype(np.float32).astype(np.float64))
    got, info = pb.load_stiffness(theirs)
    assert info["format"] == pb.PRISTIF1 and info["element_id_base"] == 42
    assert np.array_equal(got[0], m)


def test_container_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTSTIF0" + b"\0" * 16)
    with pytest.raises(pb.IoError):
        pb.load_stiffness(bad)
    k = matrices(1, 1, 2, 0)
    f = tmp_path / "k.bin"
    with pytest.raises(pb.ConfigError):  # PRISTIF1 holds one matrix
        pb.save_stiffness(f, k, 1, fmt=pb.PRISTIF1)
    pb.save_stiffness(f, k, 1)
    f.write_bytes(f.read_bytes()[:-8])  # truncated payload
    with pytest.raises(pb.IoError):
        pb.load_stiffness(f)
    with pytest.raises(pb.IoError):
        pb.load_stiffness(tmp_path / "missing.bin")
