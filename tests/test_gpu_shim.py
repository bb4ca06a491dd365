"""The C++ drop-in (include/prism_b200_prismint.hpp) driven with the reference's
own types, checked against the reference's integrate_generic (tests/cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "build" / "shim_test"


@pytest.mark.gpu
def test_prismint_shim():
    if not BIN.exists():
        pytest.skip("shim_test not built (needs the reference headers at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
