"""Compile-time launch shapes of the sum-factorised kernels (tools/sumfact_configs.cu,
host-compiled with nvcc): every configuration fits the SM's shared memory at
its CTAs-per-SM target, and the natural-order consumers' H loads stay at the
conflict-free wavefront count the stride search promises."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SMEM_PER_SM = 228 * 1024   # B200: 228 KB per SM, 227 KB max per CTA, 1 KB reserved per CTA
SMEM_PER_CTA = 227 * 1024


@pytest.fixture(scope="module")
def configs(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    exe = tmp_path_factory.mktemp("cfg") / "sumfact_configs"
    subprocess.run([nvcc, "-std=c++17", "--expt-relaxed-constexpr", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", str(ROOT / "include"), str(ROOT / "tools" / "sumfact_configs.cu"), "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    rows = []
    for line in out.splitlines():
        kv = dict(re.findall(r"([\w/-]+)=\s*([\d.]+)", line))
        rows.append(kv)
    assert len(rows) == 15  # 13 (p, n_eq) shapes + the symmetric p = 3, 4 shapes
    return rows


def test_shared_memory_fits(configs):
    for c in configs:
        smem = float(c["smem"]) * 1024
        minb = int(c["minb"])
        assert smem <= SMEM_PER_CTA, c
        assert minb * (smem + 1024) <= SMEM_PER_SM, c


def test_natural_order_h_loads_conflict_free(configs):
    # per (k-step, n-tile): 4 quarter-warp wavefronts (16-byte plane) + 2 half-warp ones (8-byte plane)
    for c in configs:
        if int(c["tmajor"]) == 0:
            ntile = min(int(c["NTILE"]), 8)
            ideal = 3 * ntile * (4 + 2)
            assert int(c["cons-wavefronts"]) <= ideal * 1.25, c


def test_ring_depths(configs):
    for c in configs:
        assert 2 <= int(c["nbuf"]) <= 6, c
