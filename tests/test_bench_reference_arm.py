"""bench.py's reference arm (the reference's own CPU integrate_generic on the
host cores) keeps the driver's JSON contract, prints the same config dict as
our arm, and never loads the product library -- runs here without a GPU."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

from oracle_lib import REF_SO

ROOT = Path(__file__).resolve().parent.parent

PROBE = r"""
import io, json, sys, contextlib
sys.path.insert(0, {root!r})
import bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    rc = bench.main(["--impl", "reference", "--steps", "1", "--warmup", "1", "--p", "1,2"] + {extra!r})
maps = open("/proc/self/maps").read()
print(json.dumps({{"rc": rc, "line": buf.getvalue().strip().splitlines()[-1],
                  "product_loaded": "libprism_b200" in maps, "ref_loaded": "libprismint_ref" in maps}}))
"""


def run_arm(extra):
    r = subprocess.run([sys.executable, "-c", PROBE.format(root=str(ROOT), extra=extra)], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["rc"] == 0
    return out


@pytest.mark.skipif(not REF_SO.exists(), reason="reference library not built")
def test_reference_arm_json_contract():
    out = run_arm([])
    line = json.loads(out["line"])
    assert not out["product_loaded"], "the reference arm must not load libprism_b200.so"
    assert out["ref_loaded"]
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "elements/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    # ms_per_step is the measured wall time of the sampled step (fits the run)
    assert 0 < line["ms_per_step"] < 120_000


@pytest.mark.skipif(not REF_SO.exists(), reason="reference library not built")
def test_reference_arm_config_equals_ours():
    import bench

    line = json.loads(run_arm(["--coeff", "cdr"])["line"])
    args = bench.parse(["--p", "1,2", "--coeff", "cdr"])
    assert line["config"] == json.loads(json.dumps(bench.Workload(args, 1, 0).config()))


def test_workload_partitions():
    import bench

    a = bench.parse(["--scaling", "strong"])
    ws = 3
    spans = [(bench.Workload(a, ws, r).first, bench.Workload(a, ws, r).E) for r in range(ws)]
    assert spans[0][0] == 0 and sum(e for _, e in spans) == 16777216
    for (f0, e0), (f1, _) in zip(spans, spans[1:]):
        assert f0 + e0 == f1
    w = bench.Workload(bench.parse([]), 4, 2)
    assert (w.E, w.first, w.total, w.mesh) == (1048576, 2 * 1048576, 4 * 1048576, (128, 64, 256))
    assert [bench.sample_count(p) for p in range(1, 8)] == [256, 256, 256, 256, 64, 16, 16]
