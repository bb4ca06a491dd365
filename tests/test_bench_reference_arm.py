"""bench.py's reference arm (the reference's own CPU integrate_generic on the
host cores) keeps the driver's JSON contract -- runs here without a GPU."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

from oracle_lib import REF_SO

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not REF_SO.exists(), reason="reference library not built")
def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--p", "1,2"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "elements/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
