"""bench.py's reference arm runs on CPU and prints one contract-shaped JSON line."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle import oracle as O


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-seconds", "0.2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"


def test_model_flops_matches_survey():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.model_flops(32, 32, 8, 2) == 3891200
    assert bench.model_flops(64, 64, 16, 10) == 32645120   # C3
    assert bench.model_flops(32, 32, 8, 2, "d") == 282624


def test_newton_model_flops():
    sys.path.insert(0, ROOT)
    import bench
    # n = 32: 11,968 complex products and 11,440 complex additions per solve (docstring of the model)
    assert bench.newton_model_flops(32) == 11968 * 80 + 11440 * 40
    assert bench.newton_model_flops(1) == 2 * 80 + 1 * 40  # one inverse, one dx product, x + dx
