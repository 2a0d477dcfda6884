"""The driver-facing bench.py contract on a small configuration: one JSON line
with the required keys (metric / value / unit / ... / roofline / e2e /
gpu_launches / clocks) and internally consistent numbers.  The headline run
itself is the driver's (`python bench.py`); this only guards the format."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks")


@pytest.mark.timeout(300)
def test_bench_json_line_cfg1():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--config", "cfg1", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-extras", "--e2e-steps", "2", "--no-as-shipped"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    missing = [k for k in REQUIRED if k not in line]
    assert not missing, missing
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["higher_is_better"] is False and line["unit"] == "ms/call"
    assert line["value"] > 0 and abs(line["value"] - line["ms_per_step"]) < 1e-9
    assert line["gpu_launches"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-6
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
