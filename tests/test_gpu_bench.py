"""The bench contract on the GPU: `bench.py` prints one JSON line with the keys the driver
reads, a roofline object against the MUFU peak, e2e through the public API, the launch
count and the clocks sampled during the timed region."""
import json
import os
import subprocess
import sys

import pytest

from gpu_helpers import require_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line():
    require_gpu()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--no-cpu"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["scaling"] == "weak"
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 1_000_000 * 7 * 4 and e["d2h_bytes_per_step"] == 5_000_000
    assert line["gpu_launches"] >= 2 * 2  # FK + score (+ finalize) per step
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
