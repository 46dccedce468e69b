"""bench.py's JSON line keeps the driver contract (a short run on the GPU: small batch, no
CPU baseline) -- every key the contract names, with consistent values."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--batch", "16", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--converge-games", "4",
                          "--converge-max-steps", "40"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["dtype"] == "f64"
    assert line["value"] == pytest.approx(4 * 16 * 3 / (line["ms_per_step"] * 3 / 1e3), rel=1e-6)
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"])
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] == 8 * 16 and 0 < e2e["value"] < line["value"]
    assert line["gpu_launches"] > 0 and line["clocks"]["samples"] >= 1
    assert "workload" in line["config"] and "l2" in line["config"]
