"""bench.py's JSON line contract (the driver parses it): the reference arm on CPU,
the B200 arm on the GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["unit"] == "ms/step" and d["higher_is_better"] is False
    assert d["metric"].startswith("PowerSGD") and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "resnet18 rank 2, W=1"  # identical to the B200 arm's
    assert "numpy" in d["cpu_baseline"] and "cpu_model" in d["cpu_baseline"]


@pytest.mark.gpu
def test_b200_arm_line():
    d = run_bench("--steps", "5", "--warmup", "3", "--no-cpu")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["higher_is_better"] is False
    assert d["config"]["workload"] == "resnet18 rank 2, W=1" and "l2" in d["config"]
    assert d["config"]["back_to_back_ms"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5 and r["peak"] > 1000
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert d["value"] < 1.0  # ms/step: ResNet-18 rank 2 on one B200
