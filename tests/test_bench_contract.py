"""The bench.py contract on the CPU-only arm (`--impl reference`, the oracle on the host cores): one JSON line
with the keys the driver reads (test infrastructure: the reference arm is the one place bench.py runs the
oracle)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    assert b["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in b, k
    assert b["value"] > 0 and b["higher_is_better"] is True and b["n_gpus"] == 1
    assert b["cpu_baseline"]["kind"] == "oracle" and b["cpu_baseline"]["cores"] >= 1
    assert b["e2e"]["h2d_bytes_per_step"] == 0 and b["e2e"]["d2h_bytes_per_step"] == 0
    assert b["config"]["workload"].startswith("c1")


import pytest  # noqa: E402


@pytest.mark.gpu
def test_our_arm_json_line():
    """Our arm on a small config: the roofline, e2e, clocks and launch-count keys the driver checks."""
    out = subprocess.run([sys.executable, "bench.py", "--config", "c2", "--steps", "3", "--warmup", "3",
                          "--no-stages", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    assert b["value"] > 0 and b["n_gpus"] == 1 and b["warmup"] >= 3
    r = b["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] <= 1.0 and r["bound"] in ("tensor", "hbm", "alu")
    assert b["e2e"]["value"] > 0 and b["e2e"]["h2d_bytes_per_step"] > 0 and b["e2e"]["d2h_bytes_per_step"] > 0
    assert b["gpu_launches"] > 0
    assert "sm_mhz" in b["clocks"] and "reasons" in b["clocks"]
