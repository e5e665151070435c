"""bench.py's JSON contract on a small workload (config A, 20k x 64): the keys
the driver reads, for both arms."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_line_keys():
    d = _line("--config", "A", "--steps", "4", "--warmup", "3", "--replay-epochs", "1")
    for key in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]:
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    r = d["roofline"]
    for key in ["bound", "achieved", "peak", "unit", "frac", "traffic"]:
        assert key in r, key
    cb = d["cpu_baseline"]
    for key in ["value", "unit", "cores", "kind", "sample"]:
        assert key in cb, key
    e = d["e2e"]
    for key in ["value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"]:
        assert key in e, key
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    for key in ["sm_mhz", "sm_max_mhz", "reasons"]:
        assert key in d["clocks"], key


def test_reference_arm_line_keys():
    d = _line("--impl", "reference", "--config", "A", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "edge-updates/s"
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
