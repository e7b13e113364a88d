"""The driver's contract for bench.py: one JSON line with the required keys, for the reference
arm (the CPU oracle, runnable without a GPU) and for this implementation (on a B200)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


SHARED_CONFIG_KEYS = {"workload", "streams_per_gpu", "n_per_stream", "seed",
                      "bytes_written_per_step_per_gpu", "parallelism", "method_flags",
                      "base_generator", "write_outputs"}


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the same workload keys as this implementation's line (bench.shared_config), plus the sample
    assert d["config"]["workload"].startswith("cfg3: ")
    assert SHARED_CONFIG_KEYS <= set(d["config"]) and "sample" in d["config"]
    assert d["config"]["streams_per_gpu"] == 1 << 20 and d["config"]["n_per_stream"] == 1024


@pytest.mark.gpu
def test_implementation_line():
    d = _run(["--steps", "3", "--warmup", "3", "--workload", "cfg1", "--sustained-s", "0.05",
              "--e2e-steps", "1", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d)
    assert d["metric"].startswith("Gdoubles/s") and d["unit"] == "Gdoubles/s"
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["scaling"] == "weak"
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert roof["bound"] == "hbm" and roof["frac"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["d2h_bytes_per_step"] == 8 * 1024 * 1024
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] == 3
    assert SHARED_CONFIG_KEYS <= set(d["config"]) and d["config"]["workload"].startswith("cfg1: ")
    assert "L2 flush" in d["config"]["l2"] or "flush" in d["config"]["l2"]
