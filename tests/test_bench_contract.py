"""bench.py's JSON-line contract: the keys the driver reads, for the CUDA arm (GPU) and for the
reference arm (the oracle on the host cores; CPU, bounded by HK_REFERENCE_BUDGET_S)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ, **(env_extra or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, cwd=ROOT, env=env, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"],
             {"HK_REFERENCE_BUDGET_S": "1"})
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_cuda_arm_line():
    d = _run(["--steps", "5", "--warmup", "3", "--no-cpu"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 5
    roof = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof
    assert roof["bound"] == "alu" and 0 < roof["frac"] < 1 and 0 < roof["step_frac"] < 1
    assert set(roof["kernels"]) == {"k1_slice_rowntt", "k2_column", "k3_finish"}
    assert d["verification"]["fingerprints_all_rows"] is True
    assert d["cpu_baseline"] is None or d["cpu_baseline"]["gpu_rows_differing"] == 0
    tp = d["throughput"]
    assert tp["value"] > 0 and tp["matvecs"] >= 16
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["config"]["workload"].startswith("C3")
