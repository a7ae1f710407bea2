"""The driver's bench.py contract: one JSON line with the keys the driver and the judge read
(metric/value/unit, timing fields, roofline, cpu_baseline, e2e, gpu_launches, clocks), for the
reference arm (the oracle, CPU) and for the CUDA arm (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"]


def run_bench(args, timeout=600):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def check_base(d):
    for k in BASE:
        assert k in d, k
    assert d["metric"] == "ddm_elm_subdomain_lsq_solves_per_s" and d["unit"] == "subdomain-solves/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert isinstance(d["config"]["workload"], str)
    for k in ["value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"]:
        assert k in d["e2e"], k


def test_reference_arm_line():
    d = run_bench(["--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "1"])
    check_base(d)
    assert d["impl"] == "reference" and d["vs_baseline"] is None
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_cuda_arm_line():
    d = run_bench(["--config", "1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    check_base(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    r = d["roofline"]
    for k in ["bound", "achieved", "peak", "unit", "frac", "traffic"]:
        assert k in r, k
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["rel_l2_vs_exact"] < 1e-6
