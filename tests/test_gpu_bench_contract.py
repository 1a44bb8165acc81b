"""bench.py on the GPU: the one JSON line the driver parses (contract keys and their
meaning), from a short run of the real default workload (16384^3, 1 GPU)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_contract(cuda_lib):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout            # exactly one line on stdout
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == base["metric"] and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("dgemm_n16384") and d["scaling"] == "weak"
    flops = 2.0 * 16384 ** 3
    assert abs(d["value"] - flops / (d["ms_per_step"] * 1e-3) / 1e12) < 1e-6 * d["value"]
    r = d["roofline"]
    # peak = the FP64 tensor-pipe roof measured in the same run (DMMA probe); 37.0 is context
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and r["peak_datasheet"] == 37.0
    assert 30.0 < r["peak"] < 40.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0.5 < r["frac"] <= 1.02               # a DMMA kernel can not beat the measured FP64 roof
    # every rank checked its own result after the timed region
    assert d["parity"]["ok"] is True and d["parity"]["b_bitwise"] is True
    assert d["parity"]["rows_checked_total"] >= 2 and d["parity"]["max_ratio"] < 0.05
    assert r["kernel"] == d["impl_detail"]["kernel_cfg"]
    assert d["gpu_launches"] == 3 * r["launches_per_gemm"] >= 3
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
