"""Host logic of bench.py (no GPU): workloads, clock-record parsing, JSON contract keys."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_workloads():
    assert bench.workload("square", 1)[:3] == (16384, 16384, 16384)
    M, N, K, scaling, _ = bench.workload("square", 8)
    assert (M, N, K, scaling) == (16384 * 8, 16384, 16384, "weak")
    assert bench.workload("rect", 4)[:4] == (32768, 4096, 4096, "strong")
    assert bench.workload("large", 8)[:3] == (65536, 65536, 65536)


def test_clock_summary_parsing():
    s = bench.ClockSampler(0)
    s.rows = [["0", "1965", "1965", "700.5", "0x0", "Not Active", "Not Active", "Not Active", "Not Active"],
              ["0", "1900", "1965", "990.0", "0x4", "Not Active", "Not Active", "Not Active", "Active"],
              ["0", "1950", "1965", "800.0", "0x0", "Not Active", "Not Active", "Not Active", "Not Active"]]
    out = s.summary()
    assert out["sm_mhz"] == 1950 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]


def test_metric_matches_baseline_json():
    import json
    b = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert bench.METRIC == b["metric"]
