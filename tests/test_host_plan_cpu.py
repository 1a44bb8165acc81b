"""gemm_f64_host's block schedule (csrc/host_api.cu host_geometry / plan_geometry), host-only
arithmetic queried through gemm_host_plan -- no GPU.  The library's copy/compute simulation is
pinned against the independent Python model in tools/e2e_sim.py (same calibration, written
separately), and the geometries the measurements in DESIGN.md §e2e rest on are pinned."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_1706_10086_b200 import build
    build.build()
    from paper_1706_10086_b200 import gemm
    return gemm


@pytest.fixture(scope="module")
def sim():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import e2e_sim
    e2e_sim.gemm_t = e2e_sim.gemm_t64     # the round-2 wave model (tools/e2e_sim.py --r02)
    return e2e_sim


def _py_time(sim, M, N, K, g):
    return sim.simulate(K, sim.schedule(M, N, K, g["R0"], g["Ra"], g["cb0"], g["cb"], g["Rp"], g["Rlast"],
                                        g["nlast"]))[0]


def test_headline_shape_keeps_the_rule_geometry(G, sim):
    g, t = G.host_plan(16384, 16384, 16384, num_sms=148)
    assert g == dict(R0=3072, Ra=768, cb0=1024, cb=1536, Rp=3840, Rlast=256, nlast=2)
    assert t == pytest.approx(0.25109, rel=2e-4)                       # measured 250.8-252.0 ms
    assert t == pytest.approx(_py_time(sim, 16384, 16384, 16384, g), rel=1e-12)


def test_config4_takes_the_searched_geometry(G, sim):
    g, t = G.host_plan(32768, 4096, 4096, num_sms=148)
    assert g == dict(R0=3072, Ra=768, cb0=1024, cb=1024, Rp=2048, Rlast=128, nlast=1)
    rule = dict(R0=3072, Ra=768, cb0=1024, cb=1536, Rp=5888, Rlast=256, nlast=2)
    t_rule = _py_time(sim, 32768, 4096, 4096, rule)
    assert t_rule == pytest.approx(0.03867, rel=1e-3)                  # measured 38.5 ms (28.6 TFLOP/s)
    assert t < 0.99 * t_rule and t == pytest.approx(0.03398, rel=1e-3)   # measured 34.2 ms (32.1 TFLOP/s)
    assert t == pytest.approx(_py_time(sim, 32768, 4096, 4096, g), rel=1e-12)


@pytest.mark.parametrize("shape", [(8192, 4096, 4096), (10000, 9999, 7001), (4096, 16384, 16384),
                                   (6003, 1001, 2002), (20000, 3000, 5000)])
def test_library_simulation_equals_python_model(G, sim, shape):
    g, t = G.host_plan(*shape, num_sms=148)
    assert t == pytest.approx(_py_time(sim, *shape, g), rel=1e-12)
    assert 0 < g["Ra"] <= g["R0"] <= shape[0] and 0 < g["cb0"] <= shape[1] and g["nlast"] in (1, 2)


def test_tiny_problems_run_in_one_shot(G):
    g, _ = G.host_plan(300, 200, 100, num_sms=148)
    assert g == dict(R0=300, Ra=300, cb0=200, cb=200, Rp=300, Rlast=0, nlast=1)
    g, _ = G.host_plan(0, 5, 5, num_sms=148)
    assert g["R0"] == 0


def test_host_plan_errors(G):
    with pytest.raises(G.GemmError):
        G.host_plan(-1, 4, 4, num_sms=148)
    assert G.lib().gemm_host_plan(4, 4, 4, 0, 148, None, None) == G.GEMM_ERR_ARG
