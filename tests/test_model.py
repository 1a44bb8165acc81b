"""Pins for the performance model (paper_1706_10086_b200/model.py) against PAPER.md's own
numbers: every Tab. 4 K(S,T) entry, the Tab. 2 / SPEC Power8 peaks (Eq. (8)), and closed
forms of Eqs. (2), (3), (6), (7)."""

import json
import os

import pytest

from paper_1706_10086_b200 import model

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tab4_tile_sizes.json")))


def _bytes(txt):
    v, u = txt.split()
    return int(float(v) * {"B": 1, "KB": 1024, "MB": 1024 ** 2}[u])


@pytest.mark.parametrize("row", GOLDEN["rows"], ids=lambda r: "-".join(map(str, r[:3])))
def test_tab4_tile_bytes(row):
    arch, comp, prec, T, kst = row
    S = 4 if prec == "single" else 8
    assert model.tile_bytes(S, T) == _bytes(kst)


@pytest.mark.parametrize("key", ["power8_sp_gflops", "power8_dp_gflops"])
def test_eq8_power8_peak(key):
    f, o, n, expect = GOLDEN["peaks"][key]
    assert model.peak(f * 1e9, o, n) / 1e9 == pytest.approx(expect, rel=1e-12)


def test_closed_forms():
    assert model.flops_eq2(10) == 2300
    assert model.flops(7, 5, 3) == 210
    assert model.blocks(1024, 16, 4) == 16                       # Eq. (3) with t=16, e=4
    assert model.mem_ops(8, 4) == 8 * 8 * (2 * 8 / 4 + 1)        # Eq. (6)
    assert model.ratio(10 ** 9, 64) == pytest.approx(64, rel=1e-6)  # Eq. (7): R -> T
    assert model.ratio(64, 64) == pytest.approx(2 * 64 * 64 / (3 * 64))
    assert model.gflops(1000, 2.0) == pytest.approx(1.0)
    # R = O / M with O = 2N^3 (the identity in Eq. (7))
    n, t = 512, 32
    assert model.ratio(n, t) == pytest.approx(2 * n ** 3 / model.mem_ops(n, t))


def test_b200_mapping():
    assert model.b200_peak() / 1e12 == pytest.approx(37.22496)
    assert model.stage_bytes(128, 128, 16) == 32768
    # square tile T: L2->SM traffic equals Eq. (6) (in 8-byte words, C counted once) when BM=BN=T
    n, t = 4096, 128
    assert model.l2_to_sm_bytes(n, n, n, t, t) / 8 == pytest.approx(model.mem_ops(n, t))
    assert model.tile_intensity(128, 128) == pytest.approx(128 * 128 * 2 / (8 * 256))   # = 16
    assert model.compulsory_bytes(16384, 16384, 16384) == 3 * 8 * 16384 ** 2


def test_report_rows_cover_every_cfg():
    from paper_1706_10086_b200 import build
    build.build()
    from paper_1706_10086_b200 import gemm as G
    rows = model.report(8192)
    assert [r["cfg"] for r in rows] == [c["name"] for c in G.cfgs()]
    for r in rows:
        assert r["stage_bytes"] * 2 <= r["smem_bytes"]
