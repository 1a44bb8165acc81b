"""Host logic of the auto-tuner (§2.3), no GPU."""

import pytest


@pytest.fixture(scope="module")
def T():
    from paper_1706_10086_b200 import build
    build.build()
    from paper_1706_10086_b200 import tuner
    return tuner


def test_select_argmax_with_deterministic_tie_break(T):
    res = {(5, 1): 1.0000, (3, 1): 1.0005, (7, 2): 0.9996, (2, 4): 1.2}
    # 0.9996 is best; 1.0000 and 1.0005 are within 0.1 % -> tie -> smallest (cfg, splits)
    assert T.select(res) == (3, 1)
    assert T.select(res, tol=0.0) == (7, 2)
    assert T.select({(9, 1): 2.0}) == (9, 1)
    with pytest.raises(ValueError):
        T.select({})


def test_candidates_cover_tma_cfgs_and_split_counts(T):
    from paper_1706_10086_b200 import gemm as G
    c = T.candidates(1024, 1024, 1024)
    ids = {cid for cid, _ in c}
    assert {i["id"] for i in G.cfgs() if i["tma"]} == ids
    assert any(s > 1 for _, s in c)
    assert all(s == 1 for cid, s in c if G.cfg_info(cid)["split_k"] not in (0, -3))
    assert all(s <= 8 for cid, s in c if G.cfg_info(cid)["split_k"] == -3)   # cluster split-K: portable size
    assert any(s > 1 for cid, s in c if G.cfg_info(cid)["split_k"] == -3)
    assert all(not G.cfg_info(i)["tma"] for i, _ in T.candidates(64, 64, 64, tma=False))


def test_table_round_trip_pins_the_plan(T, tmp_path):
    from paper_1706_10086_b200 import gemm as G
    G.plan_clear()
    cfg = G.cfg_id("tma_64x64x16_w32x16_s6_splitk")
    path = str(tmp_path / "tuned.txt")
    T.write_table(path, [(777, 555, 333, True, cfg, 3), (10240, 10240, 10240, True, G.cfg_id("tma_128x128x16_w32x32_s4"), 1)])
    assert G.tune_load(path) == 2
    assert G.plan(777, 555, 333, 0, 334, 0, 556) == (cfg, 3)        # 16-B aligned, even lds: TMA-eligible
    assert G.plan(10240, 10240, 10240, 0, 10240, 0, 10240)[0] == G.cfg_id("tma_128x128x16_w32x32_s4")
    G.plan_clear()


def test_table_errors(T, tmp_path):
    from paper_1706_10086_b200 import gemm as G
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2 3 1 no_such_cfg 1\n")
    with pytest.raises(G.GemmError, match="unknown configuration"):
        G.tune_load(str(bad))
    bad.write_text("1 2 three\n")
    with pytest.raises(G.GemmError, match="expected"):
        G.tune_load(str(bad))
    with pytest.raises(G.GemmError):
        G.plan_set(4, 4, 4, True, G.cfg_id("tma_128x128x16_w32x32_s4"), 2)   # no split-K on this cfg
    with pytest.raises(G.GemmError):
        G.plan_set(4, 4, 4, False, G.cfg_id("tma_128x128x16_w32x32_s4"), 1)  # TMA cfg for a non-TMA shape


def test_tune_save_round_trip(T, tmp_path):
    """gemm_tune_save writes every pinned plan in gemm_tune_load's format: the shipped table
    saved and re-read pins the same (M, N, K, tma) -> (cfg, splits) map."""
    from paper_1706_10086_b200 import gemm as G

    def parse(path):
        out = {}
        for line in open(path):
            if line.startswith("#") or not line.strip():
                continue
            M, N, K, tma, name, sp = line.split()
            out[(int(M), int(N), int(K), int(tma))] = (name, int(sp))
        return out

    G.plan_clear()
    n = G.tune_load(G.TUNED_TABLE)
    path = str(tmp_path / "saved.txt")
    assert G.tune_save(path) == n == len(parse(G.TUNED_TABLE))
    assert parse(path) == parse(G.TUNED_TABLE)
    G.plan_clear()
    assert G.tune_save(path) == 0 and parse(path) == {}
    G.plan_set(777, 555, 333, True, G.cfg_id("tma_64x64x16_w32x16_s6_splitk"), 3)
    assert G.tune_save(path) == 1
    G.plan_clear()
    assert G.tune_load(path) == 1
    assert G.plan(777, 555, 333, 0, 334, 0, 556) == (G.cfg_id("tma_64x64x16_w32x16_s6_splitk"), 3)
    with pytest.raises(G.GemmError, match="cannot write"):
        G.tune_save(str(tmp_path / "no_such_dir" / "t.txt"))
    G.plan_clear()
    G.tune_load(G.TUNED_TABLE)
