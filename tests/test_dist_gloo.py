"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic.

The GPU box used in this round has one GPU, so the sharded path's host-side
pieces are exercised here: NCCL unique-id creation on rank 0 and its
distribution to every rank, the row-block partition (every row of C owned by
exactly one rank), the max-over-ranks timing reduction bench.py uses, and a
row-sharded GEMM computed by the CPU oracle on each rank's rows that, gathered,
equals the unsharded oracle bitwise (the per-entry arithmetic does not depend
on the partition).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_1706_10086_b200 import gemm as G

        raw = G.share_unique_id(rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, raw)

        M, N, K = 37, 23, 19
        r0, r1 = G.row_range(M, rank, world)
        A, B, C0 = synth.problem(M, N, K, seed=21)
        local = oracle.dgemm(1.5, A[r0:r1], B, 0.5, C0[r0:r1], nthreads=1)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, local))

        t = G.max_over_ranks([10.0 + rank, 5.0 - rank], world)
        q.put((rank, ids, parts, t))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e), None))


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort(key=lambda x: x[0])
    for r in res:
        assert r[1] != "error", r
    ids = res[0][1]
    assert all(len(x) == 128 for x in ids) and len(set(ids)) == 1, "ranks got different NCCL ids"
    for r in res:
        assert r[1] == ids
    parts = sorted(res[0][2], key=lambda p: p[0])
    rows = np.vstack([p[2] for p in parts])
    assert parts[0][0] == 0 and parts[-1][1] == 37
    import oracle
    import synth
    A, B, C0 = synth.problem(37, 23, 19, seed=21)
    assert np.array_equal(rows, oracle.dgemm(1.5, A, B, 0.5, C0))
    for r in res:
        assert r[3] == [11.0, 5.0]


def _bench_parity_worker(rank, world, port, q):
    """bench.py's post-timing parity logic on each rank (host side): sampled local rows checked
    against the oracle, then the max/sum reduction over ranks.  Rank 1 corrupts one entry in
    the second scenario: every rank must then report ok = False."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        import oracle
        import synth
        M, N, K = 64, 48, 40
        r0, r1 = (rank * M) // world, ((rank + 1) * M) // world
        rows = bench.sample_rows(r1 - r0, 4, 1706 + rank)
        A = synth.matrix("uniform", 1706, synth.MAT_A, M, K)
        B = synth.matrix("uniform", 1706, synth.MAT_B, K, N)
        full = oracle.dgemm(1.0, A, B, 0.0, np.zeros((M, N)))
        col0, nc = 16, 24
        got = full[[r0 + i for i in rows], col0:col0 + nc]
        out = []
        for corrupt in (False, True):
            g = got.copy()
            if corrupt and rank == 1:
                g[-1, 3] += 1e-9
            ok, ratio = bench.check_rows(g, M, N, K, r0, rows, 1706, col0, nc)
            out.append((ok, bench.reduce_parity(ok, ratio, True, len(rows), world)))
        q.put((rank, rows, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))


def test_gloo_world2_bench_parity_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_parity_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    for rank, rows, out in res:
        assert rows[0] == 0 and rows[-1] == 31            # first and last local row always checked
        (ok0, red0), (ok1, red1) = out
        assert ok0 and red0["ok"] and red0["rows_checked_total"] == len(res[0][1]) + len(res[1][1])
        assert red0["max_ratio"] < 0.05
        assert red1["ok"] is False                          # rank 1's bad entry fails every rank
        assert ok1 == (rank == 0)
        assert red1["max_ratio"] > 1.0
