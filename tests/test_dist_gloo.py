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
