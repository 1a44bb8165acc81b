"""gemm_f64_sharded with 2 ranks on 2 GPUs (NCCL), one process per GPU -- runs only where the
box has >= 2 GPUs (the round-end driver and gpurun give 1 GPU; the 8-GPU scaling bench
self-checks instead, bench.py "parity").  Rank r owns rows [floor(rM/P), floor((r+1)M/P)) of
an UNEVEN M; B is broadcast from rank 0 (rank 1 starts from zeros).  Each rank's C rows must
equal, bitwise, the single-GPU one-k-pass call on the same rows (no split-K: the per-entry
chain does not depend on the partition), for one broadcast and for 3 column panels, and
rank 1's B must equal rank 0's bitwise after the call."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from paper_1706_10086_b200 import gemm as G
        M, N, K = 1001, 776, 520
        A, B, C0 = synth.problem(M, N, K, seed=33)
        r0, r1 = G.row_range(M, rank, world)
        comm = G.Comm(rank, world)
        res = []
        for chunks in (1, 3):
            dA = torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda()
            dC = torch.from_numpy(np.ascontiguousarray(C0[r0:r1])).cuda()
            dB = torch.from_numpy(B).cuda() if rank == 0 else torch.zeros((K, N), dtype=torch.float64, device="cuda")
            comm.gemm_sharded(dA, dB, dC, 1.5, 0.5, root=0, bcast_chunks=chunks)
            torch.cuda.synchronize()
            ref = torch.from_numpy(np.ascontiguousarray(C0[r0:r1])).cuda()
            G.gemm(dA, torch.from_numpy(B).cuda(), ref, 1.5, 0.5, splits=1)
            torch.cuda.synchronize()
            res.append((chunks, bool(torch.equal(dC, ref)), bool(np.array_equal(dB.cpu().numpy(), B))))
        comm.close()
        q.put((rank, res))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error: " + repr(e)))


def test_sharded_two_gpus_bitwise_equals_single_gpu_rows(cuda_lib):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (this box has %d)" % torch.cuda.device_count())
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for rank, r in res:
        assert not isinstance(r, str), r
        for chunks, c_ok, b_ok in r:
            assert c_ok, f"rank {rank} chunks {chunks}: C rows differ from the single-GPU call"
            assert b_ok, f"rank {rank} chunks {chunks}: broadcast B differs from rank 0's"
