"""Can two ranks share one GPU for NCCL (to run the sharded path with world 2 on a 1-GPU box)?
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_same_gpu_probe.py
Both ranks use cuda:0; tries the library's own communicator (gemm_comm_init) and, if that
works, one gemm_f64_sharded call checked bitwise against the single-GPU rows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
from paper_1706_10086_b200 import gemm as G  # noqa: E402
import synth  # noqa: E402
try:
    comm = G.Comm(rank, world)
    print(f"[rank {rank}] comm ok: {comm.info()}", flush=True)
except Exception as ex:
    print(f"[rank {rank}] comm FAILED: {type(ex).__name__}: {ex}", flush=True)
    sys.exit(0)
M, N, K = 1001, 776, 520
A, B, C0 = synth.problem(M, N, K, seed=33)
r0, r1 = G.row_range(M, rank, world)
for chunks in (1, 3):
    dA = torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda()
    dC = torch.from_numpy(np.ascontiguousarray(C0[r0:r1])).cuda()
    dB = torch.from_numpy(B).cuda() if rank == 0 else torch.zeros((K, N), dtype=torch.float64, device="cuda")
    comm.gemm_sharded(dA, dB, dC, 1.5, 0.5, root=0, bcast_chunks=chunks)
    torch.cuda.synchronize()
    ref = torch.from_numpy(np.ascontiguousarray(C0[r0:r1])).cuda()
    G.gemm(dA, torch.from_numpy(B).cuda(), ref, 1.5, 0.5, splits=1)
    torch.cuda.synchronize()
    print(f"[rank {rank}] chunks={chunks} rows [{r0},{r1}) C bitwise={bool(torch.equal(dC, ref))} "
          f"B bitwise={bool(np.array_equal(dB.cpu().numpy(), B))}", flush=True)
comm.close()
dist.destroy_process_group()
