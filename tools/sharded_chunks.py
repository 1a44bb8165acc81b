"""gemm_f64_sharded at world size 1 (NCCL communicator of one rank): cost of the
column-panel broadcast pipeline (bcast_chunks > 1) against the serial path, 16384^3 -- the
GEMM-side price of overlapping the broadcast on more ranks."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def main():
    n = 16384
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    G.fill(A, "uniform", 1706, 0)
    G.fill(B, "uniform", 1706, 1)
    comm = G.Comm(0, 1)
    out = []
    for chunks in (1, 2, 4, 8):
        comm.gemm_sharded(A, B, C, 1.0, 0.0, bcast_chunks=chunks)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            comm.gemm_sharded(A, B, C, 1.0, 0.0, bcast_chunks=chunks)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        r = {"bcast_chunks": chunks, "ms": best, "tflops": 2 * n ** 3 / best / 1e9}
        print(json.dumps(r), flush=True)
        out.append(r)
    comm.close()
    json.dump(out, open("gpurun_out/sharded_chunks.json", "w"), indent=1)


if __name__ == "__main__":
    main()
