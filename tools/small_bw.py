"""Small, latency/occupancy-bound sizes (N <= 2048): one launch per size of the product's
plan, for an ncu --metrics pass that reports achieved L2 and HBM bandwidth (north star:
"plus L2/HBM GB/s for the small, memory-bound sizes").

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
        --clock-control none -k regex:dgemm --csv --log-file gpurun_out/small_bw.csv python tools/small_bw.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

SIZES = (256, 512, 768, 1024, 1536, 2048)


def main():
    for n in SIZES:
        A = torch.empty((n, n), dtype=torch.float64, device="cuda")
        B = torch.empty_like(A)
        C = torch.empty_like(A)
        G.fill(A, "uniform", 1706, 0)
        G.fill(B, "uniform", 1706, 1)
        for _ in range(3):   # the last launch of each size is the one reported
            G.gemm(A, B, C, 1.0, 0.0)
        torch.cuda.synchronize()
        cid, sp = G.plan(n, n, n, A.data_ptr(), n, B.data_ptr(), n)
        print(n, G.cfg_name(cid), sp, flush=True)


if __name__ == "__main__":
    main()
