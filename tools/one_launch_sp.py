"""Warm gemm calls of a forced configuration with a forced split-K count (ncu captures):
    python tools/one_launch_sp.py CFG_NAME M N K SPLITS [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

name, M, N, K, S = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
A = torch.empty((M, K), dtype=torch.float64, device="cuda")
B = torch.empty((K, N), dtype=torch.float64, device="cuda")
C = torch.empty((M, N), dtype=torch.float64, device="cuda")
G.fill(A, "uniform", 1, 0)
G.fill(B, "uniform", 1, 1)
for _ in range(reps):
    G.gemm(A, B, C, 1.0, 0.0, cfg=G.cfg_id(name), splits=S)
torch.cuda.synchronize()
print("done", name, M, N, K, S)
