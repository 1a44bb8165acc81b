import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_1706_10086_b200 import gemm as G
for cfg in sys.argv[1].split(","):
    for n in [int(x) for x in sys.argv[2].split(",")]:
        A = torch.empty((n, n), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
        G.fill(A, "dyadic", 1, 0); G.fill(B, "dyadic", 1, 1)
        G.gemm(A, B, C, 1.0, 0.0, cfg=G.cfg_id(cfg)); torch.cuda.synchronize()
        R = torch.empty_like(C); G.gemm(A, B, R, 1.0, 0.0); torch.cuda.synchronize()
        print(cfg, n, "equal to plan:", torch.equal(C, R), flush=True)
