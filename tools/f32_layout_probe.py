"""Exactness probe of every single-precision configuration on small-integer inputs (tf32-exact,
sums < 2^24): any layout / descriptor error shows up as a mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

for cfg, name in enumerate(G.f32_cfg_names()):
    for (M, N, K) in ((256, 256, 64), (512, 512, 256), (300, 200, 100), (4096, 4096, 4096)):
        A = torch.randint(-8, 9, (M, K), device="cuda").float()
        B = torch.randint(-8, 9, (K, N), device="cuda").float()
        C = torch.zeros((M, N), device="cuda")
        G.gemm_f32(A, B, C, 1.0, 0.0, cfg=cfg)
        torch.cuda.synchronize()
        ref = (A.double() @ B.double()).float()
        print(name, M, N, K, "exact" if torch.equal(C, ref) else "MISMATCH", flush=True)
