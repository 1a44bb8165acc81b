"""Small shapes through every configuration, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) runs on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

SHAPES = [(130, 66, 40), (64, 64, 16), (1, 1, 1), (257, 129, 33), (96, 200, 100)]


def main():
    n = 0
    for (M, N, K) in SHAPES:
        Kp, Np = K + (K & 1), N + (N & 1)       # even leading dimensions so TMA configs run
        A = torch.empty((M, Kp), dtype=torch.float64, device="cuda")[:, :K]
        B = torch.empty((K, Np), dtype=torch.float64, device="cuda")[:, :N]
        C = torch.empty((M, Np), dtype=torch.float64, device="cuda")[:, :N]
        G.fill(A, "uniform", 1, 0)
        G.fill(B, "uniform", 1, 1)
        G.fill(C, "uniform", 1, 2)
        for info in G.cfgs():
            G.gemm(A, B, C, 1.5, 0.5, cfg=info["id"])
            n += 1
        G.gemm(A, B, C, 0.0, 0.5)            # scale path
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {n} launches")


if __name__ == "__main__":
    main()
