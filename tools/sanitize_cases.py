"""Small shapes through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) runs on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
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
            for s in ((1,) if info["split_k"] not in (0, -3) else (1, 3)):   # split-K, persistent, cluster
                G.gemm(A, B, C, 1.5, 0.5, cfg=info["id"], splits=s)
                n += 1
        G.gemm(A, B, C, 0.0, 0.5)            # scale path
        a32, b32 = A.float(), B.float()
        c32 = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        G.gemm_f32(a32, b32, c32, 1.5, 0.5)  # 3xTF32 tcgen05 path
        n += 2
    # hybrid schedule with a full wave, a cut stream-K tail and the fix-up kernel
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    M, N, K = 1000, 64 * (sms // 4 + 3), 1000
    A = torch.rand((M, K), dtype=torch.float64, device="cuda")
    B = torch.rand((K, N), dtype=torch.float64, device="cuda")
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    assert G.launches_per_call(G.cfg_id("tma_256x64x16_w64x32_s4_hybrid"), M, N, K, sms) == 3
    for info in G.cfgs():                    # every hybrid configuration (32x64: 2-quad fix-up CTAs)
        if info["split_k"] == -2:
            G.gemm(A, B, C, 1.0, 0.0, cfg=info["id"])
            n += 1
    # repack path: large problem with odd leading dimensions
    M, N, K = 1200, 1201, 1501
    A = torch.rand((M, K), dtype=torch.float64, device="cuda")
    B = torch.rand((K, N), dtype=torch.float64, device="cuda")
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    G.gemm(A, B, C, 1.0, 0.0)
    # host entry point
    hA, hB = np.random.rand(300, 200), np.random.rand(200, 100)
    hC = np.zeros((300, 100))
    G.gemm_host(hA, hB, hC, 1.0, 0.0)
    # run-time tuning: candidates into the library's scratch C, then the pinned plan
    M, N, K = 222, 350, 410
    A = torch.rand((M, K), dtype=torch.float64, device="cuda")
    B = torch.rand((K, N), dtype=torch.float64, device="cuda")
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    G.autotune(A, B, top=4)
    G.gemm(A, B, C, 1.0, 0.0)
    n += 1
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {n + 2} calls (+ one autotune)")


if __name__ == "__main__":
    main()
