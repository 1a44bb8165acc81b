"""Time the one-tile-per-CTA XP kernel against the persistent hybrid (data-parallel waves +
stream-K tail) and the heuristic's own plan on config-2/4-like shapes (timing only; parity is
in tests/test_gpu_parity.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    shapes = [(n, n, n) for n in (1024, 2048, 3072, 4096, 6144, 7168, 8192, 9216, 12288, 16384)]
    shapes += [(16384, 4096, 4096), (8192, 4096, 4096), (4096, 4096, 4096)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")]
    xp = G.cfg_id("tma_256x64x16_w64x32_s4_xp")
    hy = G.cfg_id("tma_256x64x16_w64x32_s4_hybrid")
    out = []
    for (M, N, K) in shapes:
        A = torch.empty((M, K), dtype=torch.float64, device="cuda")
        B = torch.empty((K, N), dtype=torch.float64, device="cuda")
        C = torch.empty((M, N), dtype=torch.float64, device="cuda")
        G.fill(A, "uniform", 1, 0)
        G.fill(B, "uniform", 1, 1)
        reps = max(3, min(50, int(2e12 / (2 * M * N * K))))
        fl = 2.0 * M * N * K
        r = {"shape": [M, N, K]}
        for name, cfg in (("xp", xp), ("hybrid", hy), ("plan", None)):
            ms = timeit(lambda: G.gemm(A, B, C, 1.0, 0.0, cfg=cfg), reps)
            r[name] = fl / ms / 1e9
        pc, ps = G.plan(M, N, K, A.data_ptr(), K, B.data_ptr(), N)
        r["plan_cfg"] = G.cfg_name(pc) + (f" x{ps}" if ps > 1 else "")
        print(json.dumps(r), flush=True)
        out.append(r)
        del A, B, C
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/hybrid_probe.json", "w"), indent=1)


if __name__ == "__main__":
    main()
