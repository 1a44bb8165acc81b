"""How good is the size heuristic on shapes it was not tuned on?  For seeded random shapes
(and a few skinny ones) time the product's own plan and every tuner candidate (batched
back-to-back timing, paper_1706_10086_b200.tuner), and report the plan's regret
t_plan / t_best - 1, and
with --autotune also the plan gemm_plan_autotune pins (timed the same way) and its regret.  Shapes in the tuned table are skipped (they are pinned).

    python tools/heuristic_regret.py [--n 16] [--seed 7] [--out gpurun_out/regret.csv]
"""
import argparse
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402
from paper_1706_10086_b200 import tuner  # noqa: E402


def shapes(n, seed, lo=500, hi=6000):
    rng = np.random.default_rng(seed)
    out = [tuple(int(x) for x in rng.integers(lo, hi + 1, 3)) for _ in range(n)]
    if (lo, hi) == (500, 6000):
        out += [(256, 8192, 8192), (8192, 256, 8192), (4096, 4096, 512), (640, 640, 40000), (12000, 12000, 1000)]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default="gpurun_out/regret.csv")
    ap.add_argument("--lo", type=int, default=500, help="shape range (small shapes: --lo 200 --hi 1600)")
    ap.add_argument("--hi", type=int, default=6000)
    ap.add_argument("--autotune", type=int, default=0, help="also run gemm_plan_autotune with this top (0: off)")
    ap.add_argument("--dump", default=None, help="JSONL of every candidate's seconds per shape (model fitting)")
    a = ap.parse_args()
    with open(a.out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["m", "n", "k", "plan", "plan_splits", "plan_tflops", "best", "best_splits", "best_tflops", "regret"]
                   + (["auto", "auto_splits", "auto_tflops", "auto_regret", "autotune_s"] if a.autotune else []))
        for (M, N, K) in shapes(a.n, a.seed, a.lo, a.hi):
            Ke, Ne = K + (K & 1), N + (N & 1)        # even leading dimensions: the TMA path
            A = torch.empty((M, Ke), dtype=torch.float64, device="cuda")[:, :K]
            B = torch.empty((K, Ne), dtype=torch.float64, device="cuda")[:, :N]
            C = torch.empty((M, Ne), dtype=torch.float64, device="cuda")[:, :N]
            for X, m in ((A, 0), (B, 1), (C, 2)):
                G.fill(X, "uniform", 1, m)
            cid, sp = G.plan(M, N, K, A.data_ptr(), Ke, B.data_ptr(), Ne)
            fl = 2.0 * M * N * K
            t_plan, _ = tuner._time(lambda: G.gemm(A, B, C, 1.0, 0.0), 5)
            best = (None, None, float("inf"))
            times = {}
            for cfg, s in tuner.candidates(M, N, K):
                t, _ = tuner._time(lambda: G.gemm(A, B, C, 1.0, 0.0, cfg=cfg, splits=s), 3, warm_s=0.05)
                times[f"{G.cfg_name(cfg)}:{s}"] = t
                if t < best[2]:
                    best = (cfg, s, t)
            if a.dump:
                import json
                with open(a.dump, "a") as df:
                    df.write(json.dumps({"shape": [M, N, K], "plan": f"{G.cfg_name(cid)}:{sp}", "plan_s": t_plan,
                                         "times": times}) + "\n")
            r = [M, N, K, G.cfg_name(cid), sp, f"{fl / t_plan / 1e12:.3f}", G.cfg_name(best[0]), best[1],
                 f"{fl / best[2] / 1e12:.3f}", f"{t_plan / best[2] - 1.0:.4f}"]
            if a.autotune:
                torch.cuda.synchronize()
                import time
                w0 = time.perf_counter()
                acid, asp, _ = G.autotune(A, B, top=a.autotune)
                wall = time.perf_counter() - w0
                t_auto, _ = tuner._time(lambda: G.gemm(A, B, C, 1.0, 0.0), 5)
                r += [G.cfg_name(acid), asp, f"{fl / t_auto / 1e12:.3f}", f"{t_auto / best[2] - 1.0:.4f}", f"{wall:.3f}"]
            w.writerow(r)
            f.flush()
            print(",".join(map(str, r)), flush=True)
            del A, B, C
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
    if "--dump" in sys.argv:   # per-configuration registers / smem / threads after use (occupancy)
        import json
        p = sys.argv[sys.argv.index("--dump") + 1]
        with open(p, "a") as df:
            df.write(json.dumps({"cfgs": [G.cfg_info(i) | {"name": G.cfg_name(i)} for i in range(G.num_cfgs())]}) + "\n")
