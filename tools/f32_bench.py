"""Timing of the single-precision 3xTF32 path on one B200.

    python tools/f32_bench.py [--sizes 4096,8192,16384] [--out gpurun_out/f32.json]

Reports TFLOP/s (2MNK / t, split pre-pass included) next to the roofs it is bounded by:
TF32 tensor peak / 3 (three MMA passes) and the FP32 SIMT peak (148 SMs x 128 FMA x 2 x f).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4096,8192,16384")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/f32.json")
    ap.add_argument("--cfgs", default="default", help="'default', 'all' or comma list of f32 cfg ids")
    a = ap.parse_args()
    res = []
    cfgs = [None] if a.cfgs == "default" else (list(range(len(G.f32_cfg_names()))) if a.cfgs == "all"
                                                  else [int(x) for x in a.cfgs.split(",")])
    for n, cfg in ((int(x), c) for x in a.sizes.split(",") for c in cfgs):
        A = torch.rand((n, n), dtype=torch.float32, device="cuda") * 2 - 1
        B = torch.rand((n, n), dtype=torch.float32, device="cuda") * 2 - 1
        C = torch.zeros((n, n), dtype=torch.float32, device="cuda")
        t0 = time.time()
        while time.time() - t0 < 0.3:
            G.gemm_f32(A, B, C, 1.0, 0.0, cfg=cfg)
            torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            G.gemm_f32(A, B, C, 1.0, 0.0, cfg=cfg)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        fl = 2.0 * n ** 3
        r = {"n": n, "cfg": G.f32_cfg_names()[cfg] if cfg is not None else "default", "best_s": min(ts), "median_s": statistics.median(ts), "tflops": fl / min(ts) / 1e12,
             "roof_tf32_over_3": 1100.0 / 3, "roof_fp32_simt": 148 * 128 * 2 * 1.965e9 / 1e12}
        print(json.dumps(r), flush=True)
        res.append(r)
        del A, B, C
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
