"""FP64 roof calibration + quick per-config timing on one B200 (run through gpurun).

    python tools/probe.py [--sizes 4096,8192,16384] [--out gpurun_out/probe.json]

1. Device facts: SM count, clocks.
2. DMMA.8x8x4 and DFMA throughput probes (gemm_peak_probe): FLOP/clk/SM from the
   kernel's own SM-cycle count, and FLOP/s from CUDA events -- the measured roof
   P(f, o, n) = f * o * n of PAPER.md Eq. (8) P:259-262.
3. Every configuration timed at each size (best and median of reps, CUDA events).
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


def probe(kind, blocks, warps, iters):
    out = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    G.peak_probe(kind, blocks, warps, iters, out, cyc)   # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.peak_probe(kind, blocks, warps, iters, out, cyc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if kind == "dmma":
        flops = blocks * warps * iters * 8 * 512
    else:
        flops = blocks * warps * 32 * iters * 8 * 2
    cycles = int(cyc.item())
    per_block = flops / blocks
    return {"kind": kind, "blocks": blocks, "warps": warps, "iters": iters, "ms": ms,
            "tflops": flops / ms / 1e9, "cycles_block0": cycles,
            "flop_per_clk_per_sm_if_1blk_per_sm": per_block / cycles if blocks <= 148 else None,
            "implied_mhz": cycles / (ms * 1e3)}


def time_cfg(M, N, K, cfg, reps=5):
    A = torch.empty((M, K), dtype=torch.float64, device="cuda")
    B = torch.empty((K, N), dtype=torch.float64, device="cuda")
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    G.fill(A, "uniform", 1706, 0)
    G.fill(B, "uniform", 1706, 1)
    G.fill(C, "uniform", 1706, 2)
    G.gemm(A, B, C, 1.0, 0.0, cfg=cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.gemm(A, B, C, 1.0, 0.0, cfg=cfg)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    fl = 2.0 * M * N * K
    return {"M": M, "N": N, "K": K, "cfg": G.cfg_name(cfg), "best_ms": min(ts), "median_ms": statistics.median(ts),
            "tflops_best": fl / min(ts) / 1e9, "tflops_median": fl / statistics.median(ts) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4096,8192,16384")
    ap.add_argument("--cfgs", default="all")
    ap.add_argument("--out", default="gpurun_out/probe.json")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    p = torch.cuda.get_device_properties(0)
    res = {"device": p.name, "sms": p.multi_processor_count, "probes": [], "gemm": []}
    print(json.dumps({"device": p.name, "sms": p.multi_processor_count}), flush=True)
    for kind in ("dmma", "dfma"):
        for warps in (4, 8, 16):
            r = probe(kind, 148, warps, 20000 if kind == "dmma" else 20000)
            res["probes"].append(r)
            print(json.dumps(r), flush=True)
    r = probe("dmma", 148 * 8, 8, 20000)
    res["probes"].append(r)
    print(json.dumps(r), flush=True)
    cfgs = range(G.num_cfgs()) if a.cfgs == "all" else [int(x) for x in a.cfgs.split(",")]
    for n in [int(x) for x in a.sizes.split(",")]:
        for c in cfgs:
            t0 = time.time()
            r = time_cfg(n, n, n, c, reps=a.reps)
            r["wall_s"] = time.time() - t0
            res["gemm"].append(r)
            print(json.dumps(r), flush=True)
            with open(a.out, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
