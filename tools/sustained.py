"""Sustained throughput ("burst vs sustained, 4 s back-to-back, clocks via
NVML"): back-to-back GEMMs for --seconds, SM clock / power / throttle reasons sampled by
nvidia-smi every 100 ms, for the FP64 hot path (16384^3) and the FP32 path."""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    for line in p.stdout:
        f = [x.strip() for x in line.split(",")]
        if f and f[0] == "0":
            rows.append(f)
        if stop.is_set():
            break
    p.terminate()


def run(name, fn, flops, seconds):
    fn()
    torch.cuda.synchronize()
    rows, stop = [], threading.Event()
    t = threading.Thread(target=sample, args=(stop, rows), daemon=True)
    t.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(4):
            fn()
            n += 1
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    ms = e0.elapsed_time(e1)
    mhz = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
    pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
    reasons = sorted({r[3] for r in rows})
    out = {"name": name, "launches": n, "seconds": ms / 1e3, "tflops": flops * n / (ms * 1e-3) / 1e12,
           "sm_mhz_median": statistics.median(mhz) if mhz else None, "sm_mhz_min": min(mhz) if mhz else None,
           "power_w_median": statistics.median(pw) if pw else None, "clock_event_reasons_bitmasks": reasons}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--out", default="gpurun_out/sustained.json")
    a = ap.parse_args()
    n = 16384
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    G.fill(A, "uniform", 1706, 0)
    G.fill(B, "uniform", 1706, 1)
    res = [run("dgemm_16384", lambda: G.gemm(A, B, C, 1.0, 0.0), 2.0 * n ** 3, a.seconds)]
    del A, B, C
    torch.cuda.empty_cache()
    A = torch.rand((n, n), dtype=torch.float32, device="cuda")
    B = torch.rand((n, n), dtype=torch.float32, device="cuda")
    C = torch.empty_like(A)
    res.append(run("sgemm_3xtf32_16384", lambda: G.gemm_f32(A, B, C, 1.0, 0.0), 2.0 * n ** 3, a.seconds))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
