"""The CPU oracle timed on this host (run on the GPU box through gpurun, so it is the same
machine the bench's cpu_baseline comes from) -- the table bench.py's cpu_baseline points to.

    python tools/cpu_table.py [--out profiles/r02/cpu_baseline_table.json]

Per SURVEY §8(d) "The oracle timed beside it": the oracle as it stands (oracle/oracle_dgemm.c,
plain i-k-j loop, -O2, no FMA contraction, threads over rows), square N x N x N, alpha = 1,
beta = 0, uniform inputs, at 1 thread and at all threads of the process's CPU affinity; full
runs at N = 256, 1024, 2048, 4096 (best of 3 where a run takes < 10 s, else 1), plus the
16384 row-slab extrapolation bench.py uses.  GFLOP/s = 2 N^3 / t (Eq. (4)).
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def lscpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    except OSError:
        return {}
    keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)", "CPU max MHz",
            "L3 cache", "NUMA node(s)")
    d = {}
    for line in out.splitlines():
        k, _, v = line.partition(":")
        if k.strip() in keep:
            d[k.strip()] = v.strip()
    return d


def time_full(n, threads, reps):
    A = synth.matrix("uniform", 1706, synth.MAT_A, n, n)
    B = synth.matrix("uniform", 1706, synth.MAT_B, n, n)
    C = np.zeros((n, n))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.dgemm(1.0, A, B, 0.0, C, nthreads=threads)
        ts.append(time.perf_counter() - t0)
        if ts[-1] > 10.0:
            break
    return min(ts), len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "cpu_baseline_table.json"))
    ap.add_argument("--sizes", default="256,1024,2048,4096")
    a = ap.parse_args()
    allt = oracle.default_threads()
    res = {"host": {"lscpu": lscpu(), "platform": platform.platform(), "affinity_threads": allt},
           "oracle": "oracle/oracle_dgemm.c (i-k-j, -O2 -ffp-contract=off, threads over rows)",
           "metric": "GFLOP/s = 2 N^3 / t, full N x N x N runs, alpha=1, beta=0, uniform[-1,1) inputs",
           "rows": []}
    for n in (int(x) for x in a.sizes.split(",")):
        for th in (1, allt):
            best, reps = time_full(n, th, 3)
            row = {"n": n, "threads": th, "best_s": best, "runs": reps, "gflops": 2.0 * n ** 3 / best / 1e9}
            print(json.dumps(row), flush=True)
            res["rows"].append(row)
    # the bench's 16384 extrapolation (R rows of the 16384^3 problem, all threads)
    n, R = 16384, 4 * allt
    A = synth.matrix("uniform", 1706, synth.MAT_A, n, n, row0=0, nrows=R)
    B = synth.matrix("uniform", 1706, synth.MAT_B, n, n)
    t0 = time.perf_counter()
    oracle.dgemm(1.0, A, B, 0.0, np.zeros((R, n)), nthreads=allt)
    dt = time.perf_counter() - t0
    res["rows"].append({"n": n, "threads": allt, "sample_rows": R, "sample_s": dt, "extrapolated_full_s": dt * n / R,
                        "gflops": 2.0 * R * n * n / dt / 1e9, "kind": "row slab, extrapolated linearly in M"})
    print(json.dumps(res["rows"][-1]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
