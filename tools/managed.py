"""Unified (managed) memory vs explicit device memory (PAPER.md P:216, P:892:
"all GPUs show a better performance when using unified memory").

    python tools/managed.py [--sizes 1024,2048,4096,8192,16384] [--out gpurun_out/managed.json]

For each size, the same seeded DGEMM (alpha=1, beta=0) runs on
  device   : cudaMalloc buffers (torch), inputs generated on the GPU
  managed  : cudaMallocManaged buffers, inputs generated on the GPU (first touch on device)
  host-init: cudaMallocManaged buffers written by the CPU first, no prefetch (pages migrate on
             demand during the first launch)
  prefetch : like host-init, then cudaMemPrefetchAsync to the GPU before the launch
and reports the first launch (one call between two events, right after the inputs were
written) and the steady state: device time per call of back-to-back calls (the tuner's
batched timing, so the ~10 us host cost per call overlaps the kernels at small N; best of
reps).  The managed results are checked bitwise against the device result (same plan, same
per-entry arithmetic); tests/test_gpu_managed.py checks them against the CPU oracle.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def _ok(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"CUDA runtime error {err}")
    return res[1] if isinstance(res, tuple) and len(res) > 1 else None


def managed(nbytes):
    return int(_ok(rt.cudaMallocManaged(nbytes, rt.cudaMemAttachGlobal)))


def fill_raw(ptr, rows, cols, mat, seed=1706):
    rc = G.lib().gemm_fill_f64(0, seed, mat, rows, cols, 0, rows, ptr, cols, 0)
    if rc:
        raise RuntimeError(G.last_error())


def host_fill(ptr, rows, cols, mat, seed=1706):
    """CPU writes into managed memory (values from a device-generated scratch copy)."""
    tmp = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    G.fill(tmp, "uniform", seed, mat)
    host = tmp.cpu().numpy()
    del tmp
    buf = (np.ctypeslib.as_array((ctypes_c_double * (rows * cols)).from_address(ptr)))
    buf[:] = host.reshape(-1)


import ctypes  # noqa: E402
ctypes_c_double = ctypes.c_double


def gemm_raw(n, pa, pb, pc):
    rc = G.gemm_raw(n, n, n, 1.0, pa, n, pb, n, 0.0, pc, n, -1, 0)
    if rc:
        raise RuntimeError(G.last_error())


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def steady(fn, reps):
    from paper_1706_10086_b200 import tuner
    return tuner._time(fn, reps)[0]


def run(n, reps):
    fl = 2.0 * n ** 3
    nbytes = 8 * n * n
    out = {"n": n}
    # device
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    G.fill(A, "uniform", 1706, 0)
    G.fill(B, "uniform", 1706, 1)
    first = timed(lambda: gemm_raw(n, A.data_ptr(), B.data_ptr(), C.data_ptr()))
    best = steady(lambda: gemm_raw(n, A.data_ptr(), B.data_ptr(), C.data_ptr()), reps)
    out["device"] = {"first_tflops": fl / first / 1e12, "tflops": fl / best / 1e12}
    ref = C.cpu().numpy()
    del A, B, C
    torch.cuda.empty_cache()
    dev = torch.cuda.current_device()
    for mode in ("managed", "host-init", "prefetch"):
        pa, pb, pc = managed(nbytes), managed(nbytes), managed(nbytes)
        if mode == "managed":
            fill_raw(pa, n, n, 0)
            fill_raw(pb, n, n, 1)
            torch.cuda.synchronize()
        else:
            host_fill(pa, n, n, 0)
            host_fill(pb, n, n, 1)
            if mode == "prefetch":
                for p in (pa, pb, pc):
                    _ok(rt.cudaMemPrefetchAsync(p, nbytes, dev, 0))
        t0 = time.perf_counter()
        first = timed(lambda: gemm_raw(n, pa, pb, pc))
        wall_first = time.perf_counter() - t0
        best = steady(lambda: gemm_raw(n, pa, pb, pc), reps)
        got = np.ctypeslib.as_array((ctypes_c_double * (n * n)).from_address(pc)).reshape(n, n).copy()
        out[mode] = {"first_tflops": fl / first / 1e12, "first_wall_s": wall_first, "tflops": fl / best / 1e12,
                     "bitwise_equal_to_device": bool(np.array_equal(got, ref))}
        for p in (pa, pb, pc):
            _ok(rt.cudaFree(p))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096,8192,16384")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--out", default="gpurun_out/managed.json")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    res = []
    for n in (int(x) for x in a.sizes.split(",")):
        r = run(n, a.reps)
        print(json.dumps(r), flush=True)
        res.append(r)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
