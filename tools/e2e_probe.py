"""Facts behind the end-to-end (host-buffer) schedule: PCIe bandwidths for the copy shapes
gemm_f64_host uses, and the GEMM time of each block shape."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def ev_time(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def main():
    n = 16384
    out = {}
    h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    d = torch.empty((n, n), dtype=torch.float64, device="cuda")
    t = ev_time(lambda: d.copy_(h, non_blocking=True))
    out["h2d_contig_GBs"] = 8 * n * n / t / 1e9
    t = ev_time(lambda: h.copy_(d, non_blocking=True))
    out["d2h_contig_GBs"] = 8 * n * n / t / 1e9
    t = ev_time(lambda: d[:, :2048].copy_(h[:, :2048], non_blocking=True))
    out["h2d_colblock2048_GBs"] = 8 * n * 2048 / t / 1e9
    from cuda.bindings import runtime as rt
    st0 = torch.cuda.current_stream().cuda_stream
    for w in (512, 2048, 4096):
        def c2d(w=w):
            rt.cudaMemcpy2DAsync(d.data_ptr(), n * 8, h.data_ptr(), n * 8, w * 8, n,
                                 rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st0)
        t = ev_time(c2d)
        out[f"h2d_memcpy2d_colblock{w}_GBs"] = 8 * n * w / t / 1e9
    s2 = torch.cuda.Stream()

    def both():
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
        with torch.cuda.stream(s2):
            h[n // 2:].copy_(d[n // 2:], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)
    t = ev_time(both)
    out["h2d_plus_d2h_concurrent_GBs_total"] = 8 * n * n / t / 1e9
    del h
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    G.fill(A, "uniform", 1, 0)
    G.fill(d, "uniform", 1, 1)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for (m, nn) in ((2304, 2048), (2560, 2048), (2048, n), (2048, 4096), (16384, n)):
        t = ev_time(lambda: G.gemm(A[:m], d[:, :nn], C[:m, :nn], 1.0, 0.0, splits=1))
        cid, sp = G.plan(m, nn, n, A.data_ptr(), n, d.data_ptr(), n)
        out[f"gemm_{m}x{nn}x{n}"] = {"ms": t * 1e3, "tflops": 2 * m * nn * n / t / 1e12, "plan": G.cfg_name(cid)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
