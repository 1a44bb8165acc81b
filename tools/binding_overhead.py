"""Host cost per call of the Python binding vs the bare C-ABI call (small GEMMs are host-bound)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

n = 256
A = torch.rand((n, n), dtype=torch.float64, device="cuda")
B = torch.rand((n, n), dtype=torch.float64, device="cuda")
C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
args = (n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, st)
for _ in range(200):
    G.gemm(A, B, C)
torch.cuda.synchronize()


def per_call(fn, reps=2000):
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps * 1e6


res = {
    "G.gemm": per_call(lambda: G.gemm(A, B, C)),
    "C-ABI gemm_f64_stream (fixed args)": per_call(lambda: G._lib.gemm_f64_stream(*args)),
    "fast entry gemm_f64_ex (fixed args)": per_call(lambda: G._FAST(*args[:11], -1, 0, args[11])) if G._FAST else -1.0,
    "3x _mat": per_call(lambda: (G._mat(A, "A"), G._mat(B, "B"), G._mat(C, "C"))),
    "current_stream": per_call(lambda: torch.cuda.current_stream().cuda_stream),
}
for k, v in res.items():
    print(f"{k:40s} {v:7.2f} us")
# eager Python loop of the product call: per-call wall time (GPU-paced once host cost < kernel)
for n2 in (256, 384, 512, 1024):
    X = torch.rand((n2, n2), dtype=torch.float64, device="cuda")
    Y = torch.rand((n2, n2), dtype=torch.float64, device="cuda")
    Z = torch.zeros((n2, n2), dtype=torch.float64, device="cuda")
    for _ in range(100):
        G.gemm(X, Y, Z)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        G.gemm(X, Y, Z)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) / 2000 * 1e6
    print(f"eager G.gemm {n2}^3 loop                   {us:7.2f} us/call  {2 * n2 ** 3 / us / 1e6:6.2f} TFLOP/s")
