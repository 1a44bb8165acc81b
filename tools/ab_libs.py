"""A/B device time of the same plan in two builds of the library (round-to-round regression
checks): python tools/ab_libs.py LIB_A.so LIB_B.so MxNxK[,...] [rounds]
Calls gemm_f64_stream through raw ctypes (no binding), batches of back-to-back calls between
CUDA events, alternating A and B `rounds` times; prints the best TFLOP/s of each."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def load(path):
    lib = ctypes.CDLL(path)
    f = lib.gemm_f64_stream
    i64, dbl, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
    f.argtypes = [i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp]
    f.restype = ctypes.c_int
    tl = lib.gemm_tune_load
    tl.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)]
    n = ctypes.c_int()
    tl(os.fsencode(os.path.join(ROOT, "paper_1706_10086_b200", "tuned_b200.txt")), ctypes.byref(n))
    return f


def time_batch(f, M, N, K, A, B, C, calls):
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(calls):
        rc = f(M, N, K, 1.0, A.data_ptr(), K, B.data_ptr(), N, 0.0, C.data_ptr(), N, st)
        assert rc == 0, rc
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / calls


def main():
    fa, fb = load(sys.argv[1]), load(sys.argv[2])
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    for item in sys.argv[3].split(","):
        M, N, K = (int(x) for x in item.split("x"))
        A = torch.rand((M, K), dtype=torch.float64, device="cuda")
        B = torch.rand((K, N), dtype=torch.float64, device="cuda")
        C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        est = 2.0 * M * N * K / 36e12                 # seconds per call at ~36 TFLOP/s
        calls = min(2000, max(1, int(0.5 / est)))   # ~0.5 s per timed batch
        for f in (fa, fb):
            time_batch(f, M, N, K, A, B, C, min(calls, 3))
        ta, tb = [], []
        for _ in range(rounds):
            ta.append(time_batch(fa, M, N, K, A, B, C, calls))
            tb.append(time_batch(fb, M, N, K, A, B, C, calls))
        fl = 2.0 * M * N * K
        print(json.dumps({"shape": item, "a": os.path.basename(sys.argv[1]), "b": os.path.basename(sys.argv[2]),
                          "a_tflops": fl / min(ta) / 1e12, "b_tflops": fl / min(tb) / 1e12,
                          "a_all": [fl / t / 1e12 for t in ta], "b_all": [fl / t / 1e12 for t in tb]}), flush=True)


if __name__ == "__main__":
    main()
