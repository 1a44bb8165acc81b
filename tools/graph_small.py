"""Config-1 size (N=256) and other small GEMMs replayed from a CUDA graph: per-GEMM device
time without host launch overhead (the small sizes are launch/latency-bound)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def main():
    res = []
    for n in (256, 512, 1024):
        A = torch.rand((n, n), dtype=torch.float64, device="cuda")
        B = torch.rand((n, n), dtype=torch.float64, device="cuda")
        C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            G.gemm(A, B, C, 1.0, 0.0)
        torch.cuda.synchronize()
        reps = 200
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                G.gemm(A, B, C, 1.0, 0.0)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / reps
        cid, sp = G.plan(n, n, n, A.data_ptr(), n, B.data_ptr(), n)
        r = {"n": n, "us_per_gemm": t * 1e6, "tflops": 2 * n ** 3 / t / 1e12, "plan": G.cfg_name(cid), "splits": sp}
        print(json.dumps(r), flush=True)
        res.append(r)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/graph_small.json", "w"), indent=1)


if __name__ == "__main__":
    main()
