"""Where small GEMMs lose time: host enqueue cost per call vs device time per call.

For each square size, with the product plan:
  host_us   -- wall time per gemm() call while enqueueing 300 calls without syncing
               (Python binding + C-ABI host path + launch), measured after warm-up;
  eager_us  -- device time per call for those 300 back-to-back calls (CUDA events);
  graph_us  -- device time per call when the same 300 calls are replayed from a CUDA graph.
eager_us > graph_us means the stream starved: the host could not enqueue as fast as the
GPU ran the kernels.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [256, 512, 768, 1024, 1536, 2048, 3072, 4096]
    res = []
    s = torch.cuda.Stream()
    for n in sizes:
        A = torch.rand((n, n), dtype=torch.float64, device="cuda")
        B = torch.rand((n, n), dtype=torch.float64, device="cuda")
        C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        reps = 300 if n <= 2048 else 60
        with torch.cuda.stream(s):
            for _ in range(5):
                G.gemm(A, B, C, 1.0, 0.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            t0 = time.perf_counter()
            for _ in range(reps):
                G.gemm(A, B, C, 1.0, 0.0)
            t1 = time.perf_counter()
            e1.record(s)
        torch.cuda.synchronize()
        host_us = (t1 - t0) / reps * 1e6
        eager_us = e0.elapsed_time(e1) * 1e3 / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                G.gemm(A, B, C, 1.0, 0.0)
        g.replay()
        torch.cuda.synchronize()
        e0.record(s)
        g.replay()
        e1.record(s)
        # replay runs on the capture stream's pool; record on s around it
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_us = e0.elapsed_time(e1) * 1e3 / reps
        cid, sp = G.plan(n, n, n, A.data_ptr(), n, B.data_ptr(), n)
        r = {"n": n, "plan": G.cfg_name(cid), "splits": sp, "host_us": host_us, "eager_us": eager_us,
             "graph_us": graph_us, "eager_tflops": 2 * n ** 3 / eager_us / 1e6,
             "graph_tflops": 2 * n ** 3 / graph_us / 1e6}
        print(json.dumps(r), flush=True)
        res.append(r)
        del g
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/small_overhead.json", "w"), indent=1)


if __name__ == "__main__":
    main()
