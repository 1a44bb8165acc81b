"""Device time per call of forced configurations on given shapes, launches back to back
(the tuner's batched timing, so host cost overlaps the kernels):
    python tools/cfg_time.py CFG[:SPLITS],CFG,... MxNxK|N,...
CFG may be "plan" (the product's own choice)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402
from paper_1706_10086_b200 import tuner  # noqa: E402


def main(cfgs, shapes):
    out = []
    for item in shapes.split(","):
        d = [int(x) for x in item.split("x")]
        M, N, K = d if len(d) == 3 else d * 3
        A = torch.empty((M, K), dtype=torch.float64, device="cuda")
        B = torch.empty((K, N), dtype=torch.float64, device="cuda")
        C = torch.empty((M, N), dtype=torch.float64, device="cuda")
        G.fill(A, "uniform", 1, 0)
        G.fill(B, "uniform", 1, 1)
        G.fill(C, "uniform", 1, 2)
        for c in cfgs.split(","):
            name, _, sp = c.partition(":")
            if name == "plan":
                fn = lambda: G.gemm(A, B, C, 1.0, 0.0)  # noqa: E731
                cid, s = G.plan(M, N, K, A.data_ptr(), K, B.data_ptr(), N)
                label = f"plan={G.cfg_name(cid)}x{s}"
            else:
                cfg = G.cfg_id(name)
                s = int(sp) if sp else None
                fn = lambda: G.gemm(A, B, C, 1.0, 0.0, cfg=cfg, splits=s)  # noqa: E731
                label = c
            best, med = tuner._time(fn, 7)
            r = {"m": M, "n": N, "k": K, "cfg": label, "us": best * 1e6, "median_us": med * 1e6,
                 "tflops": 2.0 * M * N * K / best / 1e12}
            print(json.dumps(r), flush=True)
            out.append(r)
        del A, B, C
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
