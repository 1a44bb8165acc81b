"""Per-CTA timelines of small GEMMs from the instrumented build (libgemm_f64_trace.so,
`python -m paper_1706_10086_b200.build --trace`): each CTA of the LAST of `reps` back-to-back
calls records globaltimer at kernel entry (0), after griddepcontrol.wait (1), when its first
pipeline stage landed (2), at the end of its (first tile's) main loop (3), before the epilogue
(4), at the end of the last tile's main loop (5, stream-K), at exit (6), and its SM id (7).

    python tools/trace_ctas.py CFG[:SPLITS]|plan MxNxK [...]  > gpurun_out/trace.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GEMM_F64_LIB"] = os.path.join(ROOT, "paper_1706_10086_b200", "libgemm_f64_trace.so")

import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

assert G.LIB_PATH.endswith("_trace.so"), G.LIB_PATH
_set = G.lib().gemm_trace_set
_set.argtypes = [ctypes.c_void_p]
_set.restype = ctypes.c_int


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))] if xs else None


def run(spec, shape, reps=8):
    name, _, sp = spec.partition(":")
    M, N, K = (int(x) for x in shape.split("x"))
    A = torch.empty((M, K), dtype=torch.float64, device="cuda")
    B = torch.empty((K, N), dtype=torch.float64, device="cuda")
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    G.fill(A, "uniform", 1, 0)
    G.fill(B, "uniform", 1, 1)
    cfg = None if name == "plan" else G.cfg_id(name)
    splits = int(sp) if sp else None
    buf = torch.zeros(8 * 65536, dtype=torch.int64, device="cuda")
    for _ in range(3):
        G.gemm(A, B, C, 1.0, 0.0, cfg=cfg, splits=splits)
    torch.cuda.synchronize()
    _set(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        G.gemm(A, B, C, 1.0, 0.0, cfg=cfg, splits=splits)
    e1.record()
    torch.cuda.synchronize()
    _set(None)
    G.gemm(A, B, C, 1.0, 0.0, cfg=cfg, splits=splits)   # re-arm with NULL for the next case
    torch.cuda.synchronize()
    per_call_us = e0.elapsed_time(e1) * 1e3 / reps
    t = buf.view(-1, 8).cpu().tolist()
    rows = [r for r in t if r[0] != 0]
    t0 = min(r[1] for r in rows)
    rel = [[(v - t0) / 1e3 if (i < 7 and v) else None for i, v in enumerate(r[:7])] + [r[7] & 0xFFFFFFFF, r[7] >> 32]
           for r in rows]
    span = max(r[6] for r in rel if r[6] is not None)
    fill = [r[2] - r[1] for r in rel if r[2] is not None and r[1] is not None]
    main = [r[3] - r[2] for r in rel if r[3] is not None and r[2] is not None]
    tail = [r[6] - r[3] for r in rel if r[6] is not None and r[3] is not None]
    start = [r[1] for r in rel]
    sms = {}
    for r in rel:
        sms.setdefault(r[7], []).append(r)
    busy = []
    for s, rs in sms.items():
        busy.append(sum(r[6] - r[1] for r in rs if r[6] is not None))
    out = {"cfg": spec, "shape": shape, "ctas": len(rel), "per_call_us": per_call_us, "span_us": span,
           "tflops_span": 2.0 * M * N * K / (span * 1e-6) / 1e12,
           "start_us_p50_p90_max": [pct(start, .5), pct(start, .9), max(start)],
           "fill_us_p10_p50_p90": [pct(fill, .1), pct(fill, .5), pct(fill, .9)],
           "main_us_p10_p50_p90": [pct(main, .1), pct(main, .5), pct(main, .9)],
           "tail_us_p10_p50_p90": [pct(tail, .1), pct(tail, .5), pct(tail, .9)],
           "ctas_per_sm_min_max": [min(len(v) for v in sms.values()), max(len(v) for v in sms.values())],
           "sms_used": len(sms),
           "cta_time_sum_per_sm_us_mean": statistics.mean(busy),
           "raw": rel}
    return out


if __name__ == "__main__":
    specs = sys.argv[1].split(",")
    shapes = sys.argv[2].split(",")
    for shape in shapes:
        for spec in specs:
            r = run(spec, shape)
            print(json.dumps(r), flush=True)
            print(json.dumps({k: v for k, v in r.items() if k != "raw"}), file=sys.stderr, flush=True)
