"""Tuning sweep and size scaling of the DGEMM (§2.3 "Multidimensional parameter
tuning"; Fig. 6 scaling P:713-798) on one B200 -- run through gpurun.

    python tools/sweep.py tune  [--n 8192] [--alpha 1.5] [--beta 0.5] [--out gpurun_out/tune.csv]
    python tools/sweep.py scale [--sizes 1024,2048,4096,8192,16384] [--out gpurun_out/scale.csv]
    python tools/sweep.py ncu   [--n 8192]     # one launch per configuration, for an ncu --metrics pass

tune  = SURVEY §8(d) config 3: every configuration (CTA tile x elements per thread, the
        paper's "tile size T" x element layer) is timed (best and median of --reps CUDA-event
        runs) with SM clock and power sampled by nvidia-smi during the timing.
scale = config 2: the heuristic plan (the product's choice) or every configuration per shape.
Parity of every configuration at these shapes is checked against the CPU oracle by the GPU
test suite (tests/test_gpu_parity.py: test_config3_every_cfg_sampled_rows and the size tests),
which is the only place the oracle runs; this tool only times.
"""

import argparse
import csv
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_10086_b200 import gemm as G  # noqa: E402

PEAK = 37.0
HEADER = ["m", "n", "k", "alpha", "beta", "cfg", "splits", "tma", "bm", "bn", "bk", "wm", "wn", "e", "stages", "regs",
          "smem_bytes", "gpus", "best_s", "median_s", "tflops", "frac_peak_datasheet", "frac_peak_clock",
          "sm_mhz_mean", "power_w_mean", "parity_max_err_over_bound", "selected_by_heuristic"]


class Smi:
    def __init__(self):
        self.rows = []

    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                   "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._rd, daemon=True)
        self.t.start()
        return self

    def _rd(self):
        for line in self.p.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) == 3 and f[0] == "0":
                try:
                    self.rows.append((float(f[1]), float(f[2])))
                except ValueError:
                    pass

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()

    def means(self):
        if not self.rows:
            return None, None
        return statistics.mean(r[0] for r in self.rows), statistics.mean(r[1] for r in self.rows)


class Problem:
    def __init__(self, M, N, K, seed=1706):
        self.M, self.N, self.K, self.seed = M, N, K, seed
        self.A = torch.empty((M, K), dtype=torch.float64, device="cuda")
        self.B = torch.empty((K, N), dtype=torch.float64, device="cuda")
        self.C = torch.empty((M, N), dtype=torch.float64, device="cuda")
        G.fill(self.A, "uniform", seed, 0)
        G.fill(self.B, "uniform", seed, 1)
        self._B_host = None

    def reset_c(self):
        G.fill(self.C, "uniform", self.seed, 2)

    def run_once(self, cfg, alpha, beta, splits=None):
        self.reset_c()
        G.gemm(self.A, self.B, self.C, alpha, beta, cfg=cfg, splits=splits)
        torch.cuda.synchronize()

    def time(self, cfg, alpha, beta, reps, splits=None, warm_s=0.25):
        # warm to a steady SM clock first (short runs otherwise see the idle-clock ramp)
        t0 = time.time()
        while time.time() - t0 < warm_s:
            for _ in range(4):
                G.gemm(self.A, self.B, self.C, alpha, beta, cfg=cfg, splits=splits)
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        G.gemm(self.A, self.B, self.C, alpha, beta, cfg=cfg, splits=splits)
        torch.cuda.synchronize()
        est = time.perf_counter() - t1
        # a batch of back-to-back calls per sample (>= ~2 ms), so the host's per-call cost
        # overlaps the kernels instead of being added to small shapes (paper_1706_10086_b200.tuner)
        batch = max(1, min(256, int(2e-3 / max(est, 1e-7))))
        ts = []
        with Smi() as smi:
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(batch):
                    G.gemm(self.A, self.B, self.C, alpha, beta, cfg=cfg, splits=splits)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3 / batch)
        mhz, pw = smi.means()
        return min(ts), statistics.median(ts), mhz, pw


def sample_rows(M, bm=128, extra=4):
    rng = np.random.default_rng(M)
    s = {0, M - 1, min(bm, M - 1), M // 2} | set(int(x) for x in rng.integers(0, M, extra))
    return sorted(s)


def row(P, cfg, alpha, beta, t_best, t_med, mhz, pw, ratio, heur, splits=1):
    info = G.cfg_info(cfg)
    fl = 2.0 * P.M * P.N * P.K
    tf = fl / t_best / 1e12
    clk_peak = 148 * 128 * mhz * 1e6 / 1e12 if mhz else None
    return [P.M, P.N, P.K, alpha, beta, info["name"], splits, info["tma"], info["bm"], info["bn"], info["bk"], info["wm"],
            info["wn"], info["e"], info["stages"], info["regs"], info["smem_bytes"], 1, f"{t_best:.6f}",
            f"{t_med:.6f}", f"{tf:.3f}", f"{tf / PEAK:.4f}", f"{tf / clk_peak:.4f}" if clk_peak else "",
            f"{mhz:.0f}" if mhz else "", f"{pw:.0f}" if pw else "", "" if ratio != ratio else f"{ratio:.3e}", int(heur)]


def tune(a):
    P = Problem(a.n, a.n, a.n)
    heur = G.cfg_select(a.n, a.n, a.n, P.A.data_ptr(), a.n, P.B.data_ptr(), a.n)
    with open(a.out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(HEADER)
        for info in G.cfgs():
            cfg = info["id"]
            tb, tm, mhz, pw = P.time(cfg, a.alpha, a.beta, a.reps)
            r = row(P, cfg, a.alpha, a.beta, tb, tm, mhz, pw, float("nan"), cfg == heur)
            w.writerow(r)
            f.flush()
            print(",".join(map(str, r)), flush=True)


def _shapes(a):
    if a.shapes:
        return [tuple(int(v) for v in item.split("x")) for item in a.shapes.split(",")]
    if a.grid:
        lo, hi, step = (int(v) for v in a.grid.split(":"))
        return [(n, n, n) for n in range(lo, hi + 1, step)]
    return [(n, n, n) for n in (int(x) for x in a.sizes.split(","))]


def scale(a):
    """Heuristic plan per shape (the product's choice), or every TMA configuration."""
    with open(a.out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(HEADER)
        for (m, n, k) in _shapes(a):
            P = Problem(m, n, k)
            heur, hs = G.plan(m, n, k, P.A.data_ptr(), k, P.B.data_ptr(), n)
            cands = [None] if not a.all_cfgs else [c["id"] for c in G.cfgs() if c["tma"]]
            for cfg in cands:
                tb, tm, mhz, pw = P.time(cfg, a.alpha, a.beta, a.reps)
                r = row(P, heur if cfg is None else cfg, a.alpha, a.beta, tb, tm, mhz, pw, float("nan"),
                        cfg is None or cfg == heur, hs if cfg is None else 1)
                w.writerow(r)
                f.flush()
                print(",".join(map(str, r)), flush=True)
            del P
            torch.cuda.empty_cache()


def small(a):
    """Small sizes (row a5): every TMA configuration, split-K ones at several slice counts
    (their parity is in tests/)."""
    with open(a.out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(HEADER)
        for n in [int(x) for x in a.sizes.split(",")]:
            P = Problem(n, n, n)
            hc, hs = G.plan(n, n, n, P.A.data_ptr(), n, P.B.data_ptr(), n)
            tb, tm, mhz, pw = P.time(None, a.alpha, a.beta, a.reps)
            r = row(P, hc, a.alpha, a.beta, tb, tm, mhz, pw, float("nan"), True, hs)
            w.writerow(r)
            print(",".join(map(str, r)), flush=True)
            for info in G.cfgs():
                if not info["tma"]:
                    continue
                for S in ((1,) if info["split_k"] != 0 else (1, 2, 3, 4, 6, 8, 12)):
                    tb, tm, mhz, pw = P.time(info["id"], a.alpha, a.beta, a.reps, splits=S)
                    r = row(P, info["id"], a.alpha, a.beta, tb, tm, mhz, pw, float("nan"), False, S)
                    w.writerow(r)
                    f.flush()
                    print(",".join(map(str, r)), flush=True)
            del P
            torch.cuda.empty_cache()


def ncu_pass(a):
    """One call per configuration (ncu --metrics over the dgemm_ kernels); prints
    "cfg_id name launches" so a joiner can group the captured kernels per configuration."""
    P = Problem(a.n, a.n, a.n)
    P.reset_c()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for info in G.cfgs():
        G.gemm(P.A, P.B, P.C, a.alpha, a.beta, cfg=info["id"])
        torch.cuda.synchronize()
        print(info["id"], info["name"], G.launches_per_call(info["id"], a.n, a.n, a.n, sms), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["tune", "scale", "small", "ncu"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--beta", type=float, default=None)
    ap.add_argument("--sizes", default="1024,2048,4096,8192,16384")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--all-cfgs", action="store_true")
    ap.add_argument("--shapes", default=None, help="comma list of MxNxK")
    ap.add_argument("--grid", default=None, help="lo:hi:step square sizes (the paper's N=1024..20480, dN=1024)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.alpha is None:
        a.alpha = 1.5 if a.mode in ("tune", "ncu") else 1.0
    if a.beta is None:
        a.beta = 0.5 if a.mode in ("tune", "ncu") else 0.0
    if a.out is None:
        a.out = f"gpurun_out/{a.mode}.csv"
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    {"tune": tune, "scale": scale, "small": small, "ncu": ncu_pass}[a.mode](a)


if __name__ == "__main__":
    main()
