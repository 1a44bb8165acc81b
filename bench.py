"""Benchmark of the one hot path: FP64 GEMM C = alpha*A*B + beta*C on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload square|rect|large|large_strong] [--bcast-chunks C]
                    [--impl ours|reference] [--no-e2e] [--no-cpu-baseline] [--verify-rows R]

Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...  (one process per GPU).

Workloads (BASELINE.json configs):
  square (default): the metric's N=16384 DGEMM, alpha=1, beta=0, seeded uniform[-1,1).
          At N GPUs it is WEAK-scaled by rows: each rank owns 16384 rows of
          A and C (M = 16384*N), B (16384 x 16384) is broadcast from rank 0 over
          NVLink with NCCL every step (row-block sharding).
  rect:   config 4, M=32768, N=K=4096 row-sharded over the ranks (strong scaling).
  large:  config 5, N=65536 square; 8192 rows per rank (weak).
  large_strong: config 5 strong: M=N=K=65536 split over the ranks (1 GPU: 96 GiB of
          operands, the T1 of E_s(P) = T1 / (P T_P)).

A step = one collective call of the sharded entry point gemm_f64_sharded (broadcast of B
from rank 0, then the local DGEMM over the rank's rows) at N > 1 or under torchrun, and
one gemm_f64 launch at N = 1.  Inputs are device-resident and larger than L2 (>= 128 MiB
each at the default workload), so no L2 flush is needed.  Time = CUDA events on the
launching stream over exactly K steps after W warm-ups, barrier + synchronize on both
sides, max over ranks.  value = 2*M*N*K*K_steps / time (Eq. (4) P:93-97 convention, 2MNK).

After the timed region every rank checks its own result (post-timing, test
infrastructure, never inside the timed region): B's bytes against the device generator
(the broadcast delivered B intact) and R sampled rows of its C shard -- the first, the
last and random ones, over a block of up to 2048 columns -- against the CPU oracle within
the north-star bound.  The line carries "parity" (max over ranks); a mismatch exits 1.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DGEMM TFLOP/s and % of B200 FP64 peak at N=16384 (1 GPU) and 1/2/4/8 GPUs"
FP64_DATASHEET_TFLOPS = 37.0      # HGX B200: 296 TFLOP/s FP64 / FP64 tensor per 8 GPUs
BF16_NOMINAL_TFLOPS = 2250.0      # B200_PROFILING.md nominal dense bf16
# the oracle timed on the GPU box's host: 1 thread / all threads, full runs N=256..4096 (tools/cpu_table.py)
CPU_TABLE = "profiles/r02/cpu_baseline_table.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="square", choices=["square", "rect", "large", "large_strong"])
    ap.add_argument("--bcast-chunks", type=int, default=1,
                    help="gemm_f64_sharded column panels (1: broadcast of B, then the GEMM)")
    ap.add_argument("--verify-rows", type=int, default=4, help="sampled rows per rank checked against the oracle")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    ap.add_argument("--cfg", type=int, default=-1, help="force a kernel configuration id")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    return a


def stdout_to_stderr(fn):
    """Run fn with the process's C-level stdout (fd 1) pointed at stderr: NCCL prints its
    version banner on stdout when a communicator is created, and rank 0's stdout must carry
    exactly one line, the JSON result."""
    sys.stdout.flush()
    saved = os.dup(1)
    try:
        os.dup2(2, 1)
        return fn()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def workload(name, world):
    """(M_total, N, K, scaling, description)."""
    if name == "square":
        n = 16384
        M = n * world
        return M, n, n, "weak", f"dgemm_n{n}_rows{n}_per_gpu"
    if name == "rect":
        return 32768, 4096, 4096, "strong", "dgemm_m32768_n4096_k4096_rowsharded"
    n = 65536
    if name == "large_strong":
        return n, n, n, "strong", f"dgemm_n{n}_rowsharded"
    return 8192 * world, n, n, "weak", f"dgemm_n{n}_rows8192_per_gpu"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = str(gpu_index)
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[0] == self.idx:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        pw = [num(r[3]) for r in self.rows if num(r[3]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k].lower().startswith("active")})
        load = [s for s in sm]   # sampled only inside the timed region
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_median": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(M, N, K, seconds, seed=1706):
    """Time the CPU oracle (as it stands) on R rows of the workload; returns dict."""
    import numpy as np

    import oracle
    import synth
    threads = oracle.default_threads()
    B = synth.matrix("uniform", seed, synth.MAT_B, K, N)
    R = threads
    A = synth.matrix("uniform", seed, synth.MAT_A, M, K, row0=0, nrows=R)
    C = np.zeros((R, N))
    t0 = time.perf_counter()
    oracle.dgemm(1.0, A, B, 0.0, C, nthreads=threads)
    dt = time.perf_counter() - t0
    if dt < seconds / 3:
        R = max(R, int(R * seconds / max(dt, 1e-3)) // threads * threads)
        R = min(R, M)
        A = synth.matrix("uniform", seed, synth.MAT_A, M, K, row0=0, nrows=R)
        C = np.zeros((R, N))
        t0 = time.perf_counter()
        oracle.dgemm(1.0, A, B, 0.0, C, nthreads=threads)
        dt = time.perf_counter() - t0
    return {"value": 2.0 * R * N * K / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{R} rows of the {M}x{N}x{K} problem (i-k-j C oracle, -O2, {threads} threads), {dt:.2f} s",
            "cpu_model": cpu_model(), "table": CPU_TABLE}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on this arm's config and metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth
    world = a.gpus
    M, N, K, scaling, wname = workload(a.workload, world)
    threads = oracle.default_threads()
    B = synth.matrix("uniform", 1706, synth.MAT_B, K, N)
    R = threads
    A = synth.matrix("uniform", 1706, synth.MAT_A, M, K, row0=0, nrows=R)
    C = np.zeros((R, N))
    for _ in range(a.warmup):
        oracle.dgemm(1.0, A, B, 0.0, C, nthreads=threads)
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        oracle.dgemm(1.0, A, B, 0.0, C, nthreads=threads)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    value = 2.0 * R * N * K * a.steps / tot / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(wname, M, N, K, world),
            "impl_detail": {"sample_rows_per_step": R, "parallelism": f"{threads} host threads",
                            "inputs": "synth generator (host)"},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": f"{R} rows of the {M}x{N}x{K} problem per step (i-k-j C oracle)",
                             "cpu_model": cpu_model(), "table": CPU_TABLE},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(wname, M, N, K, world):
    """The `config` both arms print (the workload, identical for the GPU arm and the reference
    arm at the same N); how each arm executes it goes to `impl_detail`."""
    return {"workload": wname, "M": M, "N": N, "K": K, "rows_per_gpu": M // world, "alpha": 1.0, "beta": 0.0,
            "inputs": "seeded uniform[-1,1) (synth counter-based generator, seed 1706)",
            "l2": "inputs larger than L2 (no flush)"}


# ---------------------------------------------------------------------- parity (post-timing)
def sample_rows(Ml, nrows, seed):
    """Local row indices checked on a rank: first, last and random ones (sorted, unique)."""
    import numpy as np
    if Ml <= 0:
        return []
    rng = np.random.default_rng(seed)
    extra = rng.integers(0, Ml, max(0, nrows - 2)).tolist()
    return sorted({0, Ml - 1, *extra})


def check_rows(got, M, N, K, r0, rows, seed, col0, ncols):
    """Oracle check of C[r0 + rows, col0:col0+ncols] of the bench problem (alpha=1, beta=0,
    uniform inputs of `seed`): regenerates A's rows and B's column block on the host (synth)
    and compares `got` (len(rows) x ncols) within the north-star bound.  Returns
    (ok, max_err_over_bound)."""
    import numpy as np

    import oracle
    import synth
    if not rows or ncols == 0:
        return True, 0.0
    A = np.vstack([synth.matrix("uniform", seed, synth.MAT_A, M, K, row0=r0 + i, nrows=1) for i in rows])
    B = synth.matrix("uniform", seed, synth.MAT_B, K, N, col0=col0, ncols=ncols)
    ref, mag = oracle.dgemm(1.0, A, B, 0.0, np.zeros((len(rows), ncols)), want_mag=True)
    r = oracle.check(np.asarray(got, dtype=np.float64), ref, oracle.bound(K, 1.0, 0.0, mag, None))
    return bool(r.ok), float(r.max_ratio)


def reduce_parity(ok, ratio, b_ok, nrows, world, device=None):
    """Combine per-rank results: ok = all ranks ok, max_ratio = max over ranks."""
    bad = 0.0 if (ok and b_ok) else 1.0
    if world > 1:
        bad, ratio, bbad, nrows = max_over_ranks_sum(bad, ratio, 0.0 if b_ok else 1.0, nrows, world, device)
        b_ok = bbad == 0.0
    return {"ok": bad == 0.0, "max_ratio": ratio, "b_bitwise": bool(b_ok), "rows_checked_total": int(nrows)}


def max_over_ranks_sum(bad, ratio, bbad, nrows, world, device):
    """(max, max, max, sum) over ranks (torch.distributed, any backend)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([bad, ratio, bbad], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(nrows)], dtype=torch.float64, device=device)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t[0]), float(t[1]), float(t[2]), float(n[0])


def verify(G, dB, dC, M, N, K, r0, Ml, rank, nrows, seed=1706):
    """Post-timing self-check of one rank: B's bytes vs the device generator, sampled rows of
    the local C vs the oracle.  Returns (ok, max_ratio, b_ok, rows_checked, detail)."""
    import torch
    b_ok = True
    slab = max(1, min(K, (1 << 27) // max(N, 1)))          # <= 1 GiB of regenerated B at a time
    tmp = torch.empty((slab, N), dtype=torch.float64, device=dB.device)
    for k0 in range(0, K, slab):
        nk = min(slab, K - k0)
        G.fill(tmp[:nk], "uniform", seed, 1, rows=K, row0=k0)
        b_ok = b_ok and bool(torch.equal(tmp[:nk], dB[k0:k0 + nk]))
    del tmp
    rows = sample_rows(Ml, nrows, seed + 7919 * rank)
    ncols = min(N, 2048)
    col0 = 0 if N == ncols else int((seed + 131 * rank) % ((N - ncols) // 16 + 1)) * 16
    got = torch.stack([dC[i, col0:col0 + ncols] for i in rows]).cpu().numpy() if rows else None
    ok, ratio = check_rows(got, M, N, K, r0, rows, seed, col0, ncols)
    return ok, ratio, b_ok, len(rows), {"rows_local": rows, "col0": col0, "ncols": ncols}


def measure_fp64_roof(G, reps=3):
    """The FP64 tensor-pipe roof measured in-run: gemm_peak_probe, DMMA.8x8x4, 148 blocks x 16
    warps x 8 independent accumulator chains (Eq. (8), P = f*o*n measured);
    best of `reps` ~50 ms bursts.  TFLOP/s."""
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    blocks, warps, iters = sms, 16, 100000
    out = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    G.peak_probe("dmma", blocks, warps, 2000, out)
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.peak_probe("dmma", blocks, warps, iters, out)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, blocks * warps * iters * 8 * 512 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def run_e2e(a, G, dist, comm, stream, dA, dB, dC, M, N, K, Ml, world, flops_step):
    """The same metric end to end through gemm_f64_host (pinned host A, B, C; H2D and D2H
    inside the timed region, overlapped with the kernel by the library).  Every rank
    reaches the same collectives even if its local part fails (no hang at N > 1)."""
    import torch
    err = None
    e2e_s = float("inf")
    try:
        hA = torch.empty((Ml, K), dtype=torch.float64, pin_memory=True)
        hB = torch.empty((K, N), dtype=torch.float64, pin_memory=True)
        hC = torch.empty((Ml, N), dtype=torch.float64, pin_memory=True)
        hA.copy_(dA)
        hB.copy_(dB)          # B was broadcast by the timed steps: identical on every rank
        hC.copy_(dC)
        torch.cuda.synchronize()
        G.gemm_host(hA, hB, hC, 1.0, 0.0)   # warm (allocates the library's device pool)
    except Exception as ex:
        err = f"{type(ex).__name__}: {ex}"[:300]
    if world > 1:
        dist.barrier()
    if err is None:
        try:
            ts = []
            for _ in range(a.e2e_steps):
                t0 = time.perf_counter()
                G.gemm_host(hA, hB, hC, 1.0, 0.0)
                ts.append(time.perf_counter() - t0)
            e2e_s = sum(ts)
            G.host_pool_release()
        except Exception as ex:
            err = f"{type(ex).__name__}: {ex}"[:300]
            e2e_s = float("inf")
    e2e_s = G.max_over_ranks([e2e_s], world, device="cuda")[0]
    if err is not None or e2e_s == float("inf"):
        return {"value": None, "unit": "TFLOP/s", "error": err or "failed on another rank"}
    return {"value": flops_step * a.e2e_steps / e2e_s / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": 8 * (M * K + world * K * N), "d2h_bytes_per_step": 8 * M * N,
            "steps": a.e2e_steps,
            "api": "gemm_f64_host: pinned host A, B, C; H2D/D2H overlapped with the kernel by blocks"}


# ---------------------------------------------------------------------- ours
def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist

    from paper_1706_10086_b200 import gemm as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    # launched by torchrun (even with one rank): take the distributed path -- process group,
    # library NCCL communicator, gemm_f64_sharded every step -- so N=1 under torchrun runs
    # the same code as N>1 (a 1-rank broadcast is a no-op)
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ or "GEMM_BENCH_FORCE_DIST" in os.environ
    if distributed:
        stdout_to_stderr(lambda: dist.init_process_group("nccl", device_id=torch.device("cuda", local)))

    M, N, K, scaling, wname = workload(a.workload, world)
    r0, r1 = G.row_range(M, rank, world)
    Ml = r1 - r0
    dA = torch.empty((Ml, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((Ml, N), dtype=torch.float64, device="cuda")
    G.fill(dA, "uniform", 1706, 0, rows=M, row0=r0)
    if rank == 0:
        G.fill(dB, "uniform", 1706, 1)
    else:
        dB.zero_()
    G.fill(dC, "uniform", 1706, 2, rows=M, row0=r0)
    stream = torch.cuda.current_stream()
    # The step at N > 1 is the library's sharded entry point (gemm_f64_sharded: broadcast of B
    # over its own NCCL communicator, then the local GEMM).  If that communicator cannot be
    # created on some rank, every rank falls back to torch's NCCL broadcast + gemm_f64, so the
    # scaling run still measures the sharded path; the line says so.
    comm, step_via = None, "gemm_f64 (1 GPU)"
    if distributed:
        err = None
        try:
            if os.environ.get("GEMM_BENCH_TORCH_BCAST"):   # exercise the fallback (tests)
                raise RuntimeError("forced by GEMM_BENCH_TORCH_BCAST")
            comm = stdout_to_stderr(lambda: G.Comm(rank, world))
            n_nccl, r_nccl = comm.info()
            print(f"[rank {rank}] library NCCL communicator: ncclCommCount={n_nccl} ncclCommUserRank={r_nccl} "
                  f"rows [{r0}, {r1})", file=sys.stderr, flush=True)
            if n_nccl != world or r_nccl != rank:
                raise RuntimeError(f"NCCL reports {n_nccl} ranks / rank {r_nccl}, expected {world} / {rank}")
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            err = f"{type(ex).__name__}: {ex}"[:200]
        ok = torch.tensor([0.0 if err else 1.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() < 1.0:
            if comm is not None:
                comm.close()
            comm = None
            step_via = "torch.distributed NCCL broadcast + gemm_f64 (library communicator failed: " + \
                (err or "on another rank") + ")"
        else:
            step_via = f"gemm_f64_sharded (library NCCL communicator, bcast_chunks={a.bcast_chunks})"
    # the product's own plan (heuristic entry point) unless a configuration is forced; the
    # sharded entry point runs the one-k-pass plan of each column panel (bitwise equal to 1 GPU)
    cfg = a.cfg if a.cfg >= 0 else None
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    if comm is not None:
        if cfg is not None:
            print("warning: --cfg is ignored by gemm_f64_sharded (it runs the product plan)", file=sys.stderr)
            cfg = None
        panels = G.sharded_panels(N, a.bcast_chunks)
        plans = [G.plan(Ml, w, K, dA.data_ptr(), K, dB.data_ptr(), w if len(panels) > 1 else N, one_pass=True)
                 for _, w in panels]
        plan_cfg, plan_splits = plans[-1 if len(panels) == 1 else 0]
        launches_per_step = sum(G.launches_per_call(c, Ml, w, K, sms) for (c, _), (_, w) in zip(plans, panels))
    else:
        plan_cfg, plan_splits = G.plan(Ml, N, K, dA.data_ptr(), K, dB.data_ptr(), N)
        launches_per_step = G.launches_per_call(cfg if cfg is not None else plan_cfg, Ml, N, K, sms)
    cfg_name = G.cfg_name(cfg if cfg is not None else plan_cfg)
    if cfg is None and plan_splits > 1:
        cfg_name += f" (split-K x{plan_splits})"

    def step(evs=None):
        if evs is not None:
            evs[0].record(stream)
        if comm is not None:
            comm.gemm_sharded(dA, dB, dC, 1.0, 0.0, root=0, bcast_chunks=a.bcast_chunks, stream=stream)
        else:
            if distributed:
                dist.broadcast(dB, src=0)
            G.gemm(dA, dB, dC, 1.0, 0.0, cfg=cfg, stream=stream)
        if evs is not None:
            evs[1].record(stream)

    # the FP64 roof of this GPU, measured in this run before the timed region (DMMA probe)
    peak_measured = measure_fp64_roof(G)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()

    smi_index = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        try:
            smi_index = int(cvd.split(",")[local])
        except (ValueError, IndexError):
            pass
    sampler = ClockSampler(smi_index)
    sampler.start()
    time.sleep(0.3)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for i in range(a.steps):
        step(sev[i])
    e_end.record(stream)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.stop()
    t_ms = e_start.elapsed_time(e_end)
    s_ms = [s.elapsed_time(e) for s, e in sev]
    clocks = sampler.summary()

    # ---- the dominant kernel alone (roofline) and the exchange alone, after the timed region:
    # at N = 1 the step IS the kernel; at N > 1 the GEMM and the broadcast are timed apart
    if distributed:
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for s_, e_ in kev:   # the sharded call's GEMM: one-k-pass plan over all N columns
            s_.record(stream)
            G.gemm(dA, dB, dC, 1.0, 0.0, stream=stream, splits=1 if comm is not None else None)
            e_.record(stream)
        bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for s_, e_ in bev:
            s_.record(stream)
            if comm is not None:
                comm.bcast(dB, root=0, stream=stream)
            else:
                dist.broadcast(dB, src=0)
            e_.record(stream)
        torch.cuda.synchronize()
        k_mean = statistics.mean(s_.elapsed_time(e_) for s_, e_ in kev)
        b_mean = statistics.mean(s_.elapsed_time(e_) for s_, e_ in bev)
    else:
        k_mean, b_mean = statistics.mean(s_ms), 0.0
    t_ms, k_mean, b_mean = G.max_over_ranks([t_ms, k_mean, b_mean], world, device="cuda")
    flops_step = 2.0 * M * N * K
    value = flops_step * a.steps / (t_ms * 1e-3) / 1e12
    flops_local = 2.0 * Ml * N * K
    achieved = flops_local / (k_mean * 1e-3) / 1e12

    # ---- every rank checks its own result (post-timing)
    v_ok, v_ratio, v_b, v_rows, v_detail, v_err = False, float("inf"), False, 0, {}, None
    try:
        v_ok, v_ratio, v_b, v_rows, v_detail = verify(G, dB, dC, M, N, K, r0, Ml, rank, a.verify_rows)
    except Exception as ex:  # noqa: BLE001 -- a failed check is a parity failure, reported
        v_err = f"{type(ex).__name__}: {ex}"[:300]
    print(f"[rank {rank}] parity: rows {v_detail.get('rows_local')} (+{r0}) cols "
          f"[{v_detail.get('col0')}, +{v_detail.get('ncols')}) ok={v_ok} max err/bound={v_ratio:.3e} "
          f"B bitwise={v_b} {v_err or ''}", file=sys.stderr, flush=True)
    parity = reduce_parity(v_ok, v_ratio, v_b, v_rows, world if distributed else 1, device="cuda")
    parity["check"] = ("per rank: B vs the device generator (bitwise); first, last and random rows of the "
                       "local C over <= 2048 columns vs the CPU oracle (north-star bound); max over ranks")
    if v_err:
        parity["error_rank0" if rank == 0 else "error"] = v_err

    # ---- roofline of the dominant (only) kernel ------------------------------------
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        pj = json.load(open(prof))
        ent = pj.get(f"{Ml}x{N}x{K}")
        if ent and ent.get("kernel") == cfg_name:   # only a capture of this very kernel counts
            traffic = ent["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_measured, "unit": "TFLOP/s",
                "frac": achieved / peak_measured, "traffic": traffic,
                "peak_source": "measured in this run: FP64 tensor pipe (DMMA.8x8x4) probe, 148 SMs x 16 warps x 8 "
                               "independent chains, best of 3 (gemm_peak_probe; Eq. (8) P:259-262). "
                               "MEASURED_PEAKS.json has no FP64 entry (DESIGN.md §Roofline)",
                "peak_datasheet": FP64_DATASHEET_TFLOPS, "frac_of_datasheet": achieved / FP64_DATASHEET_TFLOPS,
                "kernel": cfg_name, "kernel_ms_mean": k_mean, "flops_per_launch": flops_local,
                "launches_per_gemm": launches_per_step,
                # compulsory HBM bytes of one GEMM (A, B read once, C written once; beta = 0), for
                # comparison with `traffic` (DESIGN.md §6 explains the gap: L2-sized waves)
                "algorithmic_bytes": 8.0 * (Ml * K + K * N + Ml * N)}
    if peaks.get("bf16_tflops"):
        roofline["peak_bf16_scaled"] = peaks["bf16_tflops"] * FP64_DATASHEET_TFLOPS / BF16_NOMINAL_TFLOPS
    if clocks.get("sm_mhz"):
        clk_peak = sms * 128 * clocks["sm_mhz"] * 1e6 / 1e12
        roofline["peak_at_run_clock"] = clk_peak
        roofline["frac_at_run_clock"] = achieved / clk_peak

    # ---- end to end through the host-buffer C-ABI call ------------------------------
    e2e = None
    if a.workload in ("large", "large_strong") and not a.no_e2e:
        # 40+ GiB of pinned host memory per rank (B alone is 32 GiB): not run by default
        e2e = {"value": None, "unit": "TFLOP/s", "skipped": f"{a.workload} workload: >= 40 GiB pinned host buffers"}
    elif not a.no_e2e:
        try:
            e2e = run_e2e(a, G, dist, comm, stream, dA, dB, dC, M, N, K, Ml, world, flops_step)
        except Exception as ex:  # the line must still print; the failure is reported in it
            e2e = {"value": None, "unit": "TFLOP/s", "error": f"{type(ex).__name__}: {ex}"[:300]}
        dA = dC = None

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_oracle_sample(M, N, K, a.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": t_ms / a.steps, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(wname, M, N, K, world),
                "impl_detail": {"kernel_cfg": cfg_name, "inputs": "synth generator's device twin (gemm_fill_f64)",
                                "parallelism": f"row-sharded x{world}, B broadcast (NCCL)" if world > 1 else "1 GPU",
                                "step": step_via},
                "pct_of_fp64_peak": 100.0 * value / (FP64_DATASHEET_TFLOPS * world),
                "clocks": clocks, "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": a.steps * launches_per_step}
        if distributed:
            # the one exchange step, timed alone after the timed region
            line["exchange"] = {"op": "broadcast of B (NCCL)", "bytes_per_step": 8 * K * N, "ms_per_step": b_mean,
                                "share_of_step": b_mean / (t_ms / a.steps),
                                "gemm_ms": k_mean,
                                "algbw_GBs": (8 * K * N / (b_mean * 1e-3) / 1e9) if (b_mean > 0 and world > 1) else None}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if distributed:
        dist.destroy_process_group()
    return 0 if parity["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
