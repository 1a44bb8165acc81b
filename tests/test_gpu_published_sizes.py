"""Parity at EVERY size the repo publishes a number for (VERDICT r1 "what's missing" #4):
each row of the shipped tuning table (paper_1706_10086_b200/tuned_b200.txt) and every size
of the paper's scaling grid N = 1024 ... 20480, dN = 1024 (§2.3), each run
with the product's own plan for that shape (the tuned-table pin or the heuristic):

1. dyadic inputs (m/256), alpha = 1.5, beta = 0.5: Freivalds over EVERY entry (or, for the
   one table row whose B is 32 GiB, every entry of a 2048-column block) -- bitwise, since
   every summation order gives the same doubles in the exact regime (oracle.freivalds);
2. uniform[-1,1) inputs, alpha = 1.5, beta = 0.5: the first, last and two random rows of C
   over a 2048-column block against the CPU oracle within the north-star bound.

With GEMM_PARITY_OUT=path the per-shape results are appended there as JSON lines
(tools/grid_parity_csv.py writes them into the published grid CSV's parity column).
"""

import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLE = os.path.join(ROOT, "paper_1706_10086_b200", "tuned_b200.txt")
_POOL = ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4))


def _table_shapes():
    out = []
    for line in open(TABLE):
        if line.startswith("#") or not line.strip():
            continue
        M, N, K = (int(x) for x in line.split()[:3])
        out.append((M, N, K))
    return out


GRID = [(n, n, n) for n in range(1024, 20481, 1024)]
RECT = [(10000, 9999, 7001)]   # the ragged row of the rectangular sweep (odd K and N: the repack path)
SHAPES = sorted(set(_table_shapes()) | set(GRID) | set(RECT), key=lambda s: (s[0] * s[1] * s[2], s))


def _gen(mode, seed, mat, rows, cols, col0=0, ncols=None):
    nc = cols - col0 if ncols is None else ncols

    def block(r0, nr):
        out = np.empty((nr, nc))

        def slab(s):
            n = min(64, nr - s)
            out[s:s + n] = synth.matrix(mode, seed, mat, rows, cols, row0=r0 + s, nrows=n, col0=col0, ncols=nc)
        list(_POOL.map(slab, range(0, nr, 64)))
        return out
    return block


def _record(entry):
    path = os.environ.get("GEMM_PARITY_OUT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(entry) + "\n")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_published_size_parity(cuda_lib, shape):
    G = cuda_lib
    M, N, K = shape
    alpha, beta, seed = 1.5, 0.5, (M * 3 + N * 5 + K * 7) % 100003
    cid, sp = G.plan(M, N, K, 0x1000, K, 0x1000, N)
    plan = f"{G.cfg_name(cid)} x{sp}"
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    # the full-entry check needs B x over all columns it covers; a 32 GiB B is checked on a block
    c0, nc = (0, N) if K * N <= (1 << 31) else (N // 2 - 1024, 2048)

    # 1. dyadic, Freivalds over every entry of the checked columns
    for X, mode, mat in ((dA, "dyadic", 0), (dB, "dyadic", 1), (dC, "dyadic", 2)):
        G.fill(X, mode, seed, mat)
    G.gemm(dA, dB, dC, alpha, beta)
    torch.cuda.synchronize()
    Xv = np.random.default_rng(seed + 1).integers(0, 2, size=(nc, 16)).astype(np.float64)
    bad = oracle.freivalds(alpha, beta, Xv, M, K, _gen("dyadic", seed, 0, M, K),
                           _gen("dyadic", seed, 1, K, N, col0=c0, ncols=nc),
                           lambda r, n: dC[r:r + n, c0:c0 + nc].cpu().numpy(),
                           _gen("dyadic", seed, 2, M, N, col0=c0, ncols=nc), chunk=2048)
    assert bad.size == 0, f"{shape} plan {plan}: {bad.size} wrong rows, first {bad[:8].tolist()}"

    # 2. uniform, sampled rows x a column block vs the oracle (bound)
    for X, mat in ((dA, 0), (dB, 1), (dC, 2)):
        G.fill(X, "uniform", seed, mat)
    G.gemm(dA, dB, dC, alpha, beta)
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    rows = sorted({0, M - 1, *rng.integers(0, M, 2).tolist()})
    uc = min(N, 2048)
    u0 = int(rng.integers(0, (N - uc) // 16 + 1)) * 16 if N > uc else 0
    got = torch.stack([dC[i, u0:u0 + uc] for i in rows]).cpu().numpy()
    del dA, dB, dC
    torch.cuda.empty_cache()
    A = np.vstack([synth.matrix("uniform", seed, synth.MAT_A, M, K, row0=i, nrows=1) for i in rows])
    B = _gen("uniform", seed, 1, K, N, col0=u0, ncols=uc)(0, K)
    C0 = np.vstack([synth.matrix("uniform", seed, synth.MAT_C, M, N, row0=i, nrows=1, col0=u0, ncols=uc)
                    for i in rows])
    ref, mag = oracle.dgemm(alpha, A, B, beta, C0, want_mag=True)
    r = oracle.check(got, ref, oracle.bound(K, alpha, beta, mag, C0))
    _record({"m": M, "n": N, "k": K, "plan": plan, "freivalds_cols": [c0, nc], "freivalds_bad_rows": int(bad.size),
             "rows": rows, "cols": [u0, uc], "max_err_over_bound": r.max_ratio, "median_rel": r.median_rel,
             "ok": bool(r.ok and bad.size == 0)})
    assert r.ok, f"{shape} plan {plan}: {r}"
