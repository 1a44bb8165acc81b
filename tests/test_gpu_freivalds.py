"""Full-coverage exact checks of the large configurations ("Freivalds").

Sampled oracle rows cover a few rows of a 16384^3 or 65536-wide result; these tests check
EVERY entry (every row, all or a block of the columns) in O(N^2) host work.  Inputs are in
the exact dyadic regime (m/256), where every summation order gives the same doubles, so
    C x == alpha * A (B x) + beta * C0 x        (Eq. (1) P:77-79 applied to vectors)
must hold bitwise for 16 random 0/1 columns x (oracle.freivalds; a wrong row escapes with
probability <= 2^-16).  The GPU side runs the product's own plan (the bench launch at
16384^3, the hybrid schedule with its stream-K tail and fix-up at 8192^3 and on config 4),
with inputs from the device generator; the host regenerates them from synth (the device
generator equals synth bitwise, test_device_generator_matches_synth_bitwise).
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

_POOL = ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4))


def _gen(mode, seed, mat, rows, cols, col0=0, ncols=None):
    """(r0, nr) -> synth block rows [r0, r0+nr) x cols [col0, col0+ncols), generated in
    parallel 64-row slabs (synth's counter generator is position-addressed)."""
    nc = cols - col0 if ncols is None else ncols

    def block(r0, nr):
        out = np.empty((nr, nc))

        def slab(s):
            n = min(64, nr - s)
            out[s:s + n] = synth.matrix(mode, seed, mat, rows, cols, row0=r0 + s, nrows=n, col0=col0, ncols=nc)
        list(_POOL.map(slab, range(0, nr, 64)))
        return out
    return block


def _dev_rows(dC, c0, nc):
    return lambda r0, nr: dC[r0:r0 + nr, c0:c0 + nc].cpu().numpy()


def _run(G, M, N, K, alpha, beta, seed, mode="dyadic", rows_total=None, row0=0):
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    rt = M if rows_total is None else rows_total
    G.fill(dA, mode, seed, 0, rows=rt, row0=row0)
    G.fill(dB, mode, seed, 1)
    G.fill(dC, mode, seed, 2, rows=rt, row0=row0)
    G.gemm(dA, dB, dC, alpha, beta)
    torch.cuda.synchronize()
    del dA, dB
    return dC


def _check(G, M, N, K, alpha, beta, seed, c0=0, nc=None, rows_total=None, row0=0, inject=None):
    nc = N - c0 if nc is None else nc
    cid, sp = G.plan(M, N, K, 0x1000, K, 0x1000, N)
    dC = _run(G, M, N, K, alpha, beta, seed, rows_total=rows_total, row0=row0)
    if inject is not None:   # negative control: one entry off by one unit of the exact grid
        dC[inject] += 2.0 ** -16
    rt = M if rows_total is None else rows_total
    X = np.random.default_rng(seed + 1).integers(0, 2, size=(nc, 16)).astype(np.float64)
    a_full = _gen("dyadic", seed, 0, rt, K)
    c0_full = _gen("dyadic", seed, 2, rt, N, col0=c0, ncols=nc)
    bad = oracle.freivalds(alpha, beta, X, M, K,
                           lambda r, n: a_full(row0 + r, n),
                           _gen("dyadic", seed, 1, K, N, col0=c0, ncols=nc),
                           _dev_rows(dC, c0, nc),
                           lambda r, n: c0_full(row0 + r, n), chunk=2048)
    del dC
    torch.cuda.empty_cache()
    if inject is not None:
        assert bad.tolist() == [inject[0]], bad[:8].tolist()
        return
    assert bad.size == 0, f"plan {G.cfg_name(cid)} x{sp}: {bad.size} wrong rows, first {bad[:8].tolist()}"


def test_freivalds_n16384_bench_plan_every_entry(cuda_lib):
    """The metric's 16384^3 shape with the bench's own plan, alpha=1.5, beta=0.5: all 2^28 entries."""
    _check(cuda_lib, 16384, 16384, 16384, 1.5, 0.5, seed=21)


def test_freivalds_config3_hybrid_every_entry(cuda_lib):
    """Config 3 (N=8192, alpha=1.5, beta=0.5) with the product plan (hybrid: full waves,
    stream-K tail, tail fix-up): every entry, including all cut tail tiles."""
    _check(cuda_lib, 8192, 8192, 8192, 1.5, 0.5, seed=22)


def test_freivalds_detects_one_unit_error_on_device_result(cuda_lib):
    """Negative control on the same path: one entry of the config-3 result raised by 2^-16
    on the device is found, and only its row is reported."""
    _check(cuda_lib, 8192, 8192, 8192, 1.5, 0.5, seed=22, inject=(5000, 6001))


def test_freivalds_config4_every_entry(cuda_lib):
    """Config 4's global shape (M=32768, N=K=4096) on one GPU with the product plan."""
    _check(cuda_lib, 32768, 4096, 4096, 1.5, 0.5, seed=23)


def test_freivalds_config5_rank_shard_column_block(cuda_lib):
    """Config 5 (N=65536) as one rank of the 8-GPU run computes it: global rows
    [57344, 65536) (rank 7), all 8192 rows x a 2048-column block (16.8M entries), K=65536."""
    _check(cuda_lib, 8192, 65536, 65536, 1.0, 0.0, seed=24, c0=30720, nc=2048, rows_total=65536, row0=57344)


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (3000, 5000, 2000),
                                   (1536, 1536, 1536), (700, 9000, 3000)], ids=lambda s: "x".join(map(str, s)))
def test_freivalds_config2_and_ragged_every_entry(cuda_lib, shape):
    """Config-2 sizes and ragged shapes with whatever plan the product picks (split-K,
    hybrid, XP): every entry, alpha=1.5, beta=0.5."""
    M, N, K = shape
    _check(cuda_lib, M, N, K, 1.5, 0.5, seed=M + N + K)


def test_freivalds_odd_leading_dimension_repack_every_entry(cuda_lib):
    """Odd K and N: no TMA on the caller's buffers, so the product repacks them into aligned
    workspace and runs the TMA path (10000 x 9999 x 7001, the repack test shape)."""
    _check(cuda_lib, 10000, 9999, 7001, 1.5, 0.5, seed=31)
