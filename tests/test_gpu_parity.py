"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: elementwise
    |C_gpu - C_ref| <= 4 K 2^-53 |alpha| (|A||B|)_ij + 4 2^-53 |beta| |C0_ij| + 1e-300
on seeded uniform[-1,1) inputs (BASELINE.json north_star); BITWISE equality in the
exact dyadic regime, for integer work (index coverage, padding untouched) and for
invariants (determinism, all configurations agree).
"""

import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_gpu(G, A, B, C0, alpha, beta, cfg=None, splits=None):
    dA, dB, dC = dev(A), dev(B), dev(C0)
    G.gemm(dA, dB, dC, alpha, beta, cfg=cfg, splits=splits)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def check_vs_oracle(C_gpu, A, B, C0, alpha, beta):
    ref, mag = oracle.dgemm(alpha, A, B, beta, C0, want_mag=True)
    r = oracle.check(C_gpu, ref, oracle.bound(A.shape[1], alpha, beta, mag, C0))
    assert r.ok, str(r)
    return r


def all_cfgs(G):
    return list(range(G.num_cfgs()))


# ---------------------------------------------------------------- config 1
@pytest.mark.parametrize("seed", [1706, 1, 2, 3])
def test_config1_n256(cuda_lib, seed):
    A, B, C0 = synth.problem(256, 256, 256, seed=seed)
    C = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0)
    r = check_vs_oracle(C, A, B, C0, 1.0, 0.0)
    assert r.max_ratio < 0.05   # a ratio near 1 would signal a bug even though it passes


EDGE = [(1, 1, 1), (2, 2, 2), (7, 5, 3), (8, 16, 4), (31, 33, 17), (127, 129, 65), (129, 127, 257),
        (257, 130, 33), (300, 333, 257), (65, 200, 1), (3, 1000, 40), (1000, 3, 40), (130, 130, 2000)]


@pytest.mark.parametrize("shape", EDGE, ids=lambda s: "x".join(map(str, s)))
def test_edge_shapes_every_cfg(cuda_lib, shape):
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=M * 7 + N)
    # packed lda = K, ldb = N: TMA needs 16-byte strides (a single-row operand's stride is unused)
    tma_eligible = (K % 2 == 0 or M == 1) and (N % 2 == 0 or K == 1)
    ran = 0
    for info in cuda_lib.cfgs():
        if info["tma"] and not tma_eligible:
            with pytest.raises(cuda_lib.GemmError) as ei:
                run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=info["id"])
            assert ei.value.code == cuda_lib.GEMM_ERR_UNSUPPORTED
            continue
        C = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=info["id"])
        check_vs_oracle(C, A, B, C0, 1.5, 0.5)
        ran += 1
    assert ran >= 2
    # the heuristic path always works
    check_vs_oracle(run_gpu(cuda_lib, A, B, C0, 1.5, 0.5), A, B, C0, 1.5, 0.5)


@pytest.mark.parametrize("shape", [(0, 5, 5), (5, 0, 5)])
def test_empty_is_noop(cuda_lib, shape):
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K)
    C = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0)
    assert C.shape == (M, N)


def test_k_zero_scales_C(cuda_lib):
    C0 = synth.matrix("uniform", 1, 2, 70, 90)
    dC = dev(C0)
    dA = torch.empty((70, 0), dtype=torch.float64, device="cuda")
    dB = torch.empty((0, 90), dtype=torch.float64, device="cuda")
    cuda_lib.gemm(dA, dB, dC, 2.0, 0.25)
    torch.cuda.synchronize()
    assert np.array_equal(dC.cpu().numpy(), 0.25 * C0)


def test_alpha_zero_does_not_read_AB(cuda_lib):
    C0 = synth.matrix("uniform", 1, 2, 64, 48)
    A = np.full((64, 32), np.nan)
    B = np.full((32, 48), np.nan)
    C = run_gpu(cuda_lib, A, B, C0, 0.0, 2.0)
    assert np.array_equal(C, 2.0 * C0)


def test_beta_zero_does_not_read_C(cuda_lib):
    A, B, _ = synth.problem(200, 150, 64, seed=5)
    C = run_gpu(cuda_lib, A, B, np.full((200, 150), np.nan), 1.0, 0.0)
    assert np.all(np.isfinite(C))
    check_vs_oracle(C, A, B, np.zeros((200, 150)), 1.0, 0.0)


def test_nan_in_A_poisons_exactly_its_row(cuda_lib):
    A, B, C0 = synth.problem(300, 260, 100, seed=6)
    A[137, 42] = np.nan
    C = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0)
    assert np.all(np.isnan(C[137]))
    assert np.all(np.isfinite(np.delete(C, 137, axis=0)))


# ---------------------------------------------------------------- exact regime
@pytest.mark.parametrize("mode", ["dyadic", "int8"])
def test_exact_regime_bitwise_every_cfg(cuda_lib, mode):
    """Every partial sum is exact -> any summation order gives the same bits."""
    A, B, C0 = synth.problem(520, 390, 1000, mode=mode, seed=2)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    for cfg in all_cfgs(cuda_lib):
        C = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg)
        assert np.array_equal(C, ref), cuda_lib.cfg_name(cfg)


def test_all_cfgs_bitwise_identical_and_deterministic(cuda_lib):
    """Every configuration sums each entry in the same order (16-deep k-groups ascending,
    same k-permutation, same DMMA chain) -> identical bits; and runs repeat bitwise."""
    A, B, C0 = synth.problem(334, 290, 778, seed=3)
    # split-K configurations with one slice run the same chain as the others; stream-K and
    # the hybrid cut tiles between CTAs (a different association) and are checked separately
    ids = [c["id"] for c in cuda_lib.cfgs() if c["split_k"] >= 0]
    outs = [run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=c, splits=1) for c in ids]
    for c, o in zip(ids, outs):
        assert np.array_equal(o, outs[0]), cuda_lib.cfg_name(c)
    again = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=0)
    assert np.array_equal(again, outs[0])
    check_vs_oracle(outs[0], A, B, C0, 1.5, 0.5)


# ---------------------------------------------------------------- split-K (row a5)
def split_cfgs(G):
    return [c["id"] for c in G.cfgs() if c["split_k"] == 0]


def streamk_cfgs(G):
    return [c["id"] for c in G.cfgs() if c["split_k"] < 0]   # stream-K and hybrid


@pytest.mark.parametrize("shape", [(70, 90, 1000), (256, 256, 256), (129, 200, 777), (64, 64, 16), (31, 33, 2000)],
                         ids=lambda s: "x".join(map(str, s)))
def test_split_k_within_bound_and_deterministic(cuda_lib, shape):
    M, N, K = shape
    N += N & 1
    K += K & 1
    A, B, C0 = synth.problem(M, N, K, seed=K)
    for cfg in split_cfgs(cuda_lib):
        for S in (2, 3, 5, 16):
            C = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg, splits=S)
            check_vs_oracle(C, A, B, C0, 1.5, 0.5)
            again = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg, splits=S)
            assert np.array_equal(C, again), (cuda_lib.cfg_name(cfg), S)


def test_split_k_exact_regime_bitwise(cuda_lib):
    A, B, C0 = synth.problem(200, 300, 1500, mode="dyadic", seed=4)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    for cfg in split_cfgs(cuda_lib):
        for S in (2, 7):
            assert np.array_equal(run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg, splits=S), ref)


def test_split_k_counters_self_reset_many_launches(cuda_lib):
    """Tile counters are reset by the reducing CTA: 50 back-to-back launches on one stream
    (and a different split count in between) all give the same bits."""
    A, B, C0 = synth.problem(128, 192, 640, seed=5)
    cfg = split_cfgs(cuda_lib)[0]
    dA, dB = dev(A), dev(B)
    first = None
    for it in range(50):
        dC = dev(C0)
        cuda_lib.gemm(dA, dB, dC, 1.0, 1.0, cfg=cfg, splits=4 if it % 7 else 3)
        torch.cuda.synchronize()
        out = dC.cpu().numpy()
        if it % 7:
            first = out if first is None else first
            assert np.array_equal(out, first), it
    check_vs_oracle(first, A, B, C0, 1.0, 1.0)


def test_split_k_forced_on_plain_cfg_is_rejected(cuda_lib):
    plain = [c["id"] for c in cuda_lib.cfgs() if c["split_k"] == 1 and c["tma"]][0]
    A, B, C0 = synth.problem(64, 64, 64)
    with pytest.raises(cuda_lib.GemmError) as ei:
        run_gpu(cuda_lib, A, B, C0, 1.0, 0.0, cfg=plain, splits=2)
    assert ei.value.code == cuda_lib.GEMM_ERR_UNSUPPORTED


@pytest.mark.parametrize("n", [256, 512, 768, 1024])
def test_small_sizes_heuristic_plan(cuda_lib, n):
    """The product's own choice (possibly split-K) on config-1/2-like small sizes."""
    A, B, C0 = synth.problem(n, n, n, seed=n)
    check_vs_oracle(run_gpu(cuda_lib, A, B, C0, 1.0, 0.0), A, B, C0, 1.0, 0.0)


@pytest.mark.parametrize("shape", [(64, 64, 16), (70, 90, 1000), (256, 256, 256), (129, 200, 778), (1024, 1024, 1024),
                                   (300, 2000, 64), (2048, 2048, 2048)], ids=lambda s: "x".join(map(str, s)))
def test_stream_k_within_bound_and_deterministic(cuda_lib, shape):
    """Stream-K: tiles cut between CTAs are finished by a segment-ordered reduction."""
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=M + 3)
    for cfg in streamk_cfgs(cuda_lib):
        C = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg)
        check_vs_oracle(C, A, B, C0, 1.5, 0.5)
        assert np.array_equal(C, run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg)), cuda_lib.cfg_name(cfg)


def test_stream_k_exact_regime_bitwise_and_counters_reset(cuda_lib):
    A, B, C0 = synth.problem(700, 650, 1300, mode="dyadic", seed=6)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    dA, dB = dev(A), dev(B)
    for cfg in streamk_cfgs(cuda_lib):
        for _ in range(5):
            dC = dev(C0)
            cuda_lib.gemm(dA, dB, dC, 1.5, 0.5, cfg=cfg)
            torch.cuda.synchronize()
            assert np.array_equal(dC.cpu().numpy(), ref), cuda_lib.cfg_name(cfg)


# ---------------------------------------------------------------- layout / padding
def test_padded_leading_dimensions_untouched(cuda_lib):
    """lda > K, ldb > N, ldc > N: padding holds NaN sentinels that must be neither read
    nor written (bitwise unchanged)."""
    M, N, K = 150, 140, 90
    A, B, C0 = synth.problem(M, N, K, seed=8)
    for pad in (2, 3, 5):   # even pads -> TMA path, odd -> generic path
        Ap = np.full((M, K + pad), np.nan); Ap[:, :K] = A
        Bp = np.full((K, N + pad), np.nan); Bp[:, :N] = B
        Cp = np.full((M, N + pad), np.nan); Cp[:, :N] = C0
        dA, dB, dC = dev(Ap), dev(Bp), dev(Cp)
        cuda_lib.gemm(dA[:, :K], dB[:, :N], dC[:, :N], 1.5, 0.5)
        torch.cuda.synchronize()
        out = dC.cpu().numpy()
        assert np.all(np.isnan(out[:, N:])), "padding columns of C were written"
        check_vs_oracle(out[:, :N], A, B, C0, 1.5, 0.5)


def test_misaligned_pointers_take_generic_path(cuda_lib):
    M, N, K = 97, 101, 67
    A, B, C0 = synth.problem(M, N, K, seed=9)
    bufA = torch.zeros(M * K + 1, dtype=torch.float64, device="cuda")
    bufB = torch.zeros(K * N + 1, dtype=torch.float64, device="cuda")
    bufC = torch.zeros(M * N + 1, dtype=torch.float64, device="cuda")
    dA = bufA[1:].view(M, K); dA.copy_(dev(A))
    dB = bufB[1:].view(K, N); dB.copy_(dev(B))
    dC = bufC[1:].view(M, N); dC.copy_(dev(C0))
    cuda_lib.gemm(dA, dB, dC, 1.0, 1.0)
    torch.cuda.synchronize()
    check_vs_oracle(dC.cpu().numpy(), A, B, C0, 1.0, 1.0)
    tma_ids = [c["id"] for c in cuda_lib.cfgs() if c["tma"]]
    with pytest.raises(cuda_lib.GemmError) as ei:
        cuda_lib.gemm(dA, dB, dC, 1.0, 1.0, cfg=tma_ids[0])
    assert ei.value.code == cuda_lib.GEMM_ERR_UNSUPPORTED


def test_large_unaligned_problem_is_repacked_to_tma(cuda_lib):
    """Odd leading dimensions on a large problem: the library repacks A and B into aligned
    workspace and runs the TMA kernel -- same bits as the same shape given aligned inputs."""
    M, N, K = 1200, 1201, 1501            # odd N and K -> odd lda, ldb when packed
    A, B, C0 = synth.problem(M, N, K, seed=19)
    C_odd = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5)
    Ap = np.zeros((M, K + 1)); Ap[:, :K] = A
    Bp = np.zeros((K, N + 1)); Bp[:, :N] = B
    dA, dB, dC = dev(Ap), dev(Bp), dev(C0)
    cuda_lib.gemm(dA[:, :K], dB[:, :N], dC, 1.5, 0.5)
    torch.cuda.synchronize()
    assert np.array_equal(C_odd, dC.cpu().numpy())
    rows = _rows(M, extra=4)
    ref, mag = oracle.dgemm(1.5, A[rows], B, 0.5, C0[rows], want_mag=True)
    r = oracle.check(C_odd[rows], ref, oracle.bound(K, 1.5, 0.5, mag, C0[rows]))
    assert r.ok, str(r)


def test_argument_errors_enqueue_nothing(cuda_lib):
    G = cuda_lib
    C = torch.full((8, 8), 7.0, dtype=torch.float64, device="cuda")
    A = torch.ones((8, 8), dtype=torch.float64, device="cuda")
    rc = G.gemm_raw(8, 8, 8, 1.0, A.data_ptr(), 4, A.data_ptr(), 8, 0.0, C.data_ptr(), 8)
    assert rc == G.GEMM_ERR_ARG and "lda" in G.last_error()
    rc = G.gemm_raw(8, 8, 8, 1.0, A.data_ptr(), 8, A.data_ptr(), 8, 0.0, A.data_ptr(), 8)
    assert rc == G.GEMM_ERR_ARG and "overlap" in G.last_error()
    rc = G.gemm_raw(-1, 8, 8, 1.0, A.data_ptr(), 8, A.data_ptr(), 8, 0.0, C.data_ptr(), 8)
    assert rc == G.GEMM_ERR_ARG and "M=" in G.last_error()
    rc = G.gemm_raw(8, 8, 8, 1.0, A.data_ptr(), 8, A.data_ptr(), 8, 0.0, C.data_ptr(), 8, cfg=10 ** 6)
    assert rc == G.GEMM_ERR_ARG and "cfg_id" in G.last_error()
    torch.cuda.synchronize()
    assert torch.all(C == 7.0)


# ---------------------------------------------------------------- inputs
@pytest.mark.parametrize("mode", list(synth.MODES))
def test_device_generator_matches_synth_bitwise(cuda_lib, mode):
    rows, cols = 301, 129
    X = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    cuda_lib.fill(X, mode, 1706, 1)
    torch.cuda.synchronize()
    assert np.array_equal(X.cpu().numpy(), synth.matrix(mode, 1706, 1, rows, cols))
    slab = torch.empty((50, cols), dtype=torch.float64, device="cuda")
    cuda_lib.fill(slab, mode, 1706, 1, rows=rows, row0=100)
    torch.cuda.synchronize()
    assert np.array_equal(slab.cpu().numpy(), synth.matrix(mode, 1706, 1, rows, cols, row0=100, nrows=50))


# ---------------------------------------------------------------- sizes of config 2 / 3
def _sampled_rows_check(G, M, N, K, alpha, beta, rows, mode="uniform", seed=1706):
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    G.fill(dA, mode, seed, synth.MAT_A)
    G.fill(dB, mode, seed, synth.MAT_B)
    G.fill(dC, mode, seed, synth.MAT_C)
    G.gemm(dA, dB, dC, alpha, beta)
    torch.cuda.synchronize()
    B = synth.matrix(mode, seed, synth.MAT_B, K, N)
    A_r = np.vstack([synth.matrix(mode, seed, synth.MAT_A, M, K, row0=r, nrows=1) for r in rows])
    C0_r = np.vstack([synth.matrix(mode, seed, synth.MAT_C, M, N, row0=r, nrows=1) for r in rows])
    ref, mag = oracle.dgemm(alpha, A_r, B, beta, C0_r, want_mag=True)
    got = dC[torch.tensor(rows, device="cuda")].cpu().numpy()
    res = oracle.check(got, ref, oracle.bound(K, alpha, beta, mag, C0_r))
    assert res.ok, f"rows {rows}: {res}"
    del dA, dB, dC
    torch.cuda.empty_cache()
    return res.max_ratio


def _rows(M, bm=128, extra=8, seed=0):
    rng = np.random.default_rng(seed)
    s = {0, M - 1, bm - 1, bm, M // 2, M - bm} | set(int(x) for x in rng.integers(0, M, extra))
    return sorted(r for r in s if 0 <= r < M)


@pytest.mark.parametrize("n", [1024, 2048])
def test_config2_full_oracle(cuda_lib, n):
    A, B, C0 = synth.problem(n, n, n, seed=1706)
    C = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0)
    check_vs_oracle(C, A, B, C0, 1.0, 0.0)


def test_config3_n8192_alpha_beta_sampled_rows(cuda_lib):
    _sampled_rows_check(cuda_lib, 8192, 8192, 8192, 1.5, 0.5, _rows(8192, extra=6))


def test_config3_every_cfg_sampled_rows(cuda_lib):
    """Config 3 (N=8192, alpha=1.5, beta=0.5): every grid point of the tuning sweep
    (tools/sweep.py tune times them) passes sampled-row parity."""
    n = 8192
    dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
    dB = torch.empty((n, n), dtype=torch.float64, device="cuda")
    dC = torch.empty((n, n), dtype=torch.float64, device="cuda")
    cuda_lib.fill(dA, "uniform", 1706, 0)
    cuda_lib.fill(dB, "uniform", 1706, 1)
    rows = _rows(n, extra=3)
    B = synth.matrix("uniform", 1706, 1, n, n)
    A_r = np.vstack([synth.matrix("uniform", 1706, 0, n, n, row0=r, nrows=1) for r in rows])
    C0_r = np.vstack([synth.matrix("uniform", 1706, 2, n, n, row0=r, nrows=1) for r in rows])
    ref, mag = oracle.dgemm(1.5, A_r, B, 0.5, C0_r, want_mag=True)
    bnd = oracle.bound(n, 1.5, 0.5, mag, C0_r)
    idx = torch.tensor(rows, device="cuda")
    for info in cuda_lib.cfgs():
        cuda_lib.fill(dC, "uniform", 1706, 2)
        cuda_lib.gemm(dA, dB, dC, 1.5, 0.5, cfg=info["id"])
        torch.cuda.synchronize()
        res = oracle.check(dC[idx].cpu().numpy(), ref, bnd)
        assert res.ok, (info["name"], str(res))
    del dA, dB, dC
    torch.cuda.empty_cache()


def test_config2_n16384_sampled_rows_bench_launch(cuda_lib):
    """The bench workload (16384^3, alpha=1, beta=0, heuristic config = bench launch)."""
    _sampled_rows_check(cuda_lib, 16384, 16384, 16384, 1.0, 0.0, _rows(16384, extra=4))


def test_n16384_dyadic_sampled_rows_bitwise(cuda_lib):
    M = N = K = 16384
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    for X, m in ((dA, 0), (dB, 1), (dC, 2)):
        cuda_lib.fill(X, "dyadic", 7, m)
    cuda_lib.gemm(dA, dB, dC, 1.5, 0.5)
    torch.cuda.synchronize()
    B = synth.matrix("dyadic", 7, 1, K, N)
    rows = _rows(M, extra=2)
    A_r = np.vstack([synth.matrix("dyadic", 7, 0, M, K, row0=r, nrows=1) for r in rows])
    C0_r = np.vstack([synth.matrix("dyadic", 7, 2, M, N, row0=r, nrows=1) for r in rows])
    ref = oracle.dgemm(1.5, A_r, B, 0.5, C0_r)
    assert np.array_equal(dC[torch.tensor(rows, device="cuda")].cpu().numpy(), ref)
    del dA, dB, dC
    torch.cuda.empty_cache()


def test_config4_row_sharded_p8_equals_full(cuda_lib):
    """Config 4 (M=32768, N=K=4096) row-sharded over P=8 ranks, run rank by rank on one GPU:
    every rank's shard equals the same rows of the unsharded GEMM bitwise (no split-K)."""
    M, N, K = 32768, 4096, 4096
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    cuda_lib.fill(dA, "uniform", 1706, 0)
    cuda_lib.fill(dB, "uniform", 1706, 1)
    cuda_lib.gemm(dA, dB, dC, 1.0, 0.0, splits=1)
    for r in range(8):
        r0, r1 = cuda_lib.row_range(M, r, 8)
        part = torch.empty((r1 - r0, N), dtype=torch.float64, device="cuda")
        cuda_lib.gemm(dA[r0:r1], dB, part, 1.0, 0.0, splits=1)
        torch.cuda.synchronize()
        assert torch.equal(part, dC[r0:r1]), r
    torch.cuda.synchronize()
    rows = _rows(M, bm=4096, extra=4)
    B = synth.matrix("uniform", 1706, 1, K, N)
    A_r = np.vstack([synth.matrix("uniform", 1706, 0, M, K, row0=r, nrows=1) for r in rows])
    ref, mag = oracle.dgemm(1.0, A_r, B, 0.0, np.zeros((len(rows), N)), want_mag=True)
    res = oracle.check(dC[torch.tensor(rows, device="cuda")].cpu().numpy(), ref, oracle.bound(K, 1.0, 0.0, mag, None))
    assert res.ok, str(res)
    del dA, dB, dC
    torch.cuda.empty_cache()


def test_config5_one_rank_shard_sampled(cuda_lib):
    """Config 5 at full size for one rank of the 8-GPU weak-scaled run: 8192 rows of the
    N=65536 problem (A 4 GiB, B 32 GiB, C 4 GiB), checked on sampled rows x a 512-column
    block against the oracle (the largest shape the library is run on)."""
    M, N, K = 8192, 65536, 65536
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    cuda_lib.fill(dA, "uniform", 1706, 0, rows=65536, row0=0)
    cuda_lib.fill(dB, "uniform", 1706, 1)
    cuda_lib.gemm(dA, dB, dC, 1.0, 0.0)
    torch.cuda.synchronize()
    c0, nc = 40960, 512
    rows = [0, 1, 255, 256, 4095, 8191]
    B = synth.matrix("uniform", 1706, 1, K, N, col0=c0, ncols=nc)
    A_r = np.vstack([synth.matrix("uniform", 1706, 0, 65536, K, row0=r, nrows=1) for r in rows])
    ref, mag = oracle.dgemm(1.0, A_r, B, 0.0, np.zeros((len(rows), nc)), want_mag=True)
    got = dC[torch.tensor(rows, device="cuda")][:, c0:c0 + nc].cpu().numpy()
    res = oracle.check(got, ref, oracle.bound(K, 1.0, 0.0, mag, None))
    assert res.ok, str(res)
    del dA, dB, dC
    torch.cuda.empty_cache()


def _rows_block_vs_oracle(G, dA, dB, dC, M, N, K, rows, c0, nc, seed, alpha, beta, mode="uniform"):
    B = synth.matrix(mode, seed, 1, K, N, col0=c0, ncols=nc)
    A_r = np.vstack([synth.matrix(mode, seed, 0, M, K, row0=r, nrows=1) for r in rows])
    C0 = np.vstack([synth.matrix(mode, seed, 2, M, N, row0=r, nrows=1, col0=c0, ncols=nc) for r in rows])
    ref, mag = oracle.dgemm(alpha, A_r, B, beta, C0, want_mag=True)
    got = dC[torch.tensor(rows, device="cuda")][:, c0:c0 + nc].cpu().numpy()
    res = oracle.check(got, ref, oracle.bound(K, alpha, beta, mag, C0))
    assert res.ok, str(res)
    return res


def test_max_size_c_beyond_2_31_elements(cuda_lib):
    """Element offsets past 2^31: C is 65600 x 32800 (2.15e9 entries, 17 GB), ragged in both
    tile dimensions, so rows near the end address C at 64-bit offsets in the epilogue; the
    plan's own kernel, alpha = 1.5, beta = 0.5, last rows and a ragged right-edge block checked
    against the oracle."""
    M, N, K, seed = 65600, 32800, 40, 61
    assert M * N > 2 ** 31
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    for X, mat in ((dA, 0), (dB, 1), (dC, 2)):
        cuda_lib.fill(X, "uniform", seed, mat)
    cuda_lib.gemm(dA, dB, dC, 1.5, 0.5)
    torch.cuda.synchronize()
    rows = [0, 32767, 32768, 65535, 65536, 65599]
    _rows_block_vs_oracle(cuda_lib, dA, dB, dC, M, N, K, rows, N - 300, 300, seed, 1.5, 0.5)
    _rows_block_vs_oracle(cuda_lib, dA, dB, dC, M, N, K, rows, 0, 256, seed, 1.5, 0.5)
    del dA, dB, dC
    torch.cuda.empty_cache()


def test_max_size_k_beyond_2_20(cuda_lib):
    """Long K: 136 x 200 x (2^20 + 24) (tens of thousands of k-steps per tile, ragged K tail),
    with the product's plan and with split-K and cluster split-K forced, sampled rows against
    the oracle; and an all-ones problem of the same K must give K exactly in every entry."""
    M, N, K, seed = 136, 200, 2 ** 20 + 24, 62
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    for cfg, S in ((None, None), (cuda_lib.cfg_id("tma_64x64x32_w32x16_s3_splitk"), 16),
                   (cuda_lib.cfg_id("tma_64x64x32_w32x16_s3_csplit"), 8)):
        for X, mat in ((dA, 0), (dB, 1), (dC, 2)):
            cuda_lib.fill(X, "uniform", seed, mat)
        cuda_lib.gemm(dA, dB, dC, 1.5, 0.5, cfg=cfg, splits=S)
        torch.cuda.synchronize()
        _rows_block_vs_oracle(cuda_lib, dA, dB, dC, M, N, K, [0, 67, 135], 0, N, seed, 1.5, 0.5)
    dA.fill_(1.0)
    dB.fill_(1.0)
    cuda_lib.gemm(dA, dB, dC, 1.0, 0.0)
    torch.cuda.synchronize()
    assert bool((dC == float(K)).all())
    del dA, dB, dC
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- host entry point (e2e)
def test_host_entry_point(cuda_lib):
    A, B, C0 = synth.problem(700, 650, 300, seed=4)
    C = C0.copy()
    cuda_lib.gemm_host(A, B, C, 1.5, 0.5)
    check_vs_oracle(C, A, B, C0, 1.5, 0.5)
    # same bits as the device entry point without split-K (row panels do not change
    # per-entry arithmetic)
    assert np.array_equal(C, run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, splits=1))


def test_host_entry_point_large_pinned(cuda_lib):
    M, N, K = 5000, 3000, 1000
    A, B, C0 = synth.problem(M, N, K, seed=11)
    tA = torch.from_numpy(A).pin_memory()
    tB = torch.from_numpy(B).pin_memory()
    tC = torch.from_numpy(C0.copy()).pin_memory()
    cuda_lib.gemm_host(tA, tB, tC, 1.0, 1.0)
    assert np.array_equal(tC.numpy(), run_gpu(cuda_lib, A, B, C0, 1.0, 1.0, splits=1))
    rows = _rows(M, extra=4)
    ref, mag = oracle.dgemm(1.0, A[rows], B, 1.0, C0[rows], want_mag=True)
    r = oracle.check(tC.numpy()[rows], ref, oracle.bound(K, 1.0, 1.0, mag, C0[rows]))
    assert r.ok, str(r)


def test_host_entry_point_searched_geometry(cuda_lib):
    """A shape whose block geometry comes from the copy/compute simulation's search rather than
    the wave-fill rule (8192 x 4096 x 4096: 1024-row panels, one-block thin last panel): the
    result is still bitwise the one-pass device call's, and within the bound."""
    M, N, K = 8192, 4096, 4096
    A, B, C0 = synth.problem(M, N, K, seed=19)
    tA = torch.from_numpy(A).pin_memory()
    tB = torch.from_numpy(B).pin_memory()
    tC = torch.from_numpy(C0.copy()).pin_memory()
    cuda_lib.gemm_host(tA, tB, tC, 1.5, 0.5)
    assert np.array_equal(tC.numpy(), run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, splits=1))
    rows = _rows(M, extra=4)
    ref, mag = oracle.dgemm(1.5, A[rows], B, 0.5, C0[rows], want_mag=True)
    r = oracle.check(tC.numpy()[rows], ref, oracle.bound(K, 1.5, 0.5, mag, C0[rows]))
    assert r.ok, str(r)


def test_host_entry_point_pipelined_odd_padded(cuda_lib):
    """The blocked copy/compute pipeline (row panel 0 by column blocks, later row panels,
    last panel by column blocks) on an odd shape with padded host leading dimensions."""
    M, N, K = 6003, 1001, 2002
    A, B, C0 = synth.problem(M, N, K, seed=17)
    Ap = np.full((M, K + 3), np.nan); Ap[:, :K] = A
    Bp = np.full((K, N + 1), np.nan); Bp[:, :N] = B
    Cp = np.full((M, N + 5), np.nan); Cp[:, :N] = C0
    cuda_lib.gemm_host(Ap[:, :K], Bp[:, :N], Cp[:, :N], 1.5, 0.5)
    assert np.all(np.isnan(Cp[:, N:]))
    assert np.array_equal(Cp[:, :N], run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, splits=1))
    rows = _rows(M, extra=6)
    ref, mag = oracle.dgemm(1.5, A[rows], B, 0.5, C0[rows], want_mag=True)
    r = oracle.check(Cp[rows, :N], ref, oracle.bound(K, 1.5, 0.5, mag, C0[rows]))
    assert r.ok, str(r)


# ---------------------------------------------------------------- sharded (1 GPU, NCCL world=1)
@pytest.mark.parametrize("chunks", [1, 3])
def test_sharded_world1_equals_single_gpu(cuda_lib, chunks):
    M, N, K = 400, 520, 300
    A, B, C0 = synth.problem(M, N, K, seed=12)
    comm = cuda_lib.Comm(0, 1)
    dA, dB, dC = dev(A), dev(B), dev(C0)
    comm.gemm_sharded(dA, dB, dC, 1.5, 0.5, root=0, bcast_chunks=chunks)
    torch.cuda.synchronize()
    comm.close()
    assert np.array_equal(dC.cpu().numpy(), run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, splits=1))


def test_fake_multi_gpu_row_partition(cuda_lib):
    """The P-rank row partition run sequentially on one GPU equals the full GEMM bitwise
    (isolates partition/offset bugs from communication)."""
    M, N, K = 1001, 300, 257
    A, B, C0 = synth.problem(M, N, K, seed=13)
    full = run_gpu(cuda_lib, A, B, C0, 1.0, 1.0, splits=1)
    for P in (2, 3, 8):
        out = np.empty_like(full)
        for r in range(P):
            r0, r1 = cuda_lib.row_range(M, r, P)
            out[r0:r1] = run_gpu(cuda_lib, A[r0:r1], B, C0[r0:r1], 1.0, 1.0, splits=1)
        assert np.array_equal(out, full), P


# ---------------------------------------------------------------- microbenchmark
def test_peak_probe_runs(cuda_lib):
    out = torch.zeros(148, dtype=torch.float64, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    cuda_lib.peak_probe("dmma", 148, 8, 1000, out, cyc)
    cuda_lib.peak_probe("dfma", 148, 8, 1000, out, cyc)
    torch.cuda.synchronize()
    assert int(cyc.item()) > 0


# ---------------------------------------------------------------- CUDA graphs
def test_cuda_graph_capture_and_replay(cuda_lib):
    """The C-ABI calls are capturable after a warm-up call on the stream (workspace and tensor
    maps exist): a graph of 20 small GEMMs (split-K plan, config-1 size) replays with the same
    bits as eager launches."""
    n = 256
    A, B, C0 = synth.problem(n, n, n, seed=21)
    dA, dB = dev(A), dev(B)
    outs = [torch.zeros((n, n), dtype=torch.float64, device="cuda") for _ in range(20)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cuda_lib.gemm(dA, dB, outs[0], 1.0, 0.0)     # warm-up: workspace, plan, tensor maps
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for o in outs:
            cuda_lib.gemm(dA, dB, o, 1.0, 0.0)
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    eager = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0)
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), eager)


def test_cuda_graph_survives_workspace_growth(cuda_lib):
    """a graph captured from a split-K call keeps pointing at the workspace it was
    captured with.  A later eager call that needs a LARGER workspace on the same stream must
    not free it (it is retired, not freed), so replaying the graph afterwards still gives the
    eager bits; gemm_workspace_release() then frees everything and eager calls still work."""
    n = 256
    A, B, C0 = synth.problem(n, n, n, seed=22)
    dA, dB = dev(A), dev(B)
    out = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    sk = cuda_lib.cfg_id("tma_64x64x32_w32x16_s3_splitk")
    with torch.cuda.stream(s):
        cuda_lib.gemm(dA, dB, out, 1.0, 0.0, cfg=sk, splits=4)      # warm-up (workspace for 256^3 x4)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cuda_lib.gemm(dA, dB, out, 1.0, 0.0, cfg=sk, splits=4)
    # a much larger split-K call on the capture stream grows the workspace (old buffer retired)
    big = 2048
    bA = torch.ones((big, big), dtype=torch.float64, device="cuda")
    bC = torch.zeros((big, big), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        cuda_lib.gemm(bA, bA, bC, 1.0, 0.0, cfg=sk, splits=8)
        torch.empty((big, big), dtype=torch.float64, device="cuda").fill_(np.nan)   # reuse freed memory, if any
    torch.cuda.synchronize()
    assert float(bC[7, 9]) == big
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    eager = run_gpu(cuda_lib, A, B, C0, 1.0, 0.0, cfg=sk, splits=4)
    assert np.array_equal(out.cpu().numpy(), eager)
    del g
    cuda_lib.workspace_release()
    assert np.array_equal(run_gpu(cuda_lib, A, B, C0, 1.0, 0.0, cfg=sk, splits=4), eager)


# ---------------------------------------------------------------- hybrid (row a5)
HYBRID_SHAPES = [
    (1024, 2368, 64),     # T = 148 tiles = one full wave, no tail
    (1024, 2496, 32),     # tail of 8 tiles, KT = 2 < 16: one whole tile per tail CTA, no fix-up
    (1000, 2500, 1000),   # W = 1 + 12 cut tail tiles, ragged M / N / K
    (300, 200, 2000),     # W = 0: pure stream-K over 8 tiles
    (256, 64, 16),        # one tile, one k-step
    (520, 130, 778),
]


@pytest.mark.parametrize("shape", HYBRID_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_hybrid_within_bound_deterministic(cuda_lib, shape):
    """Persistent data-parallel waves + stream-K tail + fix-up: every wave/tail layout."""
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=M + K)
    hyb = cuda_lib.cfg_id("tma_256x64x16_w64x32_s4_hybrid")
    C = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=hyb)
    check_vs_oracle(C, A, B, C0, 1.5, 0.5)
    assert np.array_equal(C, run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=hyb))
    # tiles not cut by the tail carry the plain one-pass chain: identical to the XP kernel
    xp = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cuda_lib.cfg_id("tma_256x64x16_w64x32_s4_xp"))
    G_ = torch.cuda.get_device_properties(0).multi_processor_count
    tn = (N + 63) // 64
    T = ((M + 255) // 256) * tn
    full = T - T % G_ if T >= G_ else 0
    rows_done = np.zeros((M, N), dtype=bool)
    for bid in range(full):          # grouped raster, group_m = 8 (tile_coords)
        per = 8 * tn
        grp, r = divmod(bid, per)
        gs = min(8, (M + 255) // 256 - grp * 8)
        tm, tnn = grp * 8 + r % gs, r // gs
        rows_done[tm * 256:(tm + 1) * 256, tnn * 64:(tnn + 1) * 64] = True
    assert np.array_equal(C[rows_done], xp[rows_done])


def test_hybrid_exact_regime_bitwise(cuda_lib):
    A, B, C0 = synth.problem(1000, 2500, 1000, mode="dyadic", seed=12)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    hyb = cuda_lib.cfg_id("tma_256x64x16_w64x32_s4_hybrid")
    assert np.array_equal(run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=hyb), ref)


@pytest.mark.parametrize("shape", [(1000, 2500, 1000), (300, 200, 2000), (1024, 1024, 1024)],
                         ids=lambda s: "x".join(map(str, s)))
def test_hybrid_every_cfg_exact_regime_bitwise(cuda_lib, shape):
    """Every hybrid configuration (incl. the E = 8 32x64 tiles, whose fix-up CTAs take 2 quads
    instead of 4) against the oracle bit for bit in the exact regime, cut tail tiles included."""
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, mode="dyadic", seed=M + 7)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    hybs = [c["id"] for c in cuda_lib.cfgs() if c["split_k"] == -2]
    assert len(hybs) >= 4
    for cfg in hybs:
        assert np.array_equal(run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg), ref), cuda_lib.cfg_name(cfg)


def _tile_coords(bid, tiles_m, tiles_n, group_m=8):
    per = group_m * tiles_n
    grp, r = divmod(bid, per)
    gs = min(group_m, tiles_m - grp * group_m)
    return grp * group_m + r % gs, r // gs


@pytest.mark.parametrize("shape", [(16384, 4096, 4096), (7168, 7168, 7168)], ids=lambda s: "x".join(map(str, s)))
def test_hybrid_plan_full_size_tail_rows(cuda_lib, shape):
    """Full-size shapes through the hybrid schedule (config-4 2-GPU shard, the f1 grid; the
    product's plan for some shapes): rows through the stream-K tail tiles (cut between CTAs,
    finished by the fix-up kernel) and through data-parallel tiles, checked against the oracle."""
    M, N, K = shape
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float64, device="cuda")
    hyb = cuda_lib.cfg_id("tma_256x64x16_w64x32_s4_hybrid")
    cuda_lib.fill(dA, "uniform", 1706, 0)
    cuda_lib.fill(dB, "uniform", 1706, 1)
    cuda_lib.fill(dC, "uniform", 1706, 2)
    cuda_lib.gemm(dA, dB, dC, 1.5, 0.5, cfg=hyb)
    torch.cuda.synchronize()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    tm_n, tn_n = (M + 255) // 256, (N + 63) // 64
    T = tm_n * tn_n
    tail = list(range(T - T % sms, T))
    assert tail, "shape has no tail"
    tail_rows = sorted({_tile_coords(b, tm_n, tn_n)[0] * 256 + o for b in tail[::max(1, len(tail) // 3)]
                        for o in (0, 255)})
    rows = sorted(set(tail_rows) | {0, M // 3})
    B = synth.matrix("uniform", 1706, 1, K, N)
    A_r = np.vstack([synth.matrix("uniform", 1706, 0, M, K, row0=r, nrows=1) for r in rows])
    C0_r = np.vstack([synth.matrix("uniform", 1706, 2, M, N, row0=r, nrows=1) for r in rows])
    ref, mag = oracle.dgemm(1.5, A_r, B, 0.5, C0_r, want_mag=True)
    res = oracle.check(dC[torch.tensor(rows, device="cuda")].cpu().numpy(), ref, oracle.bound(K, 1.5, 0.5, mag, C0_r))
    assert res.ok, f"rows {rows}: {res}"
    del dA, dB, dC
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg_name,splits", [("tma_64x64x16_w32x16_s6_splitk", 2), ("tma_64x64x16_w32x16_s6_splitk", 4),
                                             ("tma_64x64x32_w32x16_s3_splitk", 4), ("tma_64x64x32_w32x16_s3_hybrid", None),
                                             ("tma_64x64x16_w32x16_s6", None), ("tma_256x64x16_w64x32_s4_xp", None),
                                             ("tma_64x64x16_w32x16_s6_hybrid", None),
                                             ("tma_128x64x16_w32x16_s6_streamk", None),
                                             ("tma_64x64x32_w32x16_s3_csplit", 4), ("tma_64x64x16_w32x16_s6_csplit", 8),
                                             ("tma_32x64x32_w16x16_s3_splitk", 2), ("tma_32x64x64_w16x16_s3_splitk", 1),
                                             ("tma_64x32x32_w16x16_s4_splitk", 3), ("tma_32x32x32_w16x16_s4_splitk", 4),
                                             ("tma_32x64x32_w16x16_s3", None),
                                             ])
def test_ring_slot_reuse_exact_k_signature(cuda_lib, cfg_name, splits):
    """Regression for the ring's write-after-read hazard (DESIGN.md §6 "Releasing a slot"):
    with A = ones and B[k][j] = k + 1, every C entry is exactly K(K+1)/2, and a warp that read
    a slot after its refill would add STAGES*16 to some k (the error the race produced).
    Many CTAs, two per SM, every k-step through the ring: 2048^3."""
    n = 2048
    A = torch.ones((n, n), dtype=torch.float64, device="cuda")
    B = torch.arange(1, n + 1, dtype=torch.float64, device="cuda")[:, None].expand(n, n).contiguous()
    for _ in range(3):
        C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        cuda_lib.gemm(A, B, C, 1.0, 0.0, cfg=cuda_lib.cfg_id(cfg_name), splits=splits)
        torch.cuda.synchronize()
        bad = int((C != n * (n + 1) / 2).sum())
        assert bad == 0, (cfg_name, splits, bad)


# ---------------------------------------------------------------- cluster split-K (row a5)
def cluster_cfgs(G):
    return [c["id"] for c in G.cfgs() if c["split_k"] == -3]


@pytest.mark.parametrize("shape", [(64, 64, 64), (256, 256, 256), (130, 1000, 96), (1024, 1024, 1024), (520, 390, 1000),
                                   (33, 18, 778)], ids=lambda s: "x".join(map(str, s)))
def test_cluster_split_k_equals_global_split_k_bitwise(cuda_lib, shape):
    """Cluster split-K sums the S slice partials in slice order through distributed shared
    memory -- the same order as the global-memory split-K -- so for every S <= 8 the bits equal
    the *_splitk kernel of the same tile with the same S (uniform inputs, alpha=1.5, beta=0.5),
    and the result is within the bound and repeatable."""
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=M + 2 * N + K)
    pairs = {"tma_64x64x32_w32x16_s3_csplit": "tma_64x64x32_w32x16_s3_splitk",
             "tma_64x64x16_w32x16_s6_csplit": "tma_64x64x16_w32x16_s6_splitk"}
    for cname, gname in pairs.items():
        c, g = cuda_lib.cfg_id(cname), cuda_lib.cfg_id(gname)
        kt = -(-K // cuda_lib.cfg_info(c)["bk"])
        for S in (1, 2, 3, 4, 5, 8):
            if S > kt:
                continue
            got = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=c, splits=S)
            ref = run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=g, splits=S)
            assert np.array_equal(got, ref), (cname, S)
            assert np.array_equal(got, run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=c, splits=S)), (cname, S)
        check_vs_oracle(got, A, B, C0, 1.5, 0.5)


def test_cluster_split_k_exact_regime_every_cfg(cuda_lib):
    A, B, C0 = synth.problem(700, 650, 1300, mode="dyadic", seed=9)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    for cfg in cluster_cfgs(cuda_lib):
        for S in (2, 4, 7, 8, 16):   # 16 is clamped to the portable cluster size 8
            assert np.array_equal(run_gpu(cuda_lib, A, B, C0, 1.5, 0.5, cfg=cfg, splits=S), ref), \
                (cuda_lib.cfg_name(cfg), S)


# ---------------------------------------------------------------- TMA staging variants (a2)
_MD_SCRIPT = r"""
import sys, hashlib, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import synth
from paper_1706_10086_b200 import gemm as G
out = []
for (M, N, K, cfg, S) in [(1024, 1024, 1024, None, None), (640, 768, 512, "tma_64x64x32_w32x16_s3_splitk", 3),
                          (2048, 1536, 1024, "tma_64x64x32_w32x16_s3_hybrid", None),
                          (700, 1024, 2048, "tma_128x64x16_w32x16_s6_streamk", None),
                          (512, 512, 4096, "tma_64x64x32_w32x16_s3_csplit", 4),
                          (256, 1024, 512, "tma_256x64x16_w64x32_s4_xp", None)]:
    A, B, C0 = synth.problem(M, N, K, seed=M + K)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C0))
    G.gemm(dA, dB, dC, 1.5, 0.5, cfg=None if cfg is None else G.cfg_id(cfg), splits=S)
    torch.cuda.synchronize()
    out.append(hashlib.sha256(dC.cpu().numpy().tobytes()).hexdigest())
print(",".join(out))
"""


def test_multidim_tensor_maps_equal_2d_boxes_bitwise(cuda_lib):
    """K and N multiples of 16 stage A and B with one 3-D / 4-D TMA box per stage instead of
    KG * (1 + BN/16) 2-D boxes; the shared-memory image is the same, so every kernel family
    (data-parallel, split-K, hybrid, stream-K, cluster split-K, XP) must give the same bits
    with GEMM_TMA_MD=0 (2-D boxes forced) as with the default."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = []
    for md in ("1", "0"):
        env = dict(os.environ, GEMM_TMA_MD=md)
        p = subprocess.run([sys.executable, "-c", _MD_SCRIPT, root], capture_output=True, text=True, env=env,
                           timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        runs.append(p.stdout.strip().splitlines()[-1])
    assert runs[0] == runs[1]
