"""Pins for the CPU oracle (oracle/) against things other than itself.

Each test names what fixes the expected value: a worked example printed in
SPEC.md (tests/golden/), exact rational arithmetic, a closed form of
C = alpha*A*B + beta*C (Eq. (1)), the exact dyadic regime in
which every summation order yields the same double, or an invariant
(transposition, beta-linearity, thread count).  A dropped term, a wrong sign, a
transposed operand, a swapped leading dimension, alpha applied per product
instead of once, or beta applied to the wrong thing fails at least one of them.
"""

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def _mat(v):
    if isinstance(v, str):
        kind, n = v[:-1], int(v[-1])
        return np.eye(n) if kind == "identity" else np.zeros((n, n))
    return np.array([[float(x) for x in row] for row in v], dtype=np.float64)


@pytest.mark.parametrize("case", json.load(open(GOLDEN))["cases"], ids=lambda c: c["name"])
def test_worked_examples(case):
    """SPEC.md worked examples + hand-derived ones, bit for bit."""
    A, B, C0, C = (_mat(case[k]) for k in ("A", "B", "C0", "C"))
    got = oracle.dgemm(case["alpha"], A, B, case["beta"], C0)
    assert np.array_equal(got, C), (case["name"], got, C)


def _exact(alpha, A, B, beta, C0):
    M, K = A.shape
    N = B.shape[1]
    out = [[None] * N for _ in range(M)]
    mag = [[None] * N for _ in range(M)]
    for i in range(M):
        for j in range(N):
            s = sum((Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(K)), Fraction(0))
            m = sum((abs(Fraction(A[i, k])) * abs(Fraction(B[k, j])) for k in range(K)), Fraction(0))
            out[i][j] = Fraction(alpha) * s + Fraction(beta) * Fraction(C0[i, j])
            mag[i][j] = m
    return out, mag


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 2), (5, 3, 7), (6, 6, 6), (2, 7, 8), (8, 1, 5)])
@pytest.mark.parametrize("ab", [(1.0, 0.0), (1.5, 0.5), (-0.75, 2.0)])
def test_bruteforce_exact_rational(shape, ab):
    """Brute force in exact rational arithmetic: |oracle - exact| <= (2 K u |alpha| mag + 2u|beta||C0|)(1+small).

    The textbook bound for a recursive sum of K rounded products is gamma_K*sum|a||b|,
    gamma_K = K u/(1 - K u); the alpha product, beta product and final add contribute
    at most a few more u.  A wrong index/sign/term gives errors O(|a||b|) >> this.
    """
    M, N, K = shape
    alpha, beta = ab
    rng = np.random.default_rng(hash((shape, ab)) & 0xFFFF)
    A = rng.uniform(-1, 1, (M, K)) * 10.0 ** rng.integers(-3, 4, (M, K))
    B = rng.uniform(-1, 1, (K, N)) * 10.0 ** rng.integers(-3, 4, (K, N))
    C0 = rng.uniform(-1, 1, (M, N))
    got = oracle.dgemm(alpha, A, B, beta, C0)
    ex, mag = _exact(alpha, A, B, beta, C0)
    u = Fraction(1, 2 ** 53)
    for i in range(M):
        for j in range(N):
            err = abs(Fraction(got[i, j]) - ex[i][j])
            gam = (K + 2) * u / (1 - (K + 2) * u)
            lim = gam * abs(Fraction(alpha)) * mag[i][j] * (1 + 2 * u) \
                + 3 * u * abs(Fraction(beta) * Fraction(C0[i, j])) + 2 * u * abs(ex[i][j])
            assert err <= lim, (i, j, float(err), float(lim))


def test_k1_is_correctly_rounded_product():
    """K=1, alpha=1, beta=0: each entry is the correctly rounded exact product a*b."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((9, 1)) * 1e5
    B = rng.standard_normal((1, 11)) * 1e-7
    got = oracle.dgemm(1.0, A, B, 0.0, np.full((9, 11), np.nan))
    for i in range(9):
        for j in range(11):
            assert got[i, j] == float(Fraction(A[i, 0]) * Fraction(B[0, j]))


def test_identity_A_gives_B():
    B = synth.matrix("uniform", 3, synth.MAT_B, 37, 29)
    got = oracle.dgemm(1.0, np.eye(37), B, 0.0, np.zeros((37, 29)))
    assert np.array_equal(got, B)


@pytest.mark.parametrize("K", [1, 17, 1000])
def test_all_ones_gives_K(K):
    got = oracle.dgemm(1.0, np.ones((5, K)), np.ones((K, 7)), 0.0, np.zeros((5, 7)))
    assert np.all(got == float(K))


def test_alpha_zero_gives_beta_C_without_reading_AB():
    C0 = synth.matrix("uniform", 4, synth.MAT_C, 6, 9)
    A = np.full((6, 5), np.nan)
    B = np.full((5, 9), np.inf)
    got = oracle.dgemm(0.0, A, B, -1.25, C0)
    assert np.array_equal(got, -1.25 * C0)


def test_k_zero_gives_beta_C():
    C0 = synth.matrix("uniform", 5, synth.MAT_C, 4, 3)
    got = oracle.dgemm(2.0, np.zeros((4, 0)), np.zeros((0, 3)), 0.5, C0)
    assert np.array_equal(got, 0.5 * C0)
    got0 = oracle.dgemm(2.0, np.zeros((4, 0)), np.zeros((0, 3)), 0.0, np.full((4, 3), np.nan))
    assert np.array_equal(got0, np.zeros((4, 3)))


def test_beta_zero_does_not_read_C():
    A, B, _ = synth.problem(5, 6, 7, seed=9)
    got = oracle.dgemm(1.0, A, B, 0.0, np.full((5, 6), np.nan))
    assert np.all(np.isfinite(got))


def test_transpose_invariance_bitwise():
    """(A B)^T = B^T A^T: the oracle forms the same products in the same k order -> same bits."""
    A, B, _ = synth.problem(23, 31, 19, seed=11)
    C = oracle.dgemm(1.0, A, B, 0.0, np.zeros((23, 31)))
    Ct = oracle.dgemm(1.0, np.ascontiguousarray(B.T), np.ascontiguousarray(A.T), 0.0, np.zeros((31, 23)))
    assert np.array_equal(C.T, Ct)


@pytest.mark.parametrize("mode", ["dyadic", "int8"])
def test_exact_regime_equals_any_order(mode):
    """Dyadic (multiples of 2^-8) or small-integer inputs: every partial sum is exact, so
    the oracle must equal numpy's BLAS matmul (a different summation order) bit for bit,
    and alpha=1.5/beta=0.5 stay exact too."""
    A, B, C0 = synth.problem(45, 38, 300, mode=mode, seed=2)
    got = oracle.dgemm(1.5, A, B, 0.5, C0)
    ref = 1.5 * (A @ B) + 0.5 * C0
    assert np.array_equal(got, ref)


def test_beta_linearity_integer_inputs():
    """gemm(alpha, beta) == alpha*gemm(1, 0) + beta*C0 exactly on integer inputs."""
    A, B, C0 = synth.problem(12, 10, 40, mode="int8", seed=5)
    lhs = oracle.dgemm(3.0, A, B, -2.0, C0)
    rhs = 3.0 * oracle.dgemm(1.0, A, B, 0.0, np.zeros_like(C0)) + (-2.0) * C0
    assert np.array_equal(lhs, rhs)


def test_alpha_applied_once_on_sum():
    """Reading R5: alpha multiplies the rounded sum, not each product.  Chosen so the two differ."""
    A = np.array([[1.0, 1.0, 1.0]])
    B = np.array([[0.1], [0.2], [0.3]])
    alpha = 3.0
    got = oracle.dgemm(alpha, A, B, 0.0, np.zeros((1, 1)))[0, 0]
    once = alpha * ((0.1 + 0.2) + 0.3)
    per_product = ((alpha * 0.1) + (alpha * 0.2)) + (alpha * 0.3)
    assert once != per_product
    assert got == once


def test_numpy_crosscheck_within_bound():
    A, B, C0 = synth.problem(70, 90, 257, seed=1)
    got, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    ref = 1.5 * (A @ B) + 0.5 * C0
    r = oracle.check(ref, got, oracle.bound(257, 1.5, 0.5, mag, C0))
    assert r.ok, str(r)
    assert r.max_ratio < 0.05


def test_magnitude_closed_form():
    """mag = |A| |B| (a sum of non-negative terms; exact on integer inputs)."""
    A, B, _ = synth.problem(9, 8, 50, mode="int8", seed=3)
    _, mag = oracle.dgemm(1.0, A, B, 0.0, np.zeros((9, 8)), want_mag=True)
    assert np.array_equal(mag, np.abs(A) @ np.abs(B))


def test_thread_count_invariance():
    A, B, C0 = synth.problem(101, 67, 129, seed=4)
    r1 = oracle.dgemm(1.5, A, B, 0.5, C0, nthreads=1)
    r8 = oracle.dgemm(1.5, A, B, 0.5, C0, nthreads=8)
    assert np.array_equal(r1, r8)


def test_row_slab_equals_rows_of_full_result():
    """Sampled-row parity relies on this: rows computed alone equal the same rows of the full product."""
    A, B, C0 = synth.problem(40, 33, 65, seed=6)
    full = oracle.dgemm(1.0, A, B, 1.0, C0)
    slab = oracle.dgemm(1.0, A[17:23], B, 1.0, C0[17:23])
    assert np.array_equal(full[17:23], slab)


def test_strided_leading_dimensions():
    A, B, C0 = synth.problem(11, 13, 7, seed=8)
    Ap = np.full((11, 10), np.nan); Ap[:, :7] = A
    Bp = np.full((7, 20), np.nan); Bp[:, :13] = B
    got = oracle.dgemm(1.0, Ap[:, :7], Bp[:, :13], 0.0, np.zeros((11, 13)))
    ref = oracle.dgemm(1.0, A, B, 0.0, np.zeros((11, 13)))
    assert np.array_equal(got, ref)


def test_nan_localisation():
    """A NaN in A[i][k] poisons exactly row i of C (and nothing else)."""
    A, B, _ = synth.problem(8, 6, 5, seed=10)
    A[3, 2] = np.nan
    got = oracle.dgemm(1.0, A, B, 0.0, np.zeros((8, 6)))
    assert np.all(np.isnan(got[3]))
    assert np.all(np.isfinite(np.delete(got, 3, axis=0)))


# ---- the acceptance checker ------------------------------------------------

def _small_case():
    A, B, C0 = synth.problem(64, 64, 64, seed=1706)
    C, mag = oracle.dgemm(1.0, A, B, 0.0, C0, want_mag=True)
    return C, oracle.bound(64, 1.0, 0.0, mag, None)


def test_checker_rejects_perturbed_entry():
    C, bnd = _small_case()
    bad = C.copy()
    bad[5, 7] += 1e-6
    r = oracle.check(bad, C, bnd)
    assert not r.ok and r.worst == (5, 7) and r.n_bad == 1


def test_checker_accepts_last_bit_flip():
    C, bnd = _small_case()
    bad = C.copy()
    bad[5, 7] = np.nextafter(bad[5, 7], np.inf)
    assert oracle.check(bad, C, bnd).ok


def test_checker_rejects_nan():
    C, bnd = _small_case()
    bad = C.copy()
    bad[0, 0] = np.nan
    r = oracle.check(bad, C, bnd)
    assert not r.ok and r.n_nan == 1


def _beta_heavy_case(seed=41):
    """alpha=1.5, beta=0.5 with |C0| ~ 1e6 and |A||B| ~ 1e-6: the beta term dominates."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (24, 48)) * 1e-3
    B = rng.uniform(-1, 1, (48, 20)) * 1e-3
    C0 = rng.uniform(0.5, 1.0, (24, 20)) * 1e6 * rng.choice([-1.0, 1.0], (24, 20))
    C, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    return A, B, C0, C, mag


def test_bound_beta_term_rejects_error_far_above_rounding_of_beta_c0():
    """Fault injection at alpha=1.5, beta=0.5 (config 3): an error delta with
    u|beta||C0| << delta << |C0| must fail.  Here u|beta||C0| ~ 5e-11 and delta = 1e-4 while
    |C0| ~ 1e6: a bound whose beta term lost its u (4|beta||C0| ~ 2e6) would accept it."""
    A, B, C0, C, mag = _beta_heavy_case()
    bnd = oracle.bound(48, 1.5, 0.5, mag, C0)
    bad = C.copy()
    bad[3, 4] += 1e-4
    r = oracle.check(bad, C, bnd)
    assert not r.ok and r.worst == (3, 4) and r.n_bad == 1
    # ... and the unperturbed result, plus a last-bit flip of one entry, still pass
    assert oracle.check(C, C, bnd).ok
    flip = C.copy()
    flip[3, 4] = np.nextafter(flip[3, 4], np.inf)
    assert oracle.check(flip, C, bnd).ok


def test_bound_with_zero_a_is_the_beta_term_exactly():
    """A = 0 makes mag = 0, so the bound reduces to its beta term: 4 u |beta| |C0| + 1e-300
    (u = 2^-53, a power of two, so the expected value is computed exactly)."""
    _, B, C0, _, _ = _beta_heavy_case(seed=42)
    A = np.zeros((24, 48))
    C, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    assert np.all(mag == 0.0)
    expect = (np.abs(C0) * 0.5) * 2.0 ** -51 + 1e-300
    assert np.array_equal(oracle.bound(48, 1.5, 0.5, mag, C0), expect)
    assert np.array_equal(C, 0.5 * C0)   # beta*C0, exact (power-of-two scale)


@pytest.mark.parametrize("ab", [(1.5, 0.5), (-3.0, 2.0), (1.0, 0.0), (0.25, -8.0)])
def test_bound_is_bracketed_by_exact_rational_error(ab):
    """Two-sided pin of the whole bound against exact rational arithmetic (Fraction), at
    several alpha/beta: (lower) it is at least the oracle's true error, so a correct result
    never fails; (upper) it is at most 8x the textbook worst case gamma_K|alpha|mag +
    3u|beta||C0| + 2u|exact| (gamma_K = Ku/(1-Ku)), so a term that lost its u, a wrong K
    factor or a beta term scaled by something other than |beta| makes it too loose."""
    alpha, beta = ab
    rng = np.random.default_rng(7)
    M, N, K = 5, 6, 7
    A = rng.uniform(-1, 1, (M, K)) * 10.0 ** rng.integers(-2, 3, (M, K))
    B = rng.uniform(-1, 1, (K, N)) * 10.0 ** rng.integers(-2, 3, (K, N))
    C0 = rng.uniform(-1, 1, (M, N)) * 10.0 ** rng.integers(-2, 6, (M, N))
    got, mag = oracle.dgemm(alpha, A, B, beta, C0, want_mag=True)
    bnd = oracle.bound(K, alpha, beta, mag, C0)
    ex, exmag = _exact(alpha, A, B, beta, C0)
    u = Fraction(1, 2 ** 53)
    gam = K * u / (1 - K * u)
    for i in range(M):
        for j in range(N):
            err = abs(Fraction(got[i, j]) - ex[i][j])
            assert Fraction(bnd[i, j]) >= err, (i, j)
            worst = gam * abs(Fraction(alpha)) * exmag[i][j] + 3 * u * abs(Fraction(beta) * Fraction(C0[i, j])) \
                + 2 * u * abs(ex[i][j])
            assert Fraction(bnd[i, j]) <= 8 * worst + Fraction(1e-300), (i, j, float(bnd[i, j]), float(worst))


def test_bound_f32_beta_term_pins():
    """bound_f32 at alpha=1.5, beta=0.5 with mag = 0: exactly 4 u32 |beta||C0| + 1e-30
    (u32 = 2^-23), i.e. 2^-22 |C0| in [0.12, 0.24] for |C0| in [5e5, 1e6].  An error of 1.0
    fails and one of 0.0125 passes; a beta term that lost its u32 (~1e6) would pass both."""
    _, B, C0, _, _ = _beta_heavy_case(seed=43)
    mag = np.zeros_like(C0)
    b = oracle.bound_f32(48, 1.5, 0.5, mag, C0)
    assert np.array_equal(b, (np.abs(C0) * 0.5) * 2.0 ** -21 + 1e-30)   # 4 u32 = 2^-21
    ref = 0.5 * C0
    assert not oracle.check(ref + 1.0, ref, b).ok
    assert oracle.check(ref + 0.0125, ref, b).ok


def test_bound_is_tight_enough_to_catch_a_dropped_term():
    """Dropping one k term must exceed the bound (the bound is not vacuous)."""
    A, B, C0 = synth.problem(16, 16, 256, seed=12)
    C, mag = oracle.dgemm(1.0, A, B, 0.0, C0, want_mag=True)
    dropped = oracle.dgemm(1.0, A[:, :-1], B[:-1], 0.0, C0)
    r = oracle.check(dropped, C, oracle.bound(256, 1.0, 0.0, mag, None))
    assert not r.ok


# ---- the shared input generator ---------------------------------------------

def test_splitmix64_reference_vector():
    """synth's finaliser is SplitMix64: with base 0 the first counter value is the
    well-known first output of SplitMix64(seed=0), 0xE220A8397B1DCDAF."""
    z = np.array([0x9E3779B97F4A7C15], dtype=np.uint64)
    assert int(synth._mix(z)[0]) == 0xE220A8397B1DCDAF


def test_synth_uniform_range_and_determinism():
    X = synth.matrix("uniform", 1706, 0, 300, 200)
    assert X.min() >= -1.0 and X.max() < 1.0
    assert abs(X.mean()) < 0.01 and abs(X.var() - 1 / 3) < 0.01
    assert np.array_equal(X, synth.matrix("uniform", 1706, 0, 300, 200))
    assert not np.array_equal(X, synth.matrix("uniform", 1707, 0, 300, 200))
    assert not np.array_equal(X, synth.matrix("uniform", 1706, 1, 300, 200))


def test_synth_row_slab_consistency():
    full = synth.matrix("uniform", 3, 1, 50, 17)
    assert np.array_equal(full[20:31], synth.matrix("uniform", 3, 1, 50, 17, row0=20, nrows=11))


def test_synth_dyadic_values():
    X = synth.matrix("dyadic", 2, 0, 100, 100)
    assert np.all(X * 256 == np.round(X * 256)) and X.min() >= -1 and X.max() <= 1
    Y = synth.matrix("int8", 2, 0, 100, 100)
    assert np.all(Y == np.round(Y)) and Y.min() == -8 and Y.max() == 8


def test_synth_chunked_generation_is_identical():
    rows, cols = 700, 1000    # > 2 chunks of 2^18 elements
    for mode in ("uniform", "dyadic", "int8"):
        assert np.array_equal(synth.matrix(mode, 5, 1, rows, cols),
                              synth._matrix_block(mode, 5, 1, rows, cols, 0, rows))


def test_synth_column_block_consistency():
    full = synth.matrix("uniform", 3, 1, 40, 57)
    assert np.array_equal(full[5:17, 20:41], synth.matrix("uniform", 3, 1, 40, 57, row0=5, nrows=12, col0=20, ncols=21))
    eye = synth.matrix("identity", 0, 0, 9, 9)
    assert np.array_equal(eye[2:7, 3:8], synth.matrix("identity", 0, 0, 9, 9, row0=2, nrows=5, col0=3, ncols=5))


def test_bound_f32_catches_fp32_scale_errors():
    """The single-precision bound accepts an FP32 rounding of the fp64 oracle result and a
    one-ulp(fp32) perturbation, but rejects an error of one dropped k term."""
    A, B, C0 = synth.problem(32, 32, 512, seed=13)
    A, B, C0 = (x.astype(np.float32).astype(np.float64) for x in (A, B, C0))
    C, mag = oracle.dgemm(1.0, A, B, 0.0, C0, want_mag=True)
    bnd = oracle.bound_f32(512, 1.0, 0.0, mag, None)
    C32 = C.astype(np.float32).astype(np.float64)
    assert oracle.check(C32, C, bnd).ok
    assert oracle.check(np.nextafter(C32.astype(np.float32), np.float32(np.inf)).astype(np.float64), C, bnd).ok
    dropped = oracle.dgemm(1.0, A[:, :-1], B[:-1], 0.0, C0)
    assert not oracle.check(dropped, C, bnd).ok


# ---------------------------------------------------------------- Freivalds full-coverage check
def _freivalds_problem(M, N, K, seed=11, mode="dyadic"):
    A, B, C0 = synth.problem(M, N, K, mode=mode, seed=seed)
    X = np.random.default_rng(seed).integers(0, 2, size=(N, 16)).astype(np.float64)
    return A, B, C0, X


def _rows(Mx):
    return lambda r0, nr: Mx[r0:r0 + nr]


def test_freivalds_passes_exact_oracle_result():
    """Eq. (1) on vectors: the oracle's own exact-regime result satisfies
    C x == 1.5 A (B x) + 0.5 C0 x bitwise, with chunks that do not divide the sizes."""
    M, N, K = 150, 97, 130
    A, B, C0, X = _freivalds_problem(M, N, K)
    C = oracle.dgemm(1.5, A, B, 0.5, C0)
    bad = oracle.freivalds(1.5, 0.5, X, M, K, _rows(A), _rows(B), _rows(C), _rows(C0), chunk=37)
    assert bad.size == 0


def test_freivalds_names_a_row_off_by_one_unit():
    """One entry off by 2^-16 (the granularity of the exact products) is caught and only
    its row is reported."""
    M, N, K = 120, 80, 64
    A, B, C0, X = _freivalds_problem(M, N, K, seed=5)
    C = oracle.dgemm(1.0, A, B, 0.0, np.zeros((M, N)))
    C[77, 41] += 2.0 ** -16
    bad = oracle.freivalds(1.0, 0.0, X, M, K, _rows(A), _rows(B), _rows(C), chunk=50)
    assert bad.tolist() == [77]


def test_freivalds_catches_transposed_operand_and_dropped_beta():
    M = N = K = 64
    A, B, C0, X = _freivalds_problem(M, N, K, seed=9)
    wrong_t = oracle.dgemm(1.0, A, np.ascontiguousarray(B.T), 0.0, np.zeros((M, N)))
    assert oracle.freivalds(1.0, 0.0, X, M, K, _rows(A), _rows(B), _rows(wrong_t)).size > M // 2
    no_beta = oracle.dgemm(1.5, A, B, 0.0, np.zeros((M, N)))
    assert oracle.freivalds(1.5, 0.5, X, M, K, _rows(A), _rows(B), _rows(no_beta), _rows(C0)).size > M // 2
