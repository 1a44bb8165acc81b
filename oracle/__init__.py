"""CPU oracle for C = alpha*A*B + beta*C (Eq. (1)) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1706_10086_b200``) never imports it and shares no code
with it; if the CUDA library is missing the product fails loudly instead of
falling back here.

Contents
--------
``dgemm``        ctypes wrapper of ``oracle_dgemm.c`` (plain i-k-j triple loop,
                 ascending k, no FMA, threads over rows; see its header).
``bound``        the elementwise acceptance bound of BASELINE.json's north
                 star, generalised for alpha/beta:
                   4*K*u*|alpha|*mag + 4*u*|beta|*|C0| + 1e-300,  u = 2^-53
``check``        err/bound report: max ratio, worst index, NaN handling.
``freivalds``    full-coverage exact check of a large result in O(N^2) host work:
                 (alpha*A*B + beta*C0) x = alpha*A*(B x) + beta*C0 x for random 0/1
                 matrices x (Eq. (1) applied to vectors; Freivalds' test).  Bitwise
                 only in the exact (dyadic / small-integer) input regime.

Parity pins for every function here live in ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_dgemm.c")
_LIB = os.path.join(_HERE, "liboracle_dgemm.so")

U = 2.0 ** -53


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FMA contraction, no fast-math.  The library is
    written to a per-process temporary name and renamed into place, so ranks of a multi-GPU
    run that build concurrently never load a half-written file."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        f = lib.oracle_dgemm
        i64, dbl, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        f.argtypes = [i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp, i64, ctypes.c_int]
        f.restype = ctypes.c_int
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def _ptr(x):
    return None if x is None else x.ctypes.data


def dgemm(alpha: float, A: np.ndarray, B: np.ndarray, beta: float, C0: np.ndarray,
          want_mag: bool = False, nthreads: int | None = None):
    """Return alpha*A@B + beta*C0 computed by the oracle (and the magnitude if asked).

    A: (M, K), B: (K, N), C0: (M, N); any float64 2-D arrays whose last axis is
    contiguous (row-major with a leading dimension = row stride).
    """
    A = _rowmajor(A)
    B = _rowmajor(B)
    C = np.array(C0, dtype=np.float64, order="C", copy=True)
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or C.shape != (M, N):
        raise ValueError(f"shape mismatch A{A.shape} B{B.shape} C{C.shape}")
    mag = np.zeros((M, N), dtype=np.float64) if want_mag else None
    rc = _load().oracle_dgemm(M, N, K, float(alpha),
                              _ptr(A), _ld(A, K), _ptr(B), _ld(B, N),
                              float(beta), _ptr(C), _ld(C, N),
                              _ptr(mag), N if mag is not None else 0,
                              int(nthreads or default_threads()))
    if rc != 0:
        raise RuntimeError(f"oracle_dgemm failed with code {rc}")
    return (C, mag) if want_mag else C


def _rowmajor(X):
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if X.shape[0] == 0 or X.shape[1] == 0:
        return np.ascontiguousarray(X)
    if X.strides[1] != 8 or X.strides[0] % 8 != 0 or X.strides[0] < 8 * X.shape[1]:
        X = np.ascontiguousarray(X)
    return X


def _ld(X, cols):
    if X.shape[0] <= 1 or X.shape[1] == 0:
        return max(1, cols)
    return X.strides[0] // 8


def bound(K: int, alpha: float, beta: float, mag: np.ndarray, C0: np.ndarray | None) -> np.ndarray:
    """Elementwise acceptance bound (BASELINE.json north_star)."""
    b = 4.0 * K * U * abs(alpha) * mag + 1e-300
    if beta != 0.0 and C0 is not None:
        b = b + 4.0 * U * abs(beta) * np.abs(C0)
    return b


U32 = 2.0 ** -23   # fp32 unit roundoff allowing directed (truncating) rounding in the accumulator


def bound_f32(K: int, alpha: float, beta: float, mag: np.ndarray, C0: np.ndarray | None) -> np.ndarray:
    """Elementwise bound for the single-precision (3xTF32) path, reading R16:
    (4K + 8) u32 |alpha| mag + 4 u32 |beta| |C0| + 1e-30, u32 = 2^-23.
    4K u32 mag covers the K-term recursive FP32 accumulation of three tf32 product passes
    with a possibly truncating accumulator; 8 u32 mag covers the 3xTF32 representation
    error (dropped lo*lo term and the two tf32 roundings, <= 3 * 2^-22 |a||b|)."""
    b = (4.0 * K + 8.0) * U32 * abs(alpha) * mag + 1e-30
    if beta != 0.0 and C0 is not None:
        b = b + 4.0 * U32 * abs(beta) * np.abs(C0)
    return b


@dataclass
class CheckResult:
    ok: bool
    max_ratio: float
    worst: tuple
    n_bad: int
    n_nan: int
    median_rel: float

    def __str__(self):
        return (f"ok={self.ok} max err/bound={self.max_ratio:.3e} at {self.worst} "
                f"bad={self.n_bad} nan={self.n_nan} median rel err={self.median_rel:.3e}")


def check(C_test: np.ndarray, C_ref: np.ndarray, bnd: np.ndarray) -> CheckResult:
    """Compare elementwise; a NaN anywhere in C_test or C_ref (not both) fails."""
    C_test = np.asarray(C_test, dtype=np.float64)
    C_ref = np.asarray(C_ref, dtype=np.float64)
    if C_test.shape != C_ref.shape:
        raise ValueError(f"shape mismatch {C_test.shape} vs {C_ref.shape}")
    if C_test.size == 0:
        return CheckResult(True, 0.0, (), 0, 0, 0.0)
    err = np.abs(C_test - C_ref)
    both_nan = np.isnan(C_test) & np.isnan(C_ref)
    same_inf = np.isinf(C_test) & (C_test == C_ref)
    err = np.where(both_nan | same_inf, 0.0, err)
    nan = np.isnan(err)
    ratio = np.where(nan, np.inf, err / bnd)
    bad = ratio > 1.0
    idx = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
    denom = np.maximum(np.abs(C_ref), 1e-300)
    rel = np.where(nan, np.inf, err / denom)
    return CheckResult(bool(not bad.any()), float(ratio[idx]), tuple(int(v) for v in idx),
                       int(bad.sum()), int(nan.sum()), float(np.median(rel)))


def freivalds(alpha: float, beta: float, X: np.ndarray, M: int, K: int, a_rows, b_rows, c_rows, c0_rows=None,
              chunk: int = 1024) -> np.ndarray:
    """Rows i of a candidate C (M x n) with C x != alpha*A*(B x) + beta*C0 x, for the n x v
    0/1 matrix X -- Eq. (1) applied to the columns of X.  Every product is formed
    on row chunks supplied by callables (the matrices need not fit in memory at once):
        a_rows(r0, nr)  -> A[r0:r0+nr, :]     (nr x K)
        b_rows(k0, nk)  -> B[k0:k0+nk, cols]  (nk x n)
        c_rows(r0, nr)  -> C_test[r0:r0+nr, cols]
        c0_rows(r0, nr) -> C0[r0:r0+nr, cols] (read only when beta != 0)
    The comparison is bitwise, so it is valid only where every partial sum is exactly
    representable: dyadic inputs m/256 (|m| <= 256) with K, n <= 2^16 keep B x below 2^24
    in units of 2^-8 and A (B x), C x below 2^48 in units of 2^-16 (alpha = 1.5 adds one
    bit), so any summation order gives the same doubles and a correct C passes exactly.
    A wrong row i is missed by one random 0/1 column with probability <= 1/2 (Freivalds),
    by v independent columns with probability <= 2^-v.  Returns the sorted bad row indices."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    BX = np.zeros((K, X.shape[1]))
    for k0 in range(0, K, chunk):
        nk = min(chunk, K - k0)
        BX[k0:k0 + nk] = b_rows(k0, nk) @ X
    bad = []
    for r0 in range(0, M, chunk):
        nr = min(chunk, M - r0)
        rhs = alpha * (a_rows(r0, nr) @ BX)
        if beta != 0.0:
            rhs = rhs + beta * (c0_rows(r0, nr) @ X)
        lhs = c_rows(r0, nr) @ X
        rows = np.nonzero(np.any(lhs != rhs, axis=1))[0]
        bad.extend((r0 + rows).tolist())
    return np.asarray(bad, dtype=np.int64)
