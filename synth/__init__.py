"""Seeded synthetic matrix generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no products, no sums of
products, no alpha/beta).  It only turns (seed, matrix id, logical row,
logical column) into a double, with a counter-based generator, so that:

* the oracle tests (``oracle/``) and the GPU tests feed the SAME inputs;
* any row slab can be regenerated on the host without materialising the
  whole matrix (needed for sampled parity at N=16384/65536);
* the CUDA library carries its own implementation of the same counter-based
  generator (``gemm_fill_f64`` in ``include/gemm_f64.h``) for device-resident
  bench inputs, and a test checks the two bitwise.

Generator (SURVEY.md §8(d) "Concrete synthetic inputs"):

    mix(z)     = splitmix64 finaliser
                 z ^= z >> 30; z *= 0xBF58476D1CE4E5B9
                 z ^= z >> 27; z *= 0x94D049BB133111EB
                 z ^= z >> 31
    base       = mix(seed * 0x9E3779B97F4A7C15 + (mat + 1) * 0xD1B54A32D192ED03)
    r(i, j)    = mix(base + (i * cols + j + 1) * 0x9E3779B97F4A7C15)   (mod 2^64)

``i, j`` are LOGICAL indices into the full matrix (independent of the leading
dimension and of the row sharding), ``cols`` is the logical column count.

Modes (the value distribution):

* ``uniform``  : 2 * ((r >> 11) * 2^-53) - 1  -> uniform on [-1, 1), exact doubles
                 (the paper never states matrix contents)
* ``dyadic``   : ((r >> 11) % 513 - 256) / 256 -> multiples of 2^-8 in [-1, 1];
                 every partial sum of products is exact for K <= 2^19, so every
                 summation order gives the same bits (exact-arithmetic pin)
* ``int8``     : (r >> 11) % 17 - 8          -> integers in [-8, 8]
* ``ones``     : 1.0
* ``identity`` : 1.0 if i == j else 0.0
* ``zeros``    : 0.0
"""

from __future__ import annotations

import numpy as np

MODES = ("uniform", "dyadic", "int8", "ones", "identity", "zeros")
MODE_ID = {m: k for k, m in enumerate(MODES)}

# matrix ids used throughout (A=0, B=1, C0=2)
MAT_A, MAT_B, MAT_C = 0, 1, 2

DEFAULT_SEED = 1706

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MATK = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    z = z ^ (z >> np.uint64(31))
    return z


def _base(seed: int, mat: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.array([seed], dtype=np.uint64) * _GAMMA + np.uint64(mat + 1) * _MATK
        return _mix(z)[0]


def raw_bits(seed: int, mat: int, rows: int, cols: int, row0: int = 0, nrows: int | None = None,
             col0: int = 0, ncols: int | None = None) -> np.ndarray:
    """The raw 64-bit counter stream r(i, j) for rows [row0, row0+nrows), columns [col0, col0+ncols)."""
    if nrows is None:
        nrows = rows - row0
    if ncols is None:
        ncols = cols - col0
    if nrows < 0 or row0 < 0 or row0 + nrows > rows:
        raise ValueError(f"row slab [{row0},{row0 + nrows}) outside [0,{rows})")
    if ncols < 0 or col0 < 0 or col0 + ncols > cols:
        raise ValueError(f"column slab [{col0},{col0 + ncols}) outside [0,{cols})")
    with np.errstate(over="ignore"):
        i = np.arange(row0, row0 + nrows, dtype=np.uint64)[:, None]
        j = np.arange(col0, col0 + ncols, dtype=np.uint64)[None, :]
        ctr = i * np.uint64(cols) + j + np.uint64(1)
        return _mix(_base(seed, mat) + ctr * _GAMMA)


_CHUNK = 1 << 18   # elements per generation block (cache-resident temporaries)


def matrix(mode: str, seed: int, mat: int, rows: int, cols: int,
           row0: int = 0, nrows: int | None = None, col0: int = 0, ncols: int | None = None) -> np.ndarray:
    """Block [row0, row0+nrows) x [col0, col0+ncols) of the logical rows x cols matrix
    (default: whole rows), C-contiguous float64."""
    if mode not in MODE_ID:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    if nrows is None:
        nrows = rows - row0
    if ncols is None:
        ncols = cols - col0
    if mode in ("uniform", "dyadic", "int8") and nrows * ncols > 2 * _CHUNK and ncols > 0:
        # same values, generated in row blocks whose temporaries stay in cache
        out = np.empty((nrows, ncols), dtype=np.float64)
        step = max(1, _CHUNK // ncols)
        for r in range(0, nrows, step):
            n = min(step, nrows - r)
            out[r:r + n] = _matrix_block(mode, seed, mat, rows, cols, row0 + r, n, col0, ncols)
        return out
    return _matrix_block(mode, seed, mat, rows, cols, row0, nrows, col0, ncols)


def _matrix_block(mode, seed, mat, rows, cols, row0, nrows, col0=0, ncols=None):
    if ncols is None:
        ncols = cols - col0
    if mode == "ones":
        return np.ones((nrows, ncols), dtype=np.float64)
    if mode == "zeros":
        return np.zeros((nrows, ncols), dtype=np.float64)
    if mode == "identity":
        out = np.zeros((nrows, ncols), dtype=np.float64)
        for r in range(nrows):
            if col0 <= row0 + r < col0 + ncols:
                out[r, row0 + r - col0] = 1.0
        return out
    r = raw_bits(seed, mat, rows, cols, row0, nrows, col0, ncols) >> np.uint64(11)
    if mode == "uniform":
        return 2.0 * (r.astype(np.float64) * 2.0 ** -53) - 1.0
    if mode == "dyadic":
        return ((r % np.uint64(513)).astype(np.int64) - 256).astype(np.float64) / 256.0
    if mode == "int8":
        return ((r % np.uint64(17)).astype(np.int64) - 8).astype(np.float64)
    raise AssertionError(mode)


def problem(M: int, N: int, K: int, mode: str = "uniform", seed: int = DEFAULT_SEED,
            c_mode: str | None = None):
    """(A[M,K], B[K,N], C0[M,N]) for one seeded problem."""
    A = matrix(mode, seed, MAT_A, M, K)
    B = matrix(mode, seed, MAT_B, K, N)
    C0 = matrix(c_mode or mode, seed, MAT_C, M, N)
    return A, B, C0
