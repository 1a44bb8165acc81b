"""f4: the same GEMM on CUDA managed (unified) memory -- PAPER.md P:216 (§2.2: the GPU runs
use unified memory for some measurements) and P:892 (§4: "all GPUs show a better performance
when using unified memory instead of device memory, especially for small N").  Managed
pointers are ordinary device pointers to the library (TMA descriptors included), so the
product path is unchanged; these tests pin that it computes the right result in the three
ways managed memory gets populated:
  device   : cudaMallocManaged, inputs written by the GPU (first touch on the device);
  host     : written by the CPU, pages migrate on demand during the first launch;
  prefetch : written by the CPU, then cudaMemPrefetchAsync to the GPU before the launch.
Checks: the whole result against the CPU oracle within the north-star bound (uniform inputs,
alpha = 1.5, beta = 0.5), and every entry of a 2048^3 dyadic product by Freivalds (bitwise).
"""

import ctypes

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rt = pytest.importorskip("cuda.bindings.runtime")


def _ok(res):
    err = res[0] if isinstance(res, tuple) else res
    assert err == rt.cudaError_t.cudaSuccess, err
    return res[1] if isinstance(res, tuple) and len(res) > 1 else None


class Managed:
    def __init__(self, rows, cols):
        self.rows, self.cols = rows, cols
        self.ptr = int(_ok(rt.cudaMallocManaged(max(8, 8 * rows * cols), rt.cudaMemAttachGlobal)))

    def host(self):
        return np.ctypeslib.as_array((ctypes.c_double * (self.rows * self.cols)).from_address(self.ptr)).reshape(
            self.rows, self.cols)

    def free(self):
        _ok(rt.cudaFree(self.ptr))


def _populate(G, bufs, mats, mode, kind, seed):
    """Write the inputs into managed buffers the way `mode` says."""
    for buf, (mat, rows, cols) in zip(bufs, mats):
        if mode == "device":
            rc = G.lib().gemm_fill_f64(G.FILL_MODES[kind], seed, mat, rows, cols, 0, rows, buf.ptr, cols, 0)
            assert rc == 0, G.last_error()
        else:
            buf.host()[:] = synth.matrix(kind, seed, mat, rows, cols)
    torch.cuda.synchronize()
    if mode == "prefetch":
        dev = torch.cuda.current_device()
        for buf in bufs:
            _ok(rt.cudaMemPrefetchAsync(buf.ptr, 8 * buf.rows * buf.cols, dev, 0))
        torch.cuda.synchronize()


def _gemm(G, M, N, K, alpha, beta, a, b, c):
    rc = G.gemm_raw(M, N, K, alpha, a.ptr, K, b.ptr, N, beta, c.ptr, N, -1, 0)
    assert rc == 0, G.last_error()
    torch.cuda.synchronize()


@pytest.mark.parametrize("mode", ["device", "host", "prefetch"])
@pytest.mark.parametrize("shape", [(640, 520, 384), (1024, 1024, 1024), (301, 257, 130)], ids=lambda s: "x".join(map(str, s)))
def test_managed_memory_vs_oracle(cuda_lib, mode, shape):
    G = cuda_lib
    M, N, K = shape
    seed = 77
    bufs = [Managed(M, K), Managed(K, N), Managed(M, N)]
    try:
        _populate(G, bufs, [(0, M, K), (1, K, N), (2, M, N)], mode, "uniform", seed)
        _gemm(G, M, N, K, 1.5, 0.5, *bufs)
        got = bufs[2].host().copy()
    finally:
        for b in bufs:
            b.free()
    A, B, C0 = (synth.matrix("uniform", seed, m, r, c) for m, r, c in ((0, M, K), (1, K, N), (2, M, N)))
    ref, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    r = oracle.check(got, ref, oracle.bound(K, 1.5, 0.5, mag, C0))
    assert r.ok, f"{mode} {shape}: {r}"
    assert r.max_ratio < 0.05


@pytest.mark.parametrize("mode", ["device", "host", "prefetch"])
def test_managed_memory_dyadic_every_entry(cuda_lib, mode):
    """2048^3 on managed buffers, dyadic inputs: every entry by Freivalds (bitwise)."""
    G = cuda_lib
    n, seed = 2048, 78
    bufs = [Managed(n, n), Managed(n, n), Managed(n, n)]
    try:
        _populate(G, bufs, [(0, n, n), (1, n, n), (2, n, n)], mode, "dyadic", seed)
        _gemm(G, n, n, n, 1.5, 0.5, *bufs)
        C = bufs[2].host().copy()
    finally:
        for b in bufs:
            b.free()
    A, B, C0 = (synth.matrix("dyadic", seed, m, n, n) for m in (0, 1, 2))
    X = np.random.default_rng(seed).integers(0, 2, size=(n, 16)).astype(np.float64)
    rows = lambda Mx: (lambda r0, nr: Mx[r0:r0 + nr])  # noqa: E731
    bad = oracle.freivalds(1.5, 0.5, X, n, n, rows(A), rows(B), rows(C), rows(C0))
    assert bad.size == 0, f"{mode}: wrong rows {bad[:8].tolist()}"
