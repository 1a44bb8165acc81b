"""GPU parity of the single-precision (3xTF32 tcgen05) path, against the fp64
CPU oracle on fp32 inputs (exactly representable in fp64) within oracle.bound_f32 (DESIGN.md
reading R16); bitwise in the exact small-integer regime."""

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def run(G, A, B, C0, alpha, beta):
    dA, dB, dC = (torch.from_numpy(f32(x)).cuda() for x in (A, B, C0))
    G.gemm_f32(dA, dB, dC, alpha, beta)
    torch.cuda.synchronize()
    return dC.cpu().numpy().astype(np.float64)


def check(G, M, N, K, alpha, beta, seed=1, mode="uniform"):
    A, B, C0 = (f32(x).astype(np.float64) for x in synth.problem(M, N, K, mode=mode, seed=seed))
    got = run(G, A, B, C0, alpha, beta)
    ref, mag = oracle.dgemm(alpha, A, B, beta, C0, want_mag=True)
    r = oracle.check(got, ref, oracle.bound_f32(K, alpha, beta, mag, C0))
    assert r.ok, f"{M}x{N}x{K}: {r}"
    return r, got, ref


@pytest.mark.parametrize("shape", [(128, 128, 32), (256, 256, 256), (1, 1, 1), (7, 5, 3), (130, 300, 77),
                                   (513, 257, 1000), (1024, 1024, 1024), (64, 2000, 33)],
                         ids=lambda s: "x".join(map(str, s)))
def test_f32_uniform_within_bound(cuda_lib, shape):
    r, _, _ = check(cuda_lib, *shape, 1.5, 0.5)
    assert r.max_ratio < 0.5


def test_f32_accuracy_is_fp32_class(cuda_lib):
    """3xTF32 must be far more accurate than plain tf32: on this problem 1xTF32 (exact
    accumulation of tf32-rounded operands) has median relative error 6.8e-4, a sequential
    FP32 loop 6.3e-7 (computed on the host, R16).  The tensor-core path must stay
    within 20x of FP32 and >= 50x better than 1xTF32."""
    r, got, ref = check(cuda_lib, 512, 512, 2048, 1.0, 0.0, seed=3)
    assert r.median_rel < 20 * 6.3e-7, r


def test_f32_exact_integer_regime_bitwise(cuda_lib):
    """Small integers are tf32-exact (lo = 0) and every partial sum < 2^24 is exact in fp32:
    the tensor-core result must equal the oracle bit for bit."""
    A, B, C0 = synth.problem(300, 260, 1000, mode="int8", seed=2)
    got = run(cuda_lib, A, B, C0, 1.5, 0.5)
    ref = oracle.dgemm(1.5, A, B, 0.5, C0)
    assert np.array_equal(got, ref)


def test_f32_special_cases(cuda_lib):
    C0 = f32(synth.matrix("uniform", 1, 2, 40, 50))
    A = np.full((40, 30), np.nan, dtype=np.float32)
    B = np.full((30, 50), np.nan, dtype=np.float32)
    assert np.array_equal(run(cuda_lib, A, B, C0, 0.0, 2.0), (2.0 * C0).astype(np.float64))
    A, B, _ = synth.problem(40, 50, 30, seed=5)
    got = run(cuda_lib, A, B, np.full((40, 50), np.nan), 1.0, 0.0)
    assert np.all(np.isfinite(got))


def test_f32_padded_and_deterministic(cuda_lib):
    M, N, K = 200, 150, 90
    A, B, C0 = (f32(x) for x in synth.problem(M, N, K, seed=8))
    Ap = np.full((M, K + 3), np.nan, np.float32); Ap[:, :K] = A
    Bp = np.full((K, N + 1), np.nan, np.float32); Bp[:, :N] = B
    Cp = np.full((M, N + 5), np.nan, np.float32); Cp[:, :N] = C0
    outs = []
    for _ in range(2):
        dA, dB, dC = (torch.from_numpy(x.copy()).cuda() for x in (Ap, Bp, Cp))
        cuda_lib.gemm_f32(dA[:, :K], dB[:, :N], dC[:, :N], 1.5, 0.5)
        torch.cuda.synchronize()
        outs.append(dC.cpu().numpy())
    assert np.array_equal(outs[0], outs[1], equal_nan=True)
    assert np.all(np.isnan(outs[0][:, N:]))
    ref, mag = oracle.dgemm(1.5, A.astype(np.float64), B.astype(np.float64), 0.5, C0.astype(np.float64), want_mag=True)
    r = oracle.check(outs[0][:, :N].astype(np.float64), ref, oracle.bound_f32(K, 1.5, 0.5, mag, C0.astype(np.float64)))
    assert r.ok, str(r)


def test_f32_large_sampled_rows(cuda_lib):
    M = N = K = 8192
    dA = torch.empty((M, K), dtype=torch.float64, device="cuda")
    dB = torch.empty((K, N), dtype=torch.float64, device="cuda")
    cuda_lib.fill(dA, "uniform", 1706, 0)
    cuda_lib.fill(dB, "uniform", 1706, 1)
    a32, b32 = dA.float(), dB.float()
    del dA, dB
    c32 = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    cuda_lib.gemm_f32(a32, b32, c32, 1.0, 0.0)
    torch.cuda.synchronize()
    rows = [0, 1, 127, 128, 4095, 8191]
    B = f32(synth.matrix("uniform", 1706, 1, K, N)).astype(np.float64)
    A = np.vstack([f32(synth.matrix("uniform", 1706, 0, M, K, row0=r, nrows=1)).astype(np.float64) for r in rows])
    ref, mag = oracle.dgemm(1.0, A, B, 0.0, np.zeros((len(rows), N)), want_mag=True)
    got = c32[torch.tensor(rows, device="cuda")].cpu().numpy().astype(np.float64)
    r = oracle.check(got, ref, oracle.bound_f32(K, 1.0, 0.0, mag, None))
    assert r.ok, str(r)


@pytest.mark.parametrize("shape", [(130, 300, 77), (256, 512, 1000), (1, 1, 1)], ids=lambda s: "x".join(map(str, s)))
def test_f32_every_cfg_within_bound(cuda_lib, shape):
    M, N, K = shape
    A, B, C0 = (f32(x).astype(np.float64) for x in synth.problem(M, N, K, seed=M + K))
    ref, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    bnd = oracle.bound_f32(K, 1.5, 0.5, mag, C0)
    for cfg in range(len(cuda_lib.f32_cfg_names())):
        dA, dB, dC = (torch.from_numpy(f32(x)).cuda() for x in (A, B, C0))
        cuda_lib.gemm_f32(dA, dB, dC, 1.5, 0.5, cfg=cfg)
        torch.cuda.synchronize()
        r = oracle.check(dC.cpu().numpy().astype(np.float64), ref, bnd)
        assert r.ok, (cuda_lib.f32_cfg_names()[cfg], str(r))
