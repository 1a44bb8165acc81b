"""Run-time tuning of one shape (gemm_plan_autotune, include/gemm_f64.h): the pinned plan is
what the heuristic entry points launch afterwards, its results stay within the north-star
bound against the oracle, and the call refuses what it cannot do (capture, bad arguments).

Shapes are unique to this file (none is in tuned_b200.txt), so pinning them cannot change
the plan any other test exercises.
"""

import ctypes

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# unseen small shapes where the size model is furthest from the best plan
# (profiles/r02/regret_small_seed29_m3.csv, N and K rounded to even for the TMA path)
SHAPES = [(909, 522, 928), (1117, 572, 1004), (889, 240, 798), (206, 534, 386)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_autotune_pins_plan_and_matches_oracle(cuda_lib, shape):
    G = cuda_lib
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=M + 3 * N + 7 * K)
    dA, dB = dev(A), dev(B)
    cid, sp, sec = G.autotune(dA, dB, top=6)
    assert 0 <= cid < G.num_cfgs() and sp >= 1 and sec > 0.0
    assert G.plan(M, N, K, dA.data_ptr(), K, dB.data_ptr(), N) == (cid, sp)
    # the heuristic entry point now launches the pinned plan: bitwise equal to forcing it
    dC = dev(C0)
    G.gemm(dA, dB, dC, 1.5, 0.5)
    dF = dev(C0)
    G.gemm(dA, dB, dF, 1.5, 0.5, cfg=cid, splits=sp)
    torch.cuda.synchronize()
    assert torch.equal(dC, dF)
    C = dC.cpu().numpy()
    ref, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    r = oracle.check(C, ref, oracle.bound(K, 1.5, 0.5, mag, C0))
    assert r.ok, str(r)
    # A and B are only read
    assert np.array_equal(dA.cpu().numpy(), A) and np.array_equal(dB.cpu().numpy(), B)


def test_autotune_keeps_plan_in_force_when_it_is_among_the_fastest(cuda_lib):
    """top=1 times only the plan in force: it is returned unchanged."""
    G = cuda_lib
    M, N, K = 700, 650, 1236
    dA = torch.rand(M, K, dtype=torch.float64, device="cuda")
    dB = torch.rand(K, N, dtype=torch.float64, device="cuda")
    before = G.plan(M, N, K, dA.data_ptr(), K, dB.data_ptr(), N)
    cid, sp, sec = G.autotune(dA, dB, top=1)
    assert (cid, sp) == before and sec > 0.0


def test_autotune_non_tma_operands_return_heuristic_plan(cuda_lib):
    G = cuda_lib
    M, N, K = 301, 255, 133          # odd K and N: packed lda / ldb miss the TMA stride rule
    dA = torch.rand(M, K, dtype=torch.float64, device="cuda")
    dB = torch.rand(K, N, dtype=torch.float64, device="cuda")
    cid, sp, sec = G.autotune(dA, dB)
    assert (cid, sp) == G.plan(M, N, K, dA.data_ptr(), K, dB.data_ptr(), N)
    assert sec == 0.0 and not G.cfg_info(cid)["tma"]


def test_autotune_refuses_capture(cuda_lib):
    G = cuda_lib
    dA = torch.rand(256, 256, dtype=torch.float64, device="cuda")
    dB = torch.rand(256, 256, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        try:
            with pytest.raises(G.GemmError) as ei:
                G.autotune(dA, dB, stream=s)
        finally:
            g.capture_end()
    assert ei.value.code == G.GEMM_ERR_UNSUPPORTED


def test_autotune_argument_errors(cuda_lib):
    G = cuda_lib
    lib = G.lib()
    dA = torch.rand(64, 64, dtype=torch.float64, device="cuda")
    ci, dbl = ctypes.c_int, ctypes.c_double
    cid, sp, sec = ci(), ci(), dbl()
    p = dA.data_ptr()
    for (M, N, K, a, b, top) in [(0, 64, 64, p, p, 0), (64, 64, 0, p, p, 0), (64, 64, 64, 0, p, 0),
                                 (64, 64, 64, p, p, -1), (64, 64, 64, p, p, 65)]:
        rc = lib.gemm_plan_autotune(M, N, K, a, 64, b, 64, top, ctypes.byref(cid), ctypes.byref(sp),
                                    ctypes.byref(sec), None)
        assert rc == G.GEMM_ERR_ARG, (M, N, K, a, b, top, rc)
    assert lib.gemm_plan_autotune(64, 64, 64, p, 64, p, 64, 0, None, ctypes.byref(sp), None, None) == G.GEMM_ERR_ARG


_ENV_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth
from paper_1706_10086_b200 import gemm as G
M, N, K = {shape}
A, B, C0 = synth.problem(M, N, K, seed=5)
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
before = G.plan(M, N, K, dA.data_ptr(), K, dB.data_ptr(), N)
dC = torch.from_numpy(C0).cuda()
G.gemm(dA, dB, dC, 1.5, 0.5)                  # first heuristic call: autotunes, then launches
after = G.plan(M, N, K, dA.data_ptr(), K, dB.data_ptr(), N)
dF = torch.from_numpy(C0).cuda()
G.gemm(dA, dB, dF, 1.5, 0.5, cfg=after[0], splits=after[1])
torch.cuda.synchronize()
n = G.tune_save({saved!r})
np.savez({out!r}, C=dC.cpu().numpy(), same=np.array(torch.equal(dC, dF)), before=np.array(before),
         after=np.array(after), n=np.array(n))
"""


def test_env_autotune_on_first_use(cuda_lib, tmp_path):
    """GEMM_AUTOTUNE=1: the first heuristic call of an unpinned shape tunes and pins it; the
    result of that very call is the pinned plan's (bitwise) and within the bound; tune_save
    persists it beside the shipped table."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    shape = (1049, 624, 624)
    out, saved = str(tmp_path / "r.npz"), str(tmp_path / "saved.txt")
    code = _ENV_SCRIPT.format(root=root, shape=shape, out=out, saved=saved)
    env = dict(os.environ, GEMM_AUTOTUNE="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    r = np.load(out)
    assert bool(r["same"])
    M, N, K = shape
    A, B, C0 = synth.problem(M, N, K, seed=5)
    ref, mag = oracle.dgemm(1.5, A, B, 0.5, C0, want_mag=True)
    chk = oracle.check(r["C"], ref, oracle.bound(K, 1.5, 0.5, mag, C0))
    assert chk.ok, str(chk)
    lines = [l.split() for l in open(saved) if not l.startswith("#")]
    mine = [l for l in lines if tuple(map(int, l[:3])) == shape]
    assert len(mine) == 1 and int(mine[0][3]) == 1
    assert cuda_lib.cfg_id(mine[0][4]) == int(r["after"][0]) and int(mine[0][5]) == int(r["after"][1])
    assert int(r["n"]) == len(lines)


def test_autotune_repacked_operands(cuda_lib):
    """Odd leading dimensions on a problem large enough to be repacked: autotune times the
    TMA plan on packed copies and pins it under the TMA key, which the heuristic call (that
    repacks) then launches -- bitwise equal to forcing that plan on aligned copies."""
    G = cuda_lib
    M, N, K = 1201, 1203, 1501                   # 2MNK = 4.3e9 >= the repack threshold
    A, B, C0 = synth.problem(M, N, K, seed=77)
    dA, dB = dev(A), dev(B)                      # packed: lda = 1501, ldb = 1203 (odd)
    cid, sp, sec = G.autotune(dA, dB, top=4)
    assert sec > 0.0 and G.cfg_info(cid)["tma"]
    assert G.plan(M, N, K, 0, K + 1, 0, N + 1) == (cid, sp)
    dC = dev(C0)
    G.gemm(dA, dB, dC, 1.5, 0.5)
    aA = torch.empty((M, K + 1), dtype=torch.float64, device="cuda")[:, :K]
    aB = torch.empty((K, N + 1), dtype=torch.float64, device="cuda")[:, :N]
    aA.copy_(dA)
    aB.copy_(dB)
    aC = torch.empty((M, N + 1), dtype=torch.float64, device="cuda")[:, :N]
    aC.copy_(dev(C0))
    G.gemm(aA, aB, aC, 1.5, 0.5, cfg=cid, splits=sp)
    torch.cuda.synchronize()
    assert torch.equal(dC, aC)
    rows = [0, 1, 600, 1199, 1200]
    ref, mag = oracle.dgemm(1.5, A[rows], B, 0.5, C0[rows], want_mag=True)
    r = oracle.check(dC.cpu().numpy()[rows], ref, oracle.bound(K, 1.5, 0.5, mag, C0[rows]))
    assert r.ok, str(r)
