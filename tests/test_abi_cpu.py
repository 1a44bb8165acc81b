"""CPU-side checks of the C-ABI library (no GPU needed, no compute calls).

* the library builds for sm_100a and loads;
* it exports every symbol include/gemm_f64.h declares, and the binding knows them;
* the SASS of every GEMM kernel uses the FP64 tensor pipe (DMMA.8x8x4), TMA
  kernels issue UTMALDG, no kernel spills to local memory, and the epilogue has
  256-bit stores (the Listing-2 "disassembly inspection" analog);
* argument validation (runs before any CUDA call) rejects bad arguments with a
  message naming them, and the configuration registry is consistent.
"""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gemm_f64.h")


@pytest.fixture(scope="module")
def G():
    from paper_1706_10086_b200 import build
    build.build()
    from paper_1706_10086_b200 import gemm
    return gemm


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"GEMM_API\s+(?:const\s+)?\w+\s*\*?\s*(gemm_\w+)\s*\(", src)))


def test_header_declares_and_library_exports_every_symbol(G):
    decl = declared_symbols()
    assert len(decl) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", G.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(gemm_\w+)$", out, flags=re.M))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    assert set(decl) == set(G.EXPORTS)
    # nothing but the C ABI is exported (internal C++ symbols are hidden)
    assert all(s.startswith("gemm_") for s in exported)


def test_library_is_sm100a_only(G):
    out = subprocess.run(["cuobjdump", "--list-elf", G.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


@pytest.fixture(scope="module")
def sass(G):
    return subprocess.run(["cuobjdump", "-sass", G.LIB_PATH], capture_output=True, text=True, check=True).stdout


def _functions(sass):
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return {k: "\n".join(v) for k, v in funcs.items()}


def test_sass_gemm_kernels_use_dmma_tma_and_no_spills(sass):
    funcs = _functions(sass)
    gemm = {k: v for k, v in funcs.items() if "dgemm_" in k}
    assert gemm, "no GEMM kernels found"
    for name, body in gemm.items():
        assert not re.search(r"\b(LDL|STL)\b", body), f"local-memory spill in {name}"
        if "fixup" in name:          # hybrid tail reduction: loads partials, no MMA
            assert "STG.E.ENL2.256" in body, name
            continue
        assert "DMMA.8x8x4" in body, name
        if "dgemm_tma_kernel" in name or "dgemm_sktail_kernel" in name:
            assert "UTMALDG" in body, name
            assert "STG.E.ENL2.256" in body, name
        if "dgemm_generic_kernel" in name:
            assert "LDGSTS" in body, name


def test_ptxas_reports_no_spills(G):
    from paper_1706_10086_b200 import build
    for f in os.listdir(build.BUILD):
        if f.endswith(".ptxas.txt"):
            txt = open(os.path.join(build.BUILD, f)).read()
            for m in re.finditer(r"(\d+) bytes spill stores, (\d+) bytes spill loads", txt):
                assert m.group(1) == "0" and m.group(2) == "0", f


def test_cfg_registry(G):
    n = G.num_cfgs()
    assert n >= 5
    names = set()
    for info in G.cfgs():
        names.add(info["name"])
        assert info["bm"] % info["wm"] == 0 and info["bn"] % info["wn"] == 0
        assert info["threads"] == 32 * (info["bm"] // info["wm"]) * (info["bn"] // info["wn"])
        assert info["smem_bytes"] <= 227 * 1024
        stage = 8 * (info["bm"] + info["bn"]) * info["bk"]      # Eq. (5) analog: 2 tiles per stage
        assert info["smem_bytes"] >= info["stages"] * stage
        assert info["e"] == info["wm"] * info["wn"] // 32
        assert re.match(r"(tma|gen)_\d+x\d+x\d+_w\d+x\d+_s\d+", info["name"])
    assert len(names) == n
    # the paper's P100 optimum (16x16 threads x T=4 -> 64x64 block tile, E=16) is a grid point
    assert any(i["bm"] == 64 and i["bn"] == 64 and i["e"] == 16 for i in G.cfgs())
    with pytest.raises(G.GemmError):
        G.cfg_name(n)


def test_heuristic_selection(G):
    big = G.cfg_info(G.cfg_select(16384, 16384, 16384, 0, 16384, 0, 16384))
    assert big["tma"] == 1 and big["e"] >= 16
    # the tuned table (loaded by the binding) pins the measured best plan for the bench shape
    table = [ln.split() for ln in open(os.path.join(os.path.dirname(G.__file__), "tuned_b200.txt"))
             if ln.strip() and not ln.startswith("#")]
    pinned = [t[4] for t in table if t[:3] == ["16384", "16384", "16384"]]
    assert pinned and big["name"] == pinned[0]
    odd = G.cfg_info(G.cfg_select(1000, 1000, 1001, 0, 1001, 0, 1000))
    assert odd["tma"] == 0       # odd lda -> not TMA-eligible (2MNK < 4e9: not repacked)
    mis = G.cfg_info(G.cfg_select(512, 512, 512, 8, 512, 0, 512))
    assert mis["tma"] == 0       # 8-byte (not 16-byte) aligned A
    # large operands that miss the TMA rules are repacked by the call, which then launches the
    # TMA plan of the shape: that is the plan reported
    big_mis = G.cfg_info(G.cfg_select(4096, 4096, 4096, 8, 4096, 0, 4096))
    assert big_mis["tma"] == 1
    assert G.plan(4096, 4096, 4096, 8, 4096, 0, 4096) == G.plan(4096, 4096, 4096, 0, 4096, 0, 4096)


@pytest.mark.parametrize("args,needle", [
    ((-1, 4, 4, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "M=-1"),
    ((4, -1, 4, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "N=-1"),
    ((4, 4, -2, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "K=-2"),
    ((4, 4, 8, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "lda=4"),
    ((4, 8, 4, 1.0, 16, 4, 16, 4, 0.0, 16, 8), "ldb=4"),
    ((4, 8, 4, 1.0, 16, 4, 16, 8, 0.0, 16, 4), "ldc=4"),
    ((4, 4, 4, 1.0, 16, 4, 16, 4, 0.0, None, 4), "C is NULL"),
    ((4, 4, 4, 1.0, None, 4, 16, 4, 0.0, 4096, 4), "A is NULL"),
    ((4, 4, 4, 1.0, 16, 4, None, 4, 0.0, 4096, 4), "B is NULL"),
    ((4, 4, 4, 1.0, 12, 4, 16, 4, 0.0, 4096, 4), "A is not 8-byte aligned"),
    ((4, 4, 4, 1.0, 1024, 4, 4096, 4, 0.0, 1040, 4), "C overlaps A"),
    ((4, 4, 4, 1.0, 1024, 4, 4096, 4, 0.0, 4100 - 4, 4), "C overlaps B"),
    ((2 ** 31, 4, 4, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "< 2^31"),
    ((2 ** 31 - 100, 4, 4, 1.0, 16, 4, 16, 4, 0.0, 16, 4), "< 2^31"),
])
def test_argument_validation_messages(G, args, needle):
    rc = G.gemm_raw(*args)
    assert rc in (G.GEMM_ERR_ARG, G.GEMM_ERR_UNSUPPORTED)
    assert needle in G.last_error(), G.last_error()


def test_bad_cfg_id_rejected(G):
    rc = G.gemm_raw(4, 4, 4, 1.0, 16, 4, 16, 4, 0.0, 4096, 4, cfg=999)
    assert rc == G.GEMM_ERR_ARG and "cfg_id" in G.last_error()


def test_sharded_argument_validation(G):
    import ctypes
    lib = G.lib()
    rc = lib.gemm_f64_sharded(4, 4, 4, 1.0, 16, 4, 16, 4, 0.0, 4096, 4, None, 0, 1, None)
    assert rc == G.GEMM_ERR_ARG and "comm" in G.last_error()
    h = ctypes.c_void_p()
    rc = lib.gemm_comm_init(ctypes.byref(h), 2, ctypes.create_string_buffer(128), 5)
    assert rc == G.GEMM_ERR_ARG and "rank" in G.last_error()


def test_fill_and_probe_validation(G):
    lib = G.lib()
    assert lib.gemm_fill_f64(9, 1, 0, 4, 4, 0, 4, 16, 4, None) == G.GEMM_ERR_ARG
    assert lib.gemm_fill_f64(0, 1, 0, 4, 4, 2, 4, 16, 4, None) == G.GEMM_ERR_ARG   # slab outside
    assert lib.gemm_peak_probe(3, 1, 1, 1, 16, None, None) == G.GEMM_ERR_ARG


def test_row_range_partition(G):
    for M in (0, 1, 7, 16384, 32768, 65537):
        for P in (1, 2, 3, 4, 8):
            parts = [G.row_range(M, r, P) for r in range(P)]
            assert parts[0][0] == 0 and parts[-1][1] == M
            for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
                assert a1 == b0 and a0 <= a1
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        G.row_range(10, 2, 2)


def test_unique_id_is_128_bytes_and_fresh(G):
    a, b = G.unique_id(), G.unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b


def test_sass_f32_kernels_use_tcgen05(sass):
    """The single-precision path is Blackwell-native: tcgen05.mma (UTCHMMA), TMEM loads
    (LDTM), TMA (UTMALDG), no local-memory spills."""
    funcs = _functions(sass)
    f32 = {k: v for k, v in funcs.items() if "sgemm_3xtf32" in k}
    assert len(f32) >= 2
    for name, body in f32.items():
        assert "UTCHMMA" in body, name
        assert "LDTM" in body, name
        assert "UTMALDG" in body, name
        assert not re.search(r"\b(LDL|STL)\b", body), name


def test_hybrid_launch_count(G):
    """Host mirror of launch_hybrid: data-parallel waves, stream-K tail, fix-up when needed."""
    hyb = G.cfg_id("tma_256x64x16_w64x32_s4_hybrid")
    xp = G.cfg_id("tma_256x64x16_w64x32_s4_xp")
    assert G.launches_per_call(xp, 16384, 16384, 16384) == 1
    assert G.launches_per_call(hyb, 1024, 2368, 64) == 1          # 148 tiles: one full wave, no tail
    assert G.launches_per_call(hyb, 1024, 2496, 32) == 2          # tail CTAs own whole tiles: no fix-up
    assert G.launches_per_call(hyb, 16384, 16384, 16384) == 3     # 110 waves + 104-tile tail
    assert G.launches_per_call(hyb, 300, 200, 2000) == 2          # no full wave: tail + fix-up
    info = G.cfg_info(hyb)
    assert info["split_k"] == -2 and info["tma"] == 1


def test_binding_rejects_overlapping_and_negative_row_strides(G):
    """a zero-stride expand() (rows alias one buffer row) or a numpy row stride that
    is negative / not a multiple of 8 / overlapping must raise before any library call --
    the kernel would otherwise address rows*ld elements of a smaller buffer."""
    import numpy as np
    import torch
    ok = torch.zeros((3, 4), dtype=torch.float64)
    assert G._mat(ok, "A") == (ok.data_ptr(), 3, 4, 4)
    assert G._mat(torch.zeros((5, 8), dtype=torch.float64)[:, :3], "A")[3] == 8   # padded ld
    assert G._mat(torch.zeros((1, 8), dtype=torch.float64).expand(1, 8), "A")[3] == 8   # one row: ld unused
    with pytest.raises(ValueError, match="overlapping"):
        G._mat(torch.zeros((1, 8), dtype=torch.float64).expand(6, 8), "A")
    good = np.zeros((4, 4))
    for bad in (np.broadcast_to(np.zeros((1, 4)), (4, 4)), good[::-1], np.zeros((4, 9))[:, ::2]):
        with pytest.raises(ValueError):
            G.gemm_host(bad, good, np.zeros((4, 4)))
    with pytest.raises(ValueError, match="stride"):
        G.gemm_host(np.zeros((4, 4)), good, np.zeros((4, 4))[::-1])


def test_forced_splits_without_tma_is_rejected_explicitly(G):
    """gemm_f64_ex(cfg_id = -1, splits > 1) restricts the heuristic to split-K configurations;
    with operands that miss the TMA rules (odd lda) there is none: GEMM_ERR_UNSUPPORTED with a
    message, instead of silently running something else."""
    lib = G.lib()
    rc = lib.gemm_f64_ex(8, 8, 7, 1.0, 16, 7, 1024, 8, 0.0, 4096, 8, -1, 4, None)
    assert rc == G.GEMM_ERR_UNSUPPORTED and "splits=4" in G.last_error(), G.last_error()


def test_fast_entry_calls_the_same_library(G):
    """The vectorcall entry (csrc/pyfast.c) is built and calls gemm_f64_ex of the library
    ctypes loaded (one copy: same status codes and the same thread-local error message)."""
    import ctypes
    import sysconfig
    if not os.path.exists(os.path.join(sysconfig.get_paths()["include"], "Python.h")):
        pytest.skip("no Python headers: the binding uses ctypes")
    assert G._FAST is not None
    args_bad = (-1, 64, 64, 1.0, 16, 64, 16, 64, 0.0, 16, 64, -1, 0, None)
    assert G._FAST(*args_bad) == G.GEMM_ERR_ARG and "M=-1" in G.last_error()
    assert G._lib.gemm_f64_ex(*args_bad) == G.GEMM_ERR_ARG and "M=-1" in G.last_error()
    G._lib.gemm_last_error()          # same thread-local error state: set by one, read by the other
    assert G._FAST(0, 64, 64, 1.0, 16, 64, 16, 64, 0.0, 16, 64, -1, 0, None) == G.GEMM_OK   # M = 0: no-op
    assert G.last_error() == ""
    assert G._FAST(4, 4, 8, 1.0, 16, 4, 16, 4, 0.0, 16, 4, -1, 0, None) == G.GEMM_ERR_ARG
    assert "lda=4" in G.last_error()  # the message the C library wrote
    with pytest.raises(TypeError):
        G._FAST(1, 2, 3)
    addr = ctypes.cast(G._lib.gemm_f64_ex, ctypes.c_void_p).value
    assert addr
