"""Thin ctypes binding of libgemm_f64.so (include/gemm_f64.h).

Argument marshalling only: every step of C = alpha*A*B + beta*C (PAPER.md
Eq. (1)) runs in the CUDA kernels behind the C ABI.  PyTorch is used
for device memory and streams.  There is no fallback: if the library is
missing or fails to load, importing this module raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GEMM_F64_LIB: load another build of the same library instead (the instrumented
# libgemm_f64_trace.so of tools/trace_ctas.py); unset in every product / test / bench run
LIB_PATH = os.environ.get("GEMM_F64_LIB") or os.path.join(_HERE, "libgemm_f64.so")

GEMM_OK, GEMM_ERR_ARG, GEMM_ERR_CUDA, GEMM_ERR_NCCL, GEMM_ERR_UNSUPPORTED, GEMM_ERR_ALLOC = range(6)
STATUS_NAMES = {0: "GEMM_OK", 1: "GEMM_ERR_ARG", 2: "GEMM_ERR_CUDA", 3: "GEMM_ERR_NCCL",
                4: "GEMM_ERR_UNSUPPORTED", 5: "GEMM_ERR_ALLOC"}
FILL_MODES = {"uniform": 0, "dyadic": 1, "int8": 2, "ones": 3, "identity": 4, "zeros": 5}

# every symbol include/gemm_f64.h declares (tests check the library exports them all)
EXPORTS = ("gemm_f64", "gemm_f64_stream", "gemm_f64_cfg", "gemm_f64_ex", "gemm_f32", "gemm_f32_stream",
           "gemm_f32_cfg", "gemm_f32_num_cfgs", "gemm_f32_cfg_name", "gemm_f64_host", "gemm_host_plan", "gemm_host_pool_release",
           "gemm_workspace_release",
           "gemm_num_cfgs", "gemm_cfg_name", "gemm_cfg_info", "gemm_cfg_select", "gemm_plan", "gemm_plan_ex", "gemm_plan_set",
           "gemm_plan_clear", "gemm_tune_load", "gemm_tune_save", "gemm_plan_autotune", "gemm_last_error",
           "gemm_fill_f64", "gemm_peak_probe", "gemm_comm_unique_id", "gemm_comm_init",
           "gemm_comm_destroy", "gemm_comm_info", "gemm_f64_sharded", "gemm_bcast_f64", "gemm_version")


class GemmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class CfgDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("bm", "bn", "bk", "wm", "wn", "stages", "threads", "smem_bytes", "tma", "split_k", "regs")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1706_10086_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, dbl, vp, ci = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    core = [i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64]
    sig = {
        "gemm_f64": (ci, core),
        "gemm_f64_stream": (ci, core + [vp]),
        "gemm_f64_cfg": (ci, core + [ci, vp]),
        "gemm_f64_ex": (ci, core + [ci, ci, vp]),
        "gemm_f32": (ci, [i64, i64, i64, ctypes.c_float, vp, i64, vp, i64, ctypes.c_float, vp, i64]),
        "gemm_f32_stream": (ci, [i64, i64, i64, ctypes.c_float, vp, i64, vp, i64, ctypes.c_float, vp, i64, vp]),
        "gemm_f32_cfg": (ci, [i64, i64, i64, ctypes.c_float, vp, i64, vp, i64, ctypes.c_float, vp, i64, ci, vp]),
        "gemm_f32_num_cfgs": (ci, []),
        "gemm_f32_cfg_name": (ci, [ci, ctypes.c_char_p, ci]),
        "gemm_f64_host": (ci, core),
        "gemm_host_pool_release": (ci, []),
        "gemm_host_plan": (ci, [i64, i64, i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
        "gemm_workspace_release": (ci, []),
        "gemm_num_cfgs": (ci, []),
        "gemm_cfg_name": (ci, [ci, ctypes.c_char_p, ci]),
        "gemm_cfg_info": (ci, [ci, ctypes.POINTER(CfgDesc)]),
        "gemm_cfg_select": (ci, [i64, i64, i64, vp, i64, vp, i64]),
        "gemm_plan": (ci, [i64, i64, i64, vp, i64, vp, i64, ctypes.POINTER(ci), ctypes.POINTER(ci)]),
        "gemm_plan_ex": (ci, [i64, i64, i64, vp, i64, vp, i64, ci, ctypes.POINTER(ci), ctypes.POINTER(ci)]),
        "gemm_plan_set": (ci, [i64, i64, i64, ci, ci, ci]),
        "gemm_plan_clear": (ci, []),
        "gemm_tune_load": (ci, [ctypes.c_char_p, ctypes.POINTER(ci)]),
        "gemm_tune_save": (ci, [ctypes.c_char_p, ctypes.POINTER(ci)]),
        "gemm_plan_autotune": (ci, [i64, i64, i64, vp, i64, vp, i64, ci, ctypes.POINTER(ci), ctypes.POINTER(ci),
                                    ctypes.POINTER(dbl), vp]),
        "gemm_last_error": (ctypes.c_char_p, []),
        "gemm_fill_f64": (ci, [ci, ctypes.c_uint64, ci, i64, i64, i64, i64, vp, i64, vp]),
        "gemm_peak_probe": (ci, [ci, ci, ci, i64, vp, vp, vp]),
        "gemm_comm_unique_id": (ci, [ctypes.c_char_p]),
        "gemm_comm_init": (ci, [ctypes.POINTER(vp), ci, ctypes.c_char_p, ci]),
        "gemm_comm_destroy": (ci, [vp]),
        "gemm_comm_info": (ci, [vp, ctypes.POINTER(ci), ctypes.POINTER(ci)]),
        "gemm_f64_sharded": (ci, [i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp, ci, ci, vp]),
        "gemm_bcast_f64": (ci, [vp, i64, ci, vp, vp]),
        "gemm_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()

# The vectorcall entry (csrc/pyfast.c): the same gemm_f64_ex symbol of this very library,
# called without ctypes' per-argument conversion; absent -> ctypes.
try:
    if os.environ.get("GEMM_NO_FAST"):   # A/B of the host cost (tools/binding_overhead.py)
        raise ImportError("GEMM_NO_FAST set")
    from . import _gemm_fast as _fastmod
    _fastmod.set_target(ctypes.cast(_lib.gemm_f64_ex, ctypes.c_void_p).value)
    _FAST = _fastmod.gemm_f64_ex
except ImportError:
    _FAST = None

# The tuned plan table shipped with the package (produced on a B200 by
# `python -m paper_1706_10086_b200.tuner`); pinned plans override the size model for
# exactly these shapes.  Set GEMM_F64_NO_TUNED=1 to use the model alone.
TUNED_TABLE = os.path.join(_HERE, "tuned_b200.txt")
if os.path.exists(TUNED_TABLE) and not os.environ.get("GEMM_F64_NO_TUNED"):
    _n = ctypes.c_int()
    if _lib.gemm_tune_load(os.fsencode(TUNED_TABLE), ctypes.byref(_n)) != 0:
        raise ImportError(f"bad tuning table {TUNED_TABLE}: {_lib.gemm_last_error().decode()}")


def lib():
    return _lib


def last_error() -> str:
    return _lib.gemm_last_error().decode()


def version() -> str:
    return _lib.gemm_version().decode()


def _check(rc: int):
    if rc != GEMM_OK:
        raise GemmError(rc, last_error())


# ------------------------------------------------------------------ tensors
_DTYPES = {}


def _dtype(name):
    d = _DTYPES.get(name)
    if d is None:
        import torch
        d = _DTYPES[name] = getattr(torch, name)
    return d


def _mat(x, name, dtype="float64"):
    """(ptr, rows, cols, ld) of a 2-D float64 (or float32) tensor with unit column stride and
    non-overlapping rows (row stride >= cols; a zero-stride expand() or a negative stride is
    rejected, since the kernel would address rows*ld elements of a smaller buffer).
    Per-call cost matters for small GEMMs: one attribute access each (no string work)."""
    if x.dtype is not _dtype(dtype):
        raise TypeError(f"{name} must be {dtype}, got {x.dtype}")
    shp = x.shape
    if len(shp) != 2:
        raise ValueError(f"{name} must be 2-D")
    r, c = shp
    if r == 0 or c == 0:
        return x.data_ptr(), r, c, max(c, 1)
    s0, s1 = x.stride()
    if c > 1 and s1 != 1:
        raise ValueError(f"{name} must have unit stride along columns (row-major)")
    if r > 1:
        if s0 < c or s0 <= 0:
            raise ValueError(f"{name} has overlapping rows (row stride {s0} < {c} columns): make it contiguous")
        return x.data_ptr(), r, c, s0
    return x.data_ptr(), r, c, c   # a single row never uses its leading dimension


_RAW_STREAM = None
_CUR_DEV = None


def _current_device() -> int:
    """torch's current CUDA device index: the C-level query (~0.1 us) rather than
    torch.cuda.current_device() (~1 us, it re-checks lazy initialisation), falling back to
    the public API if the private one is absent."""
    global _CUR_DEV
    if _CUR_DEV is None:
        import torch
        fast = getattr(torch._C, "_cuda_getDevice", None)
        _CUR_DEV = fast if fast is not None else torch.cuda.current_device
    return _CUR_DEV()


def _current_raw_stream(dev=None):
    """cudaStream_t of torch's current stream on device `dev` (default: the current one).
    torch's raw-pointer query (what Triton's launcher uses) costs ~0.3 us against ~3 us for
    building a torch.cuda.Stream object, a large share of a small GEMM's host cost; the
    public API is the fallback if the private one is absent."""
    global _RAW_STREAM
    import torch
    if _RAW_STREAM is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _RAW_STREAM = raw if raw is not None else (lambda d: torch.cuda.current_stream(d).cuda_stream)
    return _RAW_STREAM(_current_device() if dev is None else dev)


def _stream_ptr(stream, dev=None):
    if stream is None:
        return _current_raw_stream(dev)
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _on_current_device(*ts, names="ABC"):
    """Every tensor is a CUDA tensor on the current device (the library launches there).
    Returns the device index."""
    dev = _current_device()
    for t, n in zip(ts, names):
        d = t.get_device()   # -1 for CPU tensors
        if d != dev:
            if d < 0:
                raise ValueError(f"{n} must be a CUDA tensor (use gemm_host for host buffers)")
            raise ValueError(f"{n} is on cuda:{d} but the current device is cuda:{dev} "
                             "(torch.cuda.set_device or move the tensor)")
    return dev


def gemm(A, B, C, alpha: float = 1.0, beta: float = 0.0, cfg: int | None = None, stream=None,
         splits: int | None = None):
    """C <- alpha*A@B + beta*C on the GPU (torch CUDA float64 tensors, row-major). Returns C."""
    pa, M, K, lda = _mat(A, "A")
    pb, K2, N, ldb = _mat(B, "B")
    pc, M2, N2, ldc = _mat(C, "C")
    if K2 != K or M2 != M or N2 != N:
        raise ValueError(f"shape mismatch A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    st = _stream_ptr(stream, _on_current_device(A, B, C))
    if _FAST is not None:   # gemm_f64_ex(cfg -1, splits 0) is gemm_f64_stream; (cfg, 0) is gemm_f64_cfg
        rc = _FAST(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc,
                   -1 if cfg is None else int(cfg), 0 if splits is None else int(splits), st)
    elif cfg is None and splits is None:
        rc = _lib.gemm_f64_stream(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc, st)
    elif splits is None:
        rc = _lib.gemm_f64_cfg(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc, int(cfg), st)
    else:
        rc = _lib.gemm_f64_ex(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc,
                              -1 if cfg is None else int(cfg), int(splits), st)
    _check(rc)
    return C


def gemm_f32(A, B, C, alpha: float = 1.0, beta: float = 0.0, stream=None, cfg: int | None = None):
    """C <- alpha*A@B + beta*C in single precision on the tensor cores (3xTF32), torch CUDA
    float32 tensors, row-major.  Returns C."""
    pa, M, K, lda = _mat(A, "A", "float32")
    pb, K2, N, ldb = _mat(B, "B", "float32")
    pc, M2, N2, ldc = _mat(C, "C", "float32")
    if K2 != K or M2 != M or N2 != N:
        raise ValueError(f"shape mismatch A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    _on_current_device(A, B, C)
    if cfg is None:
        _check(_lib.gemm_f32_stream(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc,
                                    _stream_ptr(stream)))
    else:
        _check(_lib.gemm_f32_cfg(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc, int(cfg),
                                 _stream_ptr(stream)))
    return C


def f32_cfg_names() -> list:
    out = []
    for i in range(_lib.gemm_f32_num_cfgs()):
        buf = ctypes.create_string_buffer(64)
        _check(_lib.gemm_f32_cfg_name(i, buf, 64))
        out.append(buf.value.decode())
    return out


def gemm_raw(M, N, K, alpha, A_ptr, lda, B_ptr, ldb, beta, C_ptr, ldc, cfg=-1, stream=0) -> int:
    """Raw C-ABI call with integer device pointers; returns the status code (no raise)."""
    return _lib.gemm_f64_cfg(int(M), int(N), int(K), float(alpha), A_ptr, int(lda), B_ptr, int(ldb),
                             float(beta), C_ptr, int(ldc), int(cfg), stream)


def gemm_host(A, B, C, alpha: float = 1.0, beta: float = 0.0):
    """C <- alpha*A@B + beta*C with HOST buffers (numpy arrays or CPU torch tensors)."""
    def info(x, name):
        if hasattr(x, "data_ptr"):
            if x.get_device() >= 0:
                raise ValueError(f"{name} must be a host (CPU) tensor for gemm_host")
            return _mat(x, name)
        import numpy as np
        if x.dtype != np.float64 or x.ndim != 2 or (x.shape[1] > 1 and x.strides[1] != 8):
            raise ValueError(f"{name} must be a row-major float64 2-D array")
        r, c = x.shape
        if r > 1 and x.shape[1] > 0:
            s0 = x.strides[0]
            if s0 <= 0 or s0 % 8 or s0 // 8 < c:
                raise ValueError(f"{name} row stride {s0} bytes is negative, not a multiple of 8 or "
                                 f"overlapping (< {c} doubles): make it contiguous")
            return x.ctypes.data, r, c, s0 // 8
        return x.ctypes.data, r, c, max(c, 1)
    pa, M, K, lda = info(A, "A")
    pb, K2, N, ldb = info(B, "B")
    pc, M2, N2, ldc = info(C, "C")
    if K2 != K or M2 != M or N2 != N:
        raise ValueError("shape mismatch")
    _check(_lib.gemm_f64_host(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc))
    return C


def host_plan(M: int, N: int, K: int, beta_nonzero: bool = False, num_sms: int = 0) -> tuple:
    """gemm_f64_host's block schedule for this shape: (dict of R0, Ra, cb0, cb, Rp, Rlast, nlast;
    the simulation's predicted seconds)."""
    g = (ctypes.c_int64 * 7)()
    sec = ctypes.c_double()
    _check(_lib.gemm_host_plan(M, N, K, int(bool(beta_nonzero)), int(num_sms), g, ctypes.byref(sec)))
    return dict(zip(("R0", "Ra", "cb0", "cb", "Rp", "Rlast", "nlast"), list(g))), sec.value


def host_pool_release():
    _check(_lib.gemm_host_pool_release())


def workspace_release():
    """Free the library's cached device workspace on the current device (gemm_workspace_release);
    CUDA graphs captured from earlier calls must not be replayed afterwards."""
    _check(_lib.gemm_workspace_release())


# ------------------------------------------------------------------ configs
def num_cfgs() -> int:
    return _lib.gemm_num_cfgs()


def cfg_name(i: int) -> str:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.gemm_cfg_name(i, buf, 128))
    return buf.value.decode()


def cfg_info(i: int) -> dict:
    d = CfgDesc()
    _check(_lib.gemm_cfg_info(i, ctypes.byref(d)))
    out = {n: getattr(d, n) for n, _ in CfgDesc._fields_}
    out["name"] = cfg_name(i)
    out["id"] = i
    out["e"] = out["wm"] * out["wn"] // 32
    return out


def cfgs() -> list:
    return [cfg_info(i) for i in range(num_cfgs())]


def cfg_id(name: str) -> int:
    for i in range(num_cfgs()):
        if cfg_name(i) == name:
            return i
    raise KeyError(name)


def cfg_select(M, N, K, A_ptr=0, lda=None, B_ptr=0, ldb=None) -> int:
    return _lib.gemm_cfg_select(M, N, K, A_ptr, lda if lda is not None else max(K, 1), B_ptr,
                                ldb if ldb is not None else max(N, 1))


def plan(M, N, K, A_ptr=0, lda=None, B_ptr=0, ldb=None, one_pass: bool = False) -> tuple:
    """(cfg_id, splits) the heuristic launches for this shape / alignment; one_pass=True: the
    plan of gemm(..., splits=1), gemm_host's blocks and Comm.gemm_sharded (gemm_plan_ex)."""
    cid, sp = ctypes.c_int(), ctypes.c_int()
    lda = lda if lda is not None else max(K, 1)
    ldb = ldb if ldb is not None else max(N, 1)
    if one_pass:
        _check(_lib.gemm_plan_ex(M, N, K, A_ptr, lda, B_ptr, ldb, 1, ctypes.byref(cid), ctypes.byref(sp)))
    else:
        _check(_lib.gemm_plan(M, N, K, A_ptr, lda, B_ptr, ldb, ctypes.byref(cid), ctypes.byref(sp)))
    return cid.value, sp.value


def sharded_panels(N: int, chunks: int) -> list:
    """Column panels [(n0, width)] gemm_f64_sharded uses for bcast_chunks = chunks (mirrors
    csrc/sharded.cu: at most N/64 panels, widths a multiple of 16 except the last)."""
    nch = min(chunks, max(1, N // 64))
    if nch <= 1:
        return [(0, N)]
    w = ((N + nch - 1) // nch + 15) // 16 * 16
    return [(n0, min(N, n0 + w) - n0) for n0 in range(0, N, w)]


HYB_MIN_STEPS = 16   # registry.cuh kHybMinSteps


def launches_per_call(cfg: int, M: int, N: int, K: int, sms: int = 148) -> int:
    """Kernels one gemm call with configuration `cfg` launches (alpha != 0, K > 0): 1 for the
    one-kernel schedules (plain, split-K with in-kernel reduction, stream-K); the hybrid
    (split_k = -2) launches the data-parallel waves, the stream-K tail and the tail fix-up,
    each only when needed (mirrors launch_hybrid in csrc/registry.cuh; the waves hold
    SMs x CTAs-per-SM tiles)."""
    d = cfg_info(cfg)
    if d["split_k"] != -2:
        return 1
    tiles = -(-M // d["bm"]) * -(-N // d["bn"])
    kt = -(-K // d["bk"])
    occ = 2 if 2 * (d["smem_bytes"] + 1024) <= 228 * 1024 else 1   # Cfg::MIN_BLOCKS (dgemm_kernels.cuh)
    sms = sms * occ
    tdp = tiles // sms * sms
    tail = tiles - tdp
    if tail == 0:
        return 1
    gsk = min(sms, max(tail, tail * kt // HYB_MIN_STEPS))
    fixup = not (gsk == tail and (tail * kt) % gsk == 0)
    return (1 if tdp > 0 else 0) + 1 + (1 if fixup else 0)


def plan_set(M, N, K, tma: bool, cfg: int, splits: int = 1):
    """Pin the plan used for (M, N, K, TMA-eligible) on the current device."""
    _check(_lib.gemm_plan_set(M, N, K, int(bool(tma)), int(cfg), int(splits)))


def plan_clear():
    _check(_lib.gemm_plan_clear())


def autotune(A, B, top: int = 0, stream=None) -> tuple:
    """Time the plan in force and the heuristic's next best plans for A @ B's shape on these
    operands and pin the fastest (gemm_plan_autotune).  Returns (cfg_id, splits, seconds)."""
    pa, M, K, lda = _mat(A, "A")
    pb, K2, N, ldb = _mat(B, "B")
    if K != K2:
        raise ValueError(f"inner dimensions differ: A is {M}x{K}, B is {K2}x{N}")
    _on_current_device(A, B, names="AB")
    cid, sp, sec = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check(_lib.gemm_plan_autotune(M, N, K, pa, lda, pb, ldb, int(top), ctypes.byref(cid), ctypes.byref(sp),
                                   ctypes.byref(sec), _stream_ptr(stream)))
    return cid.value, sp.value, sec.value


def tune_load(path: str) -> int:
    """Load a persisted tuning table (lines "M N K tma cfg_name splits"); returns entries loaded."""
    n = ctypes.c_int()
    _check(_lib.gemm_tune_load(os.fsencode(path), ctypes.byref(n)))
    return n.value


def tune_save(path: str) -> int:
    """Write every pinned plan (table, plan_set, autotune) in tune_load's format; returns lines written."""
    n = ctypes.c_int()
    _check(_lib.gemm_tune_save(os.fsencode(path), ctypes.byref(n)))
    return n.value


# ------------------------------------------------------------------ inputs
def fill(X, mode: str, seed: int, mat: int, rows: int | None = None, row0: int = 0, stream=None):
    """Fill device tensor X (nrows x cols) with rows [row0, row0+nrows) of the logical
    rows x cols matrix of synth's counter-based generator (bitwise identical)."""
    px, nrows, cols, ldx = _mat(X, "X")
    _on_current_device(X, names=("X",))
    if rows is None:
        rows = row0 + nrows
    _check(_lib.gemm_fill_f64(FILL_MODES[mode], int(seed) & (2 ** 64 - 1), int(mat), int(rows), int(cols),
                              int(row0), int(nrows), px, ldx, _stream_ptr(stream)))
    return X


def peak_probe(kind: str, blocks: int, warps: int, iters: int, out, cycles=None, stream=None):
    k = {"dmma": 0, "dfma": 1}[kind]
    _check(_lib.gemm_peak_probe(k, blocks, warps, iters, out.data_ptr(),
                                cycles.data_ptr() if cycles is not None else None, _stream_ptr(stream)))


# ------------------------------------------------------------------ multi-GPU
class Comm:
    """Library-owned NCCL communicator (one process per GPU).  The 128-byte id is
    created on rank 0 and distributed with torch.distributed (any backend)."""

    def __init__(self, rank: int, world: int, group=None):
        raw = share_unique_id(rank, world, group)
        self._h = ctypes.c_void_p()
        _check(_lib.gemm_comm_init(ctypes.byref(self._h), world, ctypes.create_string_buffer(raw, 128), rank))
        self.rank, self.world = rank, world

    @property
    def handle(self):
        return self._h

    def info(self) -> tuple:
        """(nranks, rank) as NCCL reports them for this communicator (gemm_comm_info)."""
        n, r = ctypes.c_int(), ctypes.c_int()
        _check(_lib.gemm_comm_info(self._h, ctypes.byref(n), ctypes.byref(r)))
        return n.value, r.value

    def bcast(self, X, root: int = 0, stream=None):
        _check(_lib.gemm_bcast_f64(X.data_ptr(), X.numel(), root, self._h, _stream_ptr(stream)))

    def gemm_sharded(self, A_local, B, C_local, alpha=1.0, beta=0.0, root=0, bcast_chunks=1, stream=None):
        pa, M, K, lda = _mat(A_local, "A_local")
        pb, K2, N, ldb = _mat(B, "B")
        pc, M2, N2, ldc = _mat(C_local, "C_local")
        if K2 != K or M2 != M or N2 != N:
            raise ValueError("shape mismatch")
        _on_current_device(A_local, B, C_local, names=("A_local", "B", "C_local"))
        _check(_lib.gemm_f64_sharded(M, N, K, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc,
                                     self._h, int(root), int(bcast_chunks), _stream_ptr(stream)))
        return C_local

    def close(self):
        if self._h:
            _check(_lib.gemm_comm_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (gemm_comm_unique_id)."""
    idbuf = ctypes.create_string_buffer(128)
    _check(_lib.gemm_comm_unique_id(idbuf))
    return bytes(idbuf.raw)


def share_unique_id(rank: int, world: int, group=None) -> bytes:
    """Rank 0 creates the id; every rank returns the same 128 bytes (torch.distributed,
    any backend -- gloo in the CPU tests, nccl in bench.py)."""
    payload = [unique_id() if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(payload, src=0, group=group)
    raw = payload[0]
    if not isinstance(raw, (bytes, bytearray)) or len(raw) != 128:
        raise RuntimeError("NCCL unique id distribution failed")
    return bytes(raw)


def max_over_ranks(values, world: int, device=None):
    """Element-wise max over ranks of a list of floats (timing is max over ranks)."""
    if world <= 1:
        return [float(v) for v in values]
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def row_range(M: int, rank: int, world: int) -> tuple:
    """Rows [floor(r*M/P), floor((r+1)*M/P)) owned by `rank` (include/gemm_f64.h sharded contract)."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError(f"bad partition M={M} rank={rank} world={world}")
    return (rank * M) // world, ((rank + 1) * M) // world
