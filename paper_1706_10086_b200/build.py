"""Build libgemm_f64.so in-tree for sm_100a (nvcc; no torch extension machinery).

    python -m paper_1706_10086_b200.build [--force] [--trace]

Compiles every csrc/*.cu with `-gencode arch=compute_100a,code=sm_100a -O3
-lineinfo` (no fast-math), links the static CUDA runtime and the NCCL shipped
with torch (nvidia/nccl), and writes paper_1706_10086_b200/libgemm_f64.so.

--trace builds an instrumented copy (-DDG_TRACE: per-CTA globaltimer timeline, see
csrc/ptx.cuh) as libgemm_f64_trace.so for tools/trace_ctas.py; the product never loads it.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgemm_f64.so")
BUILD = os.path.join(HERE, "build")
TRACE_LIB = os.path.join(HERE, "libgemm_f64_trace.so")
TRACE_BUILD = os.path.join(HERE, "build_trace")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    raise RuntimeError("NCCL headers/library (nvidia/nccl) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.inc")) + [os.path.join(ROOT, "include", "gemm_f64.h"), __file__]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    lib_out, build_dir = (TRACE_LIB, TRACE_BUILD) if trace else (LIB, BUILD)
    if not force and up_to_date(lib_out):
        if not trace:
            build_fast(verbose=verbose)
        return lib_out
    os.makedirs(build_dir, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    nvcc = _nvcc()
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
                    "-I", os.path.join(ROOT, "include"), "-I", nccl_inc] + (["-DDG_TRACE"] if trace else [])

    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [nvcc] + flags + ["-c", src, "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(p.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    nccl_so = sorted(glob.glob(os.path.join(nccl_lib, "libnccl.so*")))[0]
    tmp = lib_out + ".tmp"
    cmd = [nvcc] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + \
        ["-Xlinker", nccl_so, "-Xlinker", "-rpath=" + nccl_lib, "-lpthread", "-ldl", "-lrt"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, lib_out)
    if verbose:
        print(f"built {lib_out}")
    if not trace:
        build_fast(force=force, verbose=verbose)
    return lib_out


def fast_ext_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_gemm_fast" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_fast(force: bool = False, verbose: bool = False):
    """The binding's vectorcall entry (csrc/pyfast.c, argument marshalling only); skipped when
    Python's headers are missing (the binding then calls the same symbol through ctypes)."""
    import sysconfig
    src, out = os.path.join(CSRC, "pyfast.c"), fast_ext_path()
    inc = sysconfig.get_paths()["include"]
    if not os.path.exists(os.path.join(inc, "Python.h")):
        return None
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    tmp = out + ".tmp"
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall", "-I", inc, src, "-o", tmp]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"pyfast build failed:\n{p.stderr}")
    os.replace(tmp, out)
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv)
