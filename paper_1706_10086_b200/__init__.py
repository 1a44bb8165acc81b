"""B200-native FP64 GEMM (C = alpha*A*B + beta*C) -- the hot path of arXiv 1706.10086.

The compute lives in ``libgemm_f64.so`` (CUDA for sm_100a, C ABI in
``include/gemm_f64.h``); :mod:`paper_1706_10086_b200.gemm` is its ctypes
binding.  Importing :mod:`.gemm` fails loudly when the library is missing.
"""

__all__ = ["gemm"]
