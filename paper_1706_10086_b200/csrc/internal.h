// internal.h -- shared declarations between the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dg {
int set_error(int code, const char *fmt, ...);
void clear_error();
const char *last_error();
int cuda_check(cudaError_t e, const char *what);
int validate(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
             int64_t ldb, const double *C, int64_t ldc);
int gemm_impl(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
              int64_t ldb, double beta, double *C, int64_t ldc, int cfg_id, cudaStream_t st, int force_splits = 0);
int workspace_release_f64();          // synchronizes the device, frees the FP64 workspace cache
namespace f32 {
void workspace_release_f32();         // frees the FP32 workspace cache (device already synchronized)
}
}  // namespace dg
