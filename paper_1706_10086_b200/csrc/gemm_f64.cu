// gemm_f64.cu -- C-ABI dispatcher of libgemm_f64.so (include/gemm_f64.h).
//
// Argument validation, BLAS quick returns, the configuration registry (the
// compile-time tile instances the tuning sweep walks, Listing 1
// P:135-168 / §2.3 "Multidimensional parameter tuning" P:315-320), the size
// heuristic, TMA descriptor construction and the kernel launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "../../include/gemm_f64.h"
#include "dgemm_kernels.cuh"
#include "internal.h"

namespace dg {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

int set_error(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}
void clear_error() { g_last_error.clear(); }
const char *last_error() { return g_last_error.c_str(); }

int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return GEMM_OK;
    return set_error(GEMM_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ------------------------------------------------------------------ TMA encode
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Row-major rows x cols matrix with leading dimension ld; box = box_rows x 16 doubles (128 B).
static int make_tmap(CUtensorMap *map, const double *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return set_error(GEMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
    cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(GEMM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld", (int)r,
                         (long long)rows, (long long)cols, (long long)ld);
    return GEMM_OK;
}

// ------------------------------------------------------------------ registry
struct LaunchArgs {
    int M, N, K;
    double alpha, beta;
    const double *A;
    int64_t lda;
    const double *B;
    int64_t ldb;
    double *C;
    int64_t ldc;
    int vec;
    int group_m;
};

struct CfgEntry {
    const char *name;
    gemm_cfg_desc d;
    const void *kernel;
    int (*launch)(const LaunchArgs &, cudaStream_t);
};

template <class C>
static int launch_tma(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, a.A, a.M, a.K, a.lda, C::BM);
    if (rc) return rc;
    rc = make_tmap(&tb, a.B, a.K, a.N, a.ldb, 16);
    if (rc) return rc;
    const int tiles = ((a.M + C::BM - 1) / C::BM) * ((a.N + C::BN - 1) / C::BN);
    dgemm_tma_kernel<C><<<tiles, C::CONSUMER_THREADS, C::SMEM_BYTES, st>>>(
        ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec, a.group_m);
    return cuda_check(cudaGetLastError(), "dgemm_tma_kernel launch");
}

template <class C>
static int launch_generic(const LaunchArgs &a, cudaStream_t st) {
    const int tiles = ((a.M + C::BM - 1) / C::BM) * ((a.N + C::BN - 1) / C::BN);
    dgemm_generic_kernel<C><<<tiles, C::CONSUMER_THREADS, C::SMEM_BYTES, st>>>(
        a.A, a.lda, a.B, a.ldb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec, a.group_m);
    return cuda_check(cudaGetLastError(), "dgemm_generic_kernel launch");
}

#define DG_TMA(BM, BN, BK, WM, WN, ST)                                                                       \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST,                                            \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,         \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, 1, 0},                            \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST>>, launch_tma<Cfg<BM, BN, BK, WM, WN, ST>>}
#define DG_GEN(BM, BN, BK, WM, WN, ST)                                                                       \
    CfgEntry{"gen_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST,                                            \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 0, 1, 0},                            \
             (const void *)dgemm_generic_kernel<Cfg<BM, BN, BK, WM, WN, ST>>,                                 \
             launch_generic<Cfg<BM, BN, BK, WM, WN, ST>>}

static CfgEntry g_cfgs[] = {
#include "cfg_list.inc"
};
static constexpr int kNumCfgs = sizeof(g_cfgs) / sizeof(g_cfgs[0]);

static std::mutex g_attr_mu;
static std::set<std::pair<int, int>> g_attr_done;

static int prepare_cfg(int id) {
    int dev = 0;
    int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_done.count({dev, id})) return GEMM_OK;
    CfgEntry &e = g_cfgs[id];
    rc = cuda_check(cudaFuncSetAttribute(e.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, e.d.smem_bytes),
                    "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    if (rc) return rc;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, e.kernel) == cudaSuccess) e.d.regs = fa.numRegs;
    g_attr_done.insert({dev, id});
    return GEMM_OK;
}

static int find_cfg(const char *name) {
    for (int i = 0; i < kNumCfgs; ++i)
        if (!strcmp(g_cfgs[i].name, name)) return i;
    return -1;
}

static bool tma_ok(const double *A, int64_t lda, const double *B, int64_t ldb) {
    return ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) && (lda % 2 == 0) && (ldb % 2 == 0) &&
           lda * 8 < (int64_t(1) << 40) && ldb * 8 < (int64_t(1) << 40);
}

// Size heuristic: the largest tile that still fills the
// 148 SMs; TMA when alignment allows.
static int select_cfg(int64_t M, int64_t N, int64_t K, bool tma) {
    (void)K;
    static const char *big_t = "tma_128x128x16_w64x32_s4";
    static const char *mid_t = "tma_128x64x16_w32x32_s6";
    static const char *small_t = "tma_64x64x16_w32x16_s6";
    static const char *big_g = "gen_128x128x16_w64x32_s4";
    static const char *small_g = "gen_64x64x16_w32x16_s4";
    const int64_t tiles128 = ((M + 127) / 128) * ((N + 127) / 128);
    const int64_t tiles64x128 = ((M + 127) / 128) * ((N + 63) / 64);
    const char *name;
    if (tma)
        name = tiles128 >= 2 * 148 ? big_t : (tiles64x128 >= 148 ? mid_t : small_t);
    else
        name = tiles128 >= 2 * 148 ? big_g : small_g;
    int id = find_cfg(name);
    return id >= 0 ? id : 0;
}

static bool overlaps(const void *p, int64_t rows, int64_t cols, int64_t ld, const void *q, int64_t qrows,
                     int64_t qcols, int64_t qld) {
    if (!p || !q || rows <= 0 || cols <= 0 || qrows <= 0 || qcols <= 0) return false;
    const char *p0 = (const char *)p, *p1 = p0 + ((rows - 1) * ld + cols) * 8;
    const char *q0 = (const char *)q, *q1 = q0 + ((qrows - 1) * qld + qcols) * 8;
    return p0 < q1 && q0 < p1;
}

int validate(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
             int64_t ldb, const double *C, int64_t ldc) {
    if (M < 0) return set_error(GEMM_ERR_ARG, "M=%lld must be >= 0", (long long)M);
    if (N < 0) return set_error(GEMM_ERR_ARG, "N=%lld must be >= 0", (long long)N);
    if (K < 0) return set_error(GEMM_ERR_ARG, "K=%lld must be >= 0", (long long)K);
    const int64_t lim = (int64_t(1) << 31) - 1;
    if (M > lim || N > lim || K > lim)
        return set_error(GEMM_ERR_UNSUPPORTED, "M, N, K must be < 2^31 (M=%lld N=%lld K=%lld)", (long long)M,
                         (long long)N, (long long)K);
    if (lda < std::max<int64_t>(1, K))
        return set_error(GEMM_ERR_ARG, "lda=%lld must be >= max(1,K=%lld)", (long long)lda, (long long)K);
    if (ldb < std::max<int64_t>(1, N))
        return set_error(GEMM_ERR_ARG, "ldb=%lld must be >= max(1,N=%lld)", (long long)ldb, (long long)N);
    if (ldc < std::max<int64_t>(1, N))
        return set_error(GEMM_ERR_ARG, "ldc=%lld must be >= max(1,N=%lld)", (long long)ldc, (long long)N);
    if (M == 0 || N == 0) return GEMM_OK;
    if (!C) return set_error(GEMM_ERR_ARG, "C is NULL with M*N > 0");
    if ((uintptr_t)C % 8) return set_error(GEMM_ERR_ARG, "C is not 8-byte aligned");
    if (alpha != 0.0 && K > 0) {
        if (!A) return set_error(GEMM_ERR_ARG, "A is NULL with alpha != 0, K > 0");
        if (!B) return set_error(GEMM_ERR_ARG, "B is NULL with alpha != 0, K > 0");
        if ((uintptr_t)A % 8) return set_error(GEMM_ERR_ARG, "A is not 8-byte aligned");
        if ((uintptr_t)B % 8) return set_error(GEMM_ERR_ARG, "B is not 8-byte aligned");
        if (overlaps(C, M, N, ldc, A, M, K, lda)) return set_error(GEMM_ERR_ARG, "C overlaps A");
        if (overlaps(C, M, N, ldc, B, K, N, ldb)) return set_error(GEMM_ERR_ARG, "C overlaps B");
    }
    return GEMM_OK;
}

int gemm_impl(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
              int64_t ldb, double beta, double *C, int64_t ldc, int cfg_id, cudaStream_t st) {
    clear_error();
    int rc = validate(M, N, K, alpha, A, lda, B, ldb, C, ldc);
    if (rc) return rc;
    if (cfg_id < -1 || cfg_id >= kNumCfgs)
        return set_error(GEMM_ERR_ARG, "cfg_id=%d out of range [-1, %d)", cfg_id, kNumCfgs);
    if (M == 0 || N == 0) return GEMM_OK;
    if (alpha == 0.0 || K == 0) {
        if (beta == 1.0) return GEMM_OK;
        const int64_t total = M * N;
        const int threads = 256;
        const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
        scale_kernel<<<blocks, threads, 0, st>>>((int)M, (int)N, beta, C, ldc);
        return cuda_check(cudaGetLastError(), "scale_kernel launch");
    }
    const bool tma = tma_ok(A, lda, B, ldb);
    int id = cfg_id;
    if (id < 0) {
        id = select_cfg(M, N, K, tma);
    } else if (g_cfgs[id].d.tma && !tma) {
        return set_error(GEMM_ERR_UNSUPPORTED,
                         "cfg %s needs 16-byte aligned A/B and even lda/ldb (A%%16=%d B%%16=%d lda=%lld ldb=%lld)",
                         g_cfgs[id].name, (int)((uintptr_t)A % 16), (int)((uintptr_t)B % 16), (long long)lda,
                         (long long)ldb);
    }
    rc = prepare_cfg(id);
    if (rc) return rc;
    LaunchArgs a{(int)M, (int)N, (int)K, alpha, beta, A, lda, B, ldb, C, ldc,
                 ((uintptr_t)C % 32 == 0 && ldc % 4 == 0) ? 1 : 0, 8};
    return g_cfgs[id].launch(a, st);
}

}  // namespace dg

using namespace dg;

extern "C" {

int gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
             int64_t ldb, double beta, double *C, int64_t ldc) {
    return gemm_impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, -1, (cudaStream_t)0);
}

int gemm_f64_stream(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
                    int64_t ldb, double beta, double *C, int64_t ldc, void *stream) {
    return gemm_impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, -1, (cudaStream_t)stream);
}

int gemm_f64_cfg(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double beta, double *C, int64_t ldc, int cfg_id, void *stream) {
    return gemm_impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, cfg_id, (cudaStream_t)stream);
}

int gemm_num_cfgs(void) { return kNumCfgs; }

int gemm_cfg_name(int cfg_id, char *buf, int len) {
    clear_error();
    if (cfg_id < 0 || cfg_id >= kNumCfgs) return set_error(GEMM_ERR_ARG, "cfg_id=%d out of range", cfg_id);
    if (!buf || len <= 0) return set_error(GEMM_ERR_ARG, "buf is NULL or len <= 0");
    snprintf(buf, (size_t)len, "%s", g_cfgs[cfg_id].name);
    return GEMM_OK;
}

int gemm_cfg_info(int cfg_id, gemm_cfg_desc *out) {
    clear_error();
    if (cfg_id < 0 || cfg_id >= kNumCfgs) return set_error(GEMM_ERR_ARG, "cfg_id=%d out of range", cfg_id);
    if (!out) return set_error(GEMM_ERR_ARG, "out is NULL");
    *out = g_cfgs[cfg_id].d;
    return GEMM_OK;
}

int gemm_cfg_select(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B, int64_t ldb) {
    return select_cfg(M, N, K, tma_ok(A, lda, B, ldb));
}

const char *gemm_last_error(void) { return last_error(); }

const char *gemm_version(void) { return "gemm_f64 0.1 (sm_100a, DMMA.8x8x4, TMA/mbarrier)"; }

}  // extern "C"
