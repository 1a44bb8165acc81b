// registry.cuh -- configuration table entries and the launch templates.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/gemm_f64.h"
#include "dgemm_kernels.cuh"
#include "internal.h"

namespace dg {

int make_tmap(CUtensorMap *map, const double *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

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
    SplitArgs sk;
};

struct CfgEntry {
    const char *name;
    gemm_cfg_desc d;
    const void *kernel;
    int (*launch)(const LaunchArgs &, cudaStream_t);
};

template <class C, bool SPLIT, bool XP>
static int launch_tma(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, a.A, a.M, a.K, a.lda, C::BM);
    if (rc) return rc;
    rc = make_tmap(&tb, a.B, a.K, a.N, a.ldb, 16);
    if (rc) return rc;
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    dim3 grid((unsigned)tiles, SPLIT ? a.sk.splits : 1);
    dgemm_tma_kernel<C, SPLIT, XP><<<grid, C::CONSUMER_THREADS, C::SMEM_BYTES, st>>>(
        ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec, a.group_m, a.sk);
    return cuda_check(cudaGetLastError(), "dgemm_tma_kernel launch");
}

template <class C>
static int launch_generic(const LaunchArgs &a, cudaStream_t st) {
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    dgemm_generic_kernel<C><<<(unsigned)tiles, C::CONSUMER_THREADS, C::SMEM_BYTES, st>>>(
        a.A, a.lda, a.B, a.ldb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec, a.group_m);
    return cuda_check(cudaGetLastError(), "dgemm_generic_kernel launch");
}

// Stream-K launch: grid = min(U, SMs x resident CTAs); workspace = 2 partial slots per CTA.
int streamk_workspace(cudaStream_t st, size_t slot_doubles, int grid, size_t tiles, double **ws, int **ctr);
int streamk_grid(const void *kernel, int threads, int smem, int64_t units);

template <class C>
static int launch_streamk(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, a.A, a.M, a.K, a.lda, C::BM);
    if (rc) return rc;
    rc = make_tmap(&tb, a.B, a.K, a.N, a.ldb, 16);
    if (rc) return rc;
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    const int64_t KT = ((int64_t)a.K + C::BK - 1) / C::BK;
    if (tiles * KT > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "stream-K needs tiles*k-steps < 2^31");
    const int grid = streamk_grid((const void *)dgemm_streamk_kernel<C>, C::CONSUMER_THREADS, C::SMEM_BYTES,
                                  tiles * KT);
    if (grid <= 0) return set_error(GEMM_ERR_CUDA, "stream-K occupancy query failed");
    double *ws = nullptr;
    int *ctr = nullptr;
    rc = streamk_workspace(st, (size_t)C::BM * C::BN, grid, (size_t)tiles, &ws, &ctr);
    if (rc) return rc;
    dgemm_streamk_kernel<C><<<grid, C::CONSUMER_THREADS, C::SMEM_BYTES, st>>>(
        ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec, a.group_m, ws, ctr);
    return cuda_check(cudaGetLastError(), "dgemm_streamk_kernel launch");
}

#define DG_SK(BM, BN, BK, WM, WN, ST)                                                                        \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST "_streamk",                                 \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, -1, 0},                           \
             (const void *)dgemm_streamk_kernel<Cfg<BM, BN, BK, WM, WN, ST>>,                                 \
             launch_streamk<Cfg<BM, BN, BK, WM, WN, ST>>}

#define DG_TMA_SK(BM, BN, BK, WM, WN, ST, SK, SPLIT, XP, SUFFIX)                                              \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST SUFFIX,                                     \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, SK, 0},                           \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST>, SPLIT, XP>,                           \
             launch_tma<Cfg<BM, BN, BK, WM, WN, ST>, SPLIT, XP>}
#define DG_TMA(BM, BN, BK, WM, WN, ST) DG_TMA_SK(BM, BN, BK, WM, WN, ST, 1, false, false, "")
// split_k = 0: number of k-splits chosen per call (deterministic split-K, SplitArgs)
#define DG_TMA_SPLIT(BM, BN, BK, WM, WN, ST) DG_TMA_SK(BM, BN, BK, WM, WN, ST, 0, true, false, "_splitk")
// cross-stage fragment prefetch variant
#define DG_TMA_XP(BM, BN, BK, WM, WN, ST) DG_TMA_SK(BM, BN, BK, WM, WN, ST, 1, false, true, "_xp")
#define DG_GEN(BM, BN, BK, WM, WN, ST)                                                                       \
    CfgEntry{"gen_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST,                                            \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 0, 1, 0},                            \
             (const void *)dgemm_generic_kernel<Cfg<BM, BN, BK, WM, WN, ST>>,                                 \
             launch_generic<Cfg<BM, BN, BK, WM, WN, ST>>}

const CfgEntry *cfg_table_big(int *n);
const CfgEntry *cfg_table_small(int *n);
const CfgEntry *cfg_table_generic(int *n);

}  // namespace dg
