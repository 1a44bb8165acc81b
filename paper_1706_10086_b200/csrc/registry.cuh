// registry.cuh -- configuration table entries and the launch templates.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cuda.h>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/gemm_f64.h"
#include "dgemm_kernels.cuh"
#include "internal.h"
#include "launch.cuh"

namespace dg {

int make_tmap(CUtensorMap *map, const double *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);
int make_tmaps_md(CUtensorMap *ta, CUtensorMap *tb, const double *A, int64_t M, int64_t K, int64_t lda,
                  const double *B, int64_t N, int64_t ldb, int bm, int bn, int kg);


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

// The A / B tensor maps of a dgemm_tma_kernel launch: the multi-dimensional pair (one TMA
// instruction each per stage; vec bit 1 tells the kernel) when the shape allows, else 2-D.
template <class C>
static int tma_maps(const LaunchArgs &a, CUtensorMap *ta, CUtensorMap *tb, int *vec) {
    *vec = a.vec;
    if (make_tmaps_md(ta, tb, a.A, a.M, a.K, a.lda, a.B, a.N, a.ldb, C::BM, C::BN, C::KG) == GEMM_OK) {
        *vec |= 2;
        return GEMM_OK;
    }
    int rc = make_tmap(ta, a.A, a.M, a.K, a.lda, C::BM);
    if (rc) return rc;
    return make_tmap(tb, a.B, a.K, a.N, a.ldb, 16);
}

struct CfgEntry {
    const char *name;
    gemm_cfg_desc d;
    const void *kernel;
    int (*launch)(const LaunchArgs &, cudaStream_t);
};

// TMA kernels: the refill of k-step i is issued by warp i % kRotXP (dgemm_tma_kernel ROT)
constexpr int kRotXP = 4;

template <class C, int SPLIT, bool XP, int ROT = 1>
static int launch_tma(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int vec = 0;
    int rc = tma_maps<C>(a, &ta, &tb, &vec);
    if (rc) return rc;
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    dim3 grid((unsigned)tiles, SPLIT ? a.sk.splits : 1);
    return cuda_check(launch_k(dgemm_tma_kernel<C, SPLIT, XP, ROT>, grid, dim3(C::CONSUMER_THREADS), C::SMEM_BYTES, st,
                               ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, vec, a.group_m, a.sk),
                      "dgemm_tma_kernel launch");
}

// Cluster split-K: grid (tiles, S), clusters of (1, S, 1); S clamped to [1, min(8, KT)] (the
// portable cluster size, at least one k-step per slice); S = 1 is the plain one-pass kernel.
template <class C>
static int launch_tma_cluster(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int vec = 0;
    int rc = tma_maps<C>(a, &ta, &tb, &vec);
    if (rc) return rc;
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    const int64_t KT = ((int64_t)a.K + C::BK - 1) / C::BK;
    const int S = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(a.sk.splits, 8), KT));
    SplitArgs none{1, nullptr, nullptr};
    return cuda_check(launch_k_cluster(dgemm_tma_kernel<C, 2, false, kRotXP>, dim3((unsigned)tiles, S),
                                       dim3(C::CONSUMER_THREADS), C::SMEM_BYTES, st, 1u, (unsigned)S, ta, tb, a.M,
                                       a.N, a.K, a.alpha, a.beta, a.C, a.ldc, vec, a.group_m, none),
                      "dgemm_tma_kernel (cluster split-K) launch");
}

template <class C>
static int launch_generic(const LaunchArgs &a, cudaStream_t st) {
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    return cuda_check(launch_k(dgemm_generic_kernel<C>, dim3((unsigned)tiles), dim3(C::CONSUMER_THREADS),
                               C::SMEM_BYTES, st, a.A, a.lda, a.B, a.ldb, a.M, a.N, a.K, a.alpha, a.beta, a.C,
                               a.ldc, a.vec, a.group_m),
                      "dgemm_generic_kernel launch");
}

// Stream-K launch: grid = min(U, SMs x resident CTAs); workspace = 2 partial slots per CTA.
int streamk_workspace(cudaStream_t st, size_t slot_doubles, int grid, size_t tiles, double **ws, int **ctr);
int streamk_grid(const void *kernel, int threads, int smem, int64_t units);
constexpr int64_t kHybMinSteps = 16;   // hybrid tail: at least this many k-steps per stream-K CTA

template <class C>
static int launch_streamk(const LaunchArgs &a, cudaStream_t st) {
    CUtensorMap ta, tb;
    int vec = 0;
    int rc = tma_maps<C>(a, &ta, &tb, &vec);
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
    return cuda_check(launch_k(dgemm_streamk_kernel<C>, dim3(grid), dim3(C::CONSUMER_THREADS), C::SMEM_BYTES, st,
                               ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, vec, a.group_m, ws, ctr),
                      "dgemm_streamk_kernel launch");
}

// Hybrid launch: the W full data-parallel waves as one plain XP launch (grid = W*G tiles),
// then the tail's k-steps over gsk stream-K CTAs, then the fix-up of the cut tail tiles.
template <class C>
static int launch_hybrid(const LaunchArgs &a, cudaStream_t st) {
    // full waves: the XP kernel for the 64-accumulator warp tiles; for smaller warp tiles the
    // plain loop, in its split-K instance run with one slice (ptxas schedules that instance
    // better: 99.2 % against 98.8 % of the clock roof at 16384^3)
    constexpr bool kDpXP = C::E >= 64;
    constexpr bool kDpSplit = !kDpXP;
    const void *dp_kernel = (const void *)dgemm_tma_kernel<C, kDpSplit, kDpXP, kRotXP>;
    const void *sk_kernel = (const void *)dgemm_sktail_kernel<C>;
    int rc = cuda_check(cudaFuncSetAttribute(dp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES),
                        "cudaFuncSetAttribute(hybrid data-parallel kernel)");
    if (rc) return rc;
    CUtensorMap ta, tb;
    int vec = 0;
    rc = tma_maps<C>(a, &ta, &tb, &vec);
    if (rc) return rc;
    const int64_t tiles = ((int64_t)a.M + C::BM - 1) / C::BM * (((int64_t)a.N + C::BN - 1) / C::BN);
    const int64_t KT = ((int64_t)a.K + C::BK - 1) / C::BK;
    if (tiles * KT > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "hybrid needs tiles*k-steps < 2^31");
    const int G = streamk_grid(dp_kernel, C::CONSUMER_THREADS, C::SMEM_BYTES, 1LL << 40);
    if (G <= 0) return set_error(GEMM_ERR_CUDA, "hybrid occupancy query failed");
    const int64_t tdp = tiles / G * G, tail = tiles - tdp;
    if (tdp > 0) {
        SplitArgs none{1, nullptr, nullptr};
        rc = cuda_check(launch_k(dgemm_tma_kernel<C, kDpSplit, kDpXP, kRotXP>, dim3((unsigned)tdp), dim3(C::CONSUMER_THREADS),
                                 C::SMEM_BYTES, st, ta, tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, vec,
                                 a.group_m, none),
                        "hybrid data-parallel launch");
        if (rc || tail == 0) return rc;
    }
    HybArgs hy{(int)tdp, 0, nullptr};
    const int64_t Ut = tail * KT;
    hy.gsk = (int)std::min<int64_t>(G, std::max<int64_t>(tail, Ut / kHybMinSteps));
    int *ctr = nullptr;
    rc = streamk_workspace(st, (size_t)C::BM * C::BN, hy.gsk, 0, &hy.ws, &ctr);
    if (rc) return rc;
    rc = cuda_check(launch_k(dgemm_sktail_kernel<C>, dim3(hy.gsk), dim3(C::CONSUMER_THREADS), C::SMEM_BYTES, st, ta,
                             tb, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, vec, a.group_m, hy),
                    "dgemm_sktail_kernel launch");
    if (rc || ((int64_t)hy.gsk == tail && Ut % hy.gsk == 0)) return rc;   // every tail CTA had a whole tile
    static_assert((C::MB * C::NP) % FixQ<C> == 0, "fix-up quad split");
    return cuda_check(launch_k(dgemm_hybrid_fixup_kernel<C>, dim3((unsigned)tail, C::MB * C::NP / FixQ<C>),
                               dim3(C::CONSUMER_THREADS), 0, st, a.M, a.N, a.K, a.alpha, a.beta, a.C, a.ldc, a.vec,
                               a.group_m, (int)tdp, hy.gsk, (const double *)hy.ws),
                      "dgemm_hybrid_fixup_kernel launch");
}

#define DG_HYB(BM, BN, BK, WM, WN, ST)                                                                       \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST "_hybrid",                                  \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, -2, 0},                           \
             (const void *)dgemm_sktail_kernel<Cfg<BM, BN, BK, WM, WN, ST>>,                                  \
             launch_hybrid<Cfg<BM, BN, BK, WM, WN, ST>>}

#define DG_SK(BM, BN, BK, WM, WN, ST)                                                                     \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST "_streamk",                                 \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, -1, 0},                           \
             (const void *)dgemm_streamk_kernel<Cfg<BM, BN, BK, WM, WN, ST>>,                                 \
             launch_streamk<Cfg<BM, BN, BK, WM, WN, ST>>}

// cluster split-K: split_k = -3 (slices chosen per call, reduced through distributed shared memory)
#define DG_CSK(BM, BN, BK, WM, WN, ST)                                                                    \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST "_csplit",                                  \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, -3, 0},                           \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST>, 2, false, kRotXP>,                   \
             launch_tma_cluster<Cfg<BM, BN, BK, WM, WN, ST>>}

#define DG_TMA_SK(BM, BN, BK, WM, WN, ST, SK, SPLIT, XP, SUFFIX)                                              \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST SUFFIX,                                     \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, SK, 0},                           \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST>, SPLIT, XP, kRotXP>,                   \
             launch_tma<Cfg<BM, BN, BK, WM, WN, ST>, SPLIT, XP, kRotXP>}
#define DG_TMA(BM, BN, BK, WM, WN, ST) DG_TMA_SK(BM, BN, BK, WM, WN, ST, 1, false, false, "")
// split_k = 0: number of k-splits chosen per call (deterministic split-K, SplitArgs)
#define DG_TMA_SPLIT(BM, BN, BK, WM, WN, ST) DG_TMA_SK(BM, BN, BK, WM, WN, ST, 0, true, false, "_splitk")
// cross-stage fragment prefetch variant
// (the producer role rotates over 4 warps, kRotXP: +0.16 % at 16384^3)
#define DG_TMA_XP(BM, BN, BK, WM, WN, ST)                                                                     \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST "_xp",                                      \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST>::CONSUMER_THREADS,              \
                           (int)Cfg<BM, BN, BK, WM, WN, ST>::SMEM_BYTES, 1, 1, 0},                            \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST>, false, true, kRotXP>,                 \
             launch_tma<Cfg<BM, BN, BK, WM, WN, ST>, false, true, kRotXP>}
// split-K / plain instances with a forced launch-bounds occupancy MB (name suffix _mbMB)
#define DG_TMA_MB_SK(BM, BN, BK, WM, WN, ST, MB, SK, SPLIT, SUFFIX)                                          \
    CfgEntry{"tma_" #BM "x" #BN "x" #BK "_w" #WM "x" #WN "_s" #ST SUFFIX "_mb" #MB,                           \
             gemm_cfg_desc{BM, BN, BK, WM, WN, ST, Cfg<BM, BN, BK, WM, WN, ST, MB>::CONSUMER_THREADS,          \
                           (int)Cfg<BM, BN, BK, WM, WN, ST, MB>::SMEM_BYTES, 1, SK, 0},                       \
             (const void *)dgemm_tma_kernel<Cfg<BM, BN, BK, WM, WN, ST, MB>, SPLIT, false, kRotXP>,            \
             launch_tma<Cfg<BM, BN, BK, WM, WN, ST, MB>, SPLIT, false, kRotXP>}
#define DG_TMA_SPLIT_MB(BM, BN, BK, WM, WN, ST, MB) DG_TMA_MB_SK(BM, BN, BK, WM, WN, ST, MB, 0, true, "_splitk")
#define DG_TMA_MB(BM, BN, BK, WM, WN, ST, MB) DG_TMA_MB_SK(BM, BN, BK, WM, WN, ST, MB, 1, false, "")
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
