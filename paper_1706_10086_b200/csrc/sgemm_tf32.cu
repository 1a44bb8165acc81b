// sgemm_tf32.cu -- single-precision GEMM C = alpha*A*B + beta*C on the 5th-generation
// tensor cores (the paper's second precision, Figs. 3/7/8, Tab. 4).
//
// sm_100a has no FP32 tensor MMA; tcgen05.mma kind::tf32 multiplies 19-bit (tf32)
// operands exactly into an FP32 accumulator held in TMEM.  FP32-level accuracy comes from
// the 3xTF32 split: x = x_hi + x_lo with x_hi = rn_tf32(x), x_lo = rn_tf32(x - x_hi), and
//     A*B ~ A_lo*B_hi + A_hi*B_lo + A_hi*B_hi          (A_lo*B_lo, ~2^-22 |a||b|, dropped)
// all three products accumulated into the same TMEM accumulator.
//
// Pipeline (one CTA per 128 x BN tile of C, warp-specialised, Blackwell-native):
//   warp 0 lane 0 : TMA producer -- per 32-deep k-stage, A_hi/A_lo boxes (128 rows x 128 B)
//                   and B^T_hi/B^T_lo boxes (BN rows x 128 B), all K-major with the 128-byte
//                   swizzle, into a STAGES ring (full/empty mbarriers)
//   warp 1        : allocates BN TMEM columns; lane 0 issues tcgen05.mma (M=128, N=BN,
//                   K=8) from shared-memory descriptors, tcgen05.commit frees each stage and
//                   finally signals the epilogue
//   warps 2..5    : epilogue -- tcgen05.ld 32x32b (warp w reads TMEM lanes 32*(w%4)..),
//                   acc = acc_hihi + acc_corr (two TMEM accumulators),
//                   C = alpha*acc + beta*C, row-wise 64-byte stores
// The split is a separate bandwidth-bound pass into library workspace (row pitch padded to
// 16 bytes, so any A/B layout reaches the TMA kernel); it also transposes B, so both UMMA
// operands are K-major (fp32/tf32 MN-major operands would need the 32-byte-atom swizzle).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/gemm_f64.h"
#include "dgemm_kernels.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "launch.cuh"

namespace dg {

int make_tmap_f32(CUtensorMap *map, const float *ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                  int box_rows);

namespace f32 {

// Epilogue of 16 consecutive columns of one row (one lane per row, TMEM lane = row):
// C = alpha * (hi-chain + correction-chain) + beta * C.  With a 16-byte aligned row and all 16
// columns inside N the thread moves them with four 128-bit accesses instead of sixteen 32-bit.
__device__ __forceinline__ void store_row16(float *crow, int col, int N, const uint32_t (&v)[16],
                                            const uint32_t (&w)[16], float alpha, float beta, bool vec) {
    float o[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) o[e] = __uint_as_float(v[e]) + __uint_as_float(w[e]);
    if (vec && col + 15 < N) {
        float4 *p = reinterpret_cast<float4 *>(crow + col);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float4 r;
            if (beta != 0.0f) {
                const float4 c = p[u];
                r = make_float4(fmaf(alpha, o[4 * u], beta * c.x), fmaf(alpha, o[4 * u + 1], beta * c.y),
                                fmaf(alpha, o[4 * u + 2], beta * c.z), fmaf(alpha, o[4 * u + 3], beta * c.w));
            } else {
                r = make_float4(alpha * o[4 * u], alpha * o[4 * u + 1], alpha * o[4 * u + 2], alpha * o[4 * u + 3]);
            }
            p[u] = r;
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e)
        if (col + e < N) crow[col + e] = (beta != 0.0f) ? fmaf(alpha, o[e], beta * crow[col + e]) : alpha * o[e];
}

constexpr int BM = 128;
constexpr int UMMA_K = 8;

// BK = 32 fp32 per k-stage row (128 B, 128-byte swizzle) or 16 (64 B, 64-byte swizzle)
template <int BN_, int BK_, int STAGES_>
struct Cfg {
    static constexpr int BN = BN_, BK = BK_, STAGES = STAGES_;
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "UMMA N for M=128: multiple of 16, <= 256");
    static_assert(BK == 32 || BK == 16, "k-stage row = one 128-byte or 64-byte swizzle row");
    static constexpr uint32_t ROW_BYTES = BK * 4;                // 128 or 64
    static constexpr uint32_t SBO = 8 * ROW_BYTES;               // 8-row core-matrix group stride
    static constexpr uint32_t LAYOUT = BK == 32 ? 2u : 4u;       // UMMA SWIZZLE_128B / SWIZZLE_64B
    static constexpr uint32_t A_BYTES = BM * BK * 4;            // one of hi / lo
    static constexpr uint32_t B_BYTES = BN * BK * 4;            // BN rows of B^T, one of hi / lo
    static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    // two FP32 accumulators of BN columns each: hi*hi and the lo correction terms
    static constexpr uint32_t TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 :
                                          (2 * BN) <= 256 ? 256 : 512;
    static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int THREADS = 192;   // 6 warps
};

// ---- tcgen05 / UMMA wrappers ---------------------------------------------------------
// Shared-memory matrix descriptor (sm_100 UMMA): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset [49,52), layout type [61,64)
// (2 = 128-byte swizzle).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Instruction descriptor, kind::tf32: D f32 [4,6)=1, A tf32 [7,10)=2, B tf32 [10,13)=2,
// A K-major [15]=0, B K-major [16]=0, N>>3 [17,23), M>>4 [24,29).
template <int N>
__device__ __forceinline__ constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_nohint(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                                   uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    sgemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                        const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, int M,
                        int N, int K, float alpha, float beta, float *__restrict__ Cm, int64_t ldc, int group_m) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(base_ptr + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;
    uint64_t *tmem_full = empty + C::STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + C::BN - 1) / C::BN;
    int tm, tn;
    tile_coords(blockIdx.x, tiles_m, tiles_n, group_m, tm, tn);
    const int m0 = tm * BM, n0 = tn * C::BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int BK = C::BK;
    const int KT = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) {   // TMEM allocation by one full warp
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // PDL: setup above overlapped the previous kernel; memory from here on
    griddep_launch();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            tma_prefetch_desc(&tmAh);
            tma_prefetch_desc(&tmAl);
            tma_prefetch_desc(&tmBh);
            tma_prefetch_desc(&tmBl);
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % C::STAGES;
                if (kt >= C::STAGES) mbar_wait(&empty[s], ((kt / C::STAGES) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                uint8_t *st = base_ptr + s * C::STAGE_BYTES;
                const int k = kt * BK;
                tma_load_2d_nohint(st, &tmAh, k, m0, &full[s]);
                tma_load_2d_nohint(st + C::A_BYTES, &tmAl, k, m0, &full[s]);
                uint8_t *sb = st + 2 * C::A_BYTES;
                tma_load_2d_nohint(sb, &tmBh, k, n0, &full[s]);
                tma_load_2d_nohint(sb + C::B_BYTES, &tmBl, k, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t idesc = idesc_tf32<C::BN>();
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % C::STAGES;
                mbar_wait(&full[s], (kt / C::STAGES) & 1);
                tc_fence_after();
                const uint32_t sa = base + s * C::STAGE_BYTES;
                const uint32_t sb = sa + 2 * C::A_BYTES;
                // hi*hi chain first (same accumulator back to back), then the correction terms
                // (~2^-11 of the main term) into their own accumulator, so the tensor core's FP32
                // accumulation of the large hi*hi sum does not swallow them
#pragma unroll
                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                    // K-major, rows of 128 B (32 k), 8-row groups 1024 B apart (SBO); the
                    // 8-deep k-step advances the start address by 32 B inside the swizzle atom
                    const uint64_t a_hi = umma_desc(sa + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_hi = umma_desc(sb + kk * 32, 0, C::SBO, C::LAYOUT);
                    umma_tf32(tmem, a_hi, b_hi, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
                }
#pragma unroll
                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                    const uint64_t a_hi = umma_desc(sa + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t a_lo = umma_desc(sa + C::A_BYTES + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_hi = umma_desc(sb + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_lo = umma_desc(sb + C::B_BYTES + kk * 32, 0, C::SBO, C::LAYOUT);
                    umma_tf32(tmem + C::BN, a_lo, b_hi, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
                    umma_tf32(tmem + C::BN, a_hi, b_lo, idesc, 1u);
                }
                umma_commit(&empty[s]);   // stage s free once these MMAs have read it
            }
            umma_commit(tmem_full);       // accumulator complete
        }
    } else {
        // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31
        const int q = warp & 3;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = m0 + q * 32 + lane;
        float *crow = Cm + (int64_t)row * ldc;
        const bool row_ok = row < M;
        const bool vec = ((reinterpret_cast<uintptr_t>(Cm) & 15) == 0) && (ldc % 4 == 0);
#pragma unroll 1
        for (int c = 0; c < C::BN; c += 16) {
            uint32_t v[16], w[16];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(C::BN + c), w);
            if (KT == 0) {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0u;
            }
            if (row_ok) store_row16(crow, n0 + c, N, v, w, alpha, beta, vec);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(C::TMEM_COLS)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a 256 x BN tile
// with M=256 UMMAs issued by the leader CTA.  Each CTA stages its own 128 rows of A and its
// half (BN/2 rows) of B^T; the pair's tensor cores read both halves, so the shared-memory
// operand traffic per SM is A 4 KB + B 4 KB per K=8 step instead of 4 + 8 KB at N=256 on one
// SM.  Both CTAs' TMA bytes complete on the leader's full barrier (arrivals: leader
// expect_tx + peer remote arrive); the leader's tcgen05.commit multicasts to both CTAs'
// empty / accumulator barriers; each CTA's epilogue reads its own 128 TMEM lanes.
template <int BN_, int BK_, int STAGES_>
struct Cfg2 {
    static constexpr int BN = BN_, BK = BK_, STAGES = STAGES_, BN_HALF = BN_ / 2;
    static_assert(BN % 32 == 0 && BN >= 64 && BN <= 256, "UMMA N for M=256 (2 CTAs): multiple of 16, <= 256");
    static_assert(BK == 32 || BK == 16, "k-stage row = one 128-byte or 64-byte swizzle row");
    static constexpr uint32_t SBO = 8 * BK * 4;
    static constexpr uint32_t LAYOUT = BK == 32 ? 2u : 4u;
    static constexpr uint32_t A_BYTES = 128 * BK * 4;        // this CTA's 128 rows, one of hi / lo
    static constexpr uint32_t B_BYTES = BN_HALF * BK * 4;    // this CTA's half of B^T, one of hi / lo
    static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr uint32_t TMEM_COLS = (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
    static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int THREADS = 192;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_remote_arrive(uint64_t *bar, uint32_t cta) {
    asm volatile(
        "{\n"
        ".reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                                 uint64_t *leader_bar_local) {
    // the mbarrier address with the peer bit cleared names the leader CTA's barrier
    const uint32_t bar = smem_u32(leader_bar_local) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

template <class C>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C::THREADS, 1)
    sgemm_3xtf32_2sm_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                            const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, int M,
                            int N, int K, float alpha, float beta, float *__restrict__ Cm, int64_t ldc, int group_m) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(base_ptr + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;
    uint64_t *tmem_full = empty + C::STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const uint32_t rank = cluster_ctarank();
    const bool leader = (rank == 0);
    const int tiles_m = (M + 255) / 256, tiles_n = (N + C::BN - 1) / C::BN;
    int tm, tn;
    tile_coords(blockIdx.x >> 1, tiles_m, tiles_n, group_m, tm, tn);
    const int my_m0 = tm * 256 + (int)rank * 128;          // this CTA's 128 rows of A / C
    const int n0 = tn * C::BN;
    const int my_n0 = n0 + (int)rank * C::BN_HALF;          // this CTA's half of B^T
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int BK = C::BK;
    const int KT = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 2);    // leader's expect_tx arrive + the peer's remote arrive
            mbar_init(&empty[s], 1);   // the leader's multicast commit
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();   // both CTAs: barriers initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // PDL: setup above overlapped the previous kernel; memory from here on
    griddep_launch();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer (both CTAs)
            tma_prefetch_desc(&tmAh);
            tma_prefetch_desc(&tmAl);
            tma_prefetch_desc(&tmBh);
            tma_prefetch_desc(&tmBl);
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % C::STAGES;
                if (kt >= C::STAGES) mbar_wait(&empty[s], ((kt / C::STAGES) - 1) & 1);
                if (leader)
                    mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
                else
                    mbar_remote_arrive(&full[s], 0);
                uint8_t *st = base_ptr + s * C::STAGE_BYTES;
                const int k = kt * BK;
                tma_load_2d_pair(st, &tmAh, k, my_m0, &full[s]);
                tma_load_2d_pair(st + C::A_BYTES, &tmAl, k, my_m0, &full[s]);
                uint8_t *sb = st + 2 * C::A_BYTES;
                tma_load_2d_pair(sb, &tmBh, k, my_n0, &full[s]);
                tma_load_2d_pair(sb + C::B_BYTES, &tmBl, k, my_n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {   // ---------------- MMA issuer (leader CTA only)
            constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(C::BN >> 3) << 17) |
                                       ((uint32_t)(256 >> 4) << 24);
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % C::STAGES;
                mbar_wait(&full[s], (kt / C::STAGES) & 1);
                tc_fence_after();
                const uint32_t sa = base + s * C::STAGE_BYTES;
                const uint32_t sb = sa + 2 * C::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                    const uint64_t a_hi = umma_desc(sa + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_hi = umma_desc(sb + kk * 32, 0, C::SBO, C::LAYOUT);
                    umma_tf32_pair(tmem, a_hi, b_hi, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
                }
#pragma unroll
                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                    const uint64_t a_hi = umma_desc(sa + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t a_lo = umma_desc(sa + C::A_BYTES + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_hi = umma_desc(sb + kk * 32, 0, C::SBO, C::LAYOUT);
                    const uint64_t b_lo = umma_desc(sb + C::B_BYTES + kk * 32, 0, C::SBO, C::LAYOUT);
                    umma_tf32_pair(tmem + C::BN, a_lo, b_hi, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
                    umma_tf32_pair(tmem + C::BN, a_hi, b_lo, idesc, 1u);
                }
                umma_commit_pair(&empty[s]);
            }
            umma_commit_pair(tmem_full);
        }
    } else {
        // ---------------- epilogue warps 2..5 (both CTAs): own 128 TMEM lanes
        const int q = warp & 3;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = my_m0 + q * 32 + lane;
        float *crow = Cm + (int64_t)row * ldc;
        const bool row_ok = row < M;
        const bool vec = ((reinterpret_cast<uintptr_t>(Cm) & 15) == 0) && (ldc % 4 == 0);
#pragma unroll 1
        for (int c = 0; c < C::BN; c += 16) {
            uint32_t v[16], w[16];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(C::BN + c), w);
            if (row_ok) store_row16(crow, n0 + c, N, v, w, alpha, beta, vec);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();   // the peer's smem / TMEM stay valid until both CTAs are done
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(C::TMEM_COLS)
                     : "memory");
    }
}

// x -> (rn_tf32(x), rn_tf32(x - rn_tf32(x))), packed rows of pitch ldo.
__global__ void split_tf32_kernel(const float *__restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                  float *__restrict__ hi, float *__restrict__ lo, int64_t ldo) {
    griddep_wait();
    griddep_launch();
    const int64_t total = rows * cols;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cols, c = idx - r * cols;
        const float x = X[r * ldx + c];
        uint32_t h, l;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
        const float rest = x - __uint_as_float(h);
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(rest));
        hi[r * ldo + c] = __uint_as_float(h);
        lo[r * ldo + c] = __uint_as_float(l);
    }
}

// B (K x N, ldx) -> B^T hi / lo (N x K, pitch ldo): 32 x 32 tiles through shared memory so
// both the reads and the writes are coalesced.
__global__ void split_tf32_t_kernel(const float *__restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                    float *__restrict__ hiT, float *__restrict__ loT, int64_t ldo) {
    __shared__ float tile[32][33];
    griddep_wait();
    griddep_launch();
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t r = r0 + ty + i, c = c0 + tx;
        tile[ty + i][tx] = (r < rows && c < cols) ? X[r * ldx + c] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t c = c0 + ty + i, r = r0 + tx;   // output row = c (n), column = r (k)
        if (c < cols && r < rows) {
            const float x = tile[tx][ty + i];
            uint32_t h, l;
            asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
            const float rest = x - __uint_as_float(h);
            asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(rest));
            hiT[c * ldo + r] = __uint_as_float(h);
            loT[c * ldo + r] = __uint_as_float(l);
        }
    }
}

__global__ void scale_f32_kernel(int M, int N, float beta, float *__restrict__ Cm, int64_t ldc) {
    griddep_wait();
    griddep_launch();
    const int64_t total = (int64_t)M * N;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / N, j = idx % N;
        float *p = Cm + i * ldc + j;
        *p = (beta == 0.0f) ? 0.0f : beta * *p;
    }
}

struct F32Cfg {
    const char *name;
    int bn, bk, stages;
    uint32_t smem;
    const void *kernel;
    void (*launch)(dim3, cudaStream_t, const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                   const CUtensorMap &, int, int, int, float, float, float *, int64_t, int);
    int ctas = 1;   // 2: CTA pair (cta_group::2), 256-row tiles
};

template <class C>
static void launch_f32(dim3 grid, cudaStream_t st, const CUtensorMap &a, const CUtensorMap &b, const CUtensorMap &c,
                       const CUtensorMap &d, int M, int N, int K, float alpha, float beta, float *Cm, int64_t ldc,
                       int group_m) {
    (void)launch_k(sgemm_3xtf32_kernel<C>, grid, dim3(C::THREADS), C::SMEM_BYTES, st, a, b, c, d, M, N, K, alpha,
                   beta, Cm, ldc, group_m);   // errors surface through cudaGetLastError at the call site
}

#define F32CFG(BN, BK, ST)                                                                                   \
    F32Cfg{"tf32x3_128x" #BN "x" #BK "_s" #ST, BN, BK, ST, Cfg<BN, BK, ST>::SMEM_BYTES,                       \
           (const void *)sgemm_3xtf32_kernel<Cfg<BN, BK, ST>>, launch_f32<Cfg<BN, BK, ST>>}

template <class C>
static void launch_f32_pair(dim3 grid, cudaStream_t st, const CUtensorMap &a, const CUtensorMap &b,
                            const CUtensorMap &c, const CUtensorMap &d, int M, int N, int K, float alpha, float beta,
                            float *Cm, int64_t ldc, int group_m) {
    (void)launch_k(sgemm_3xtf32_2sm_kernel<C>, grid, dim3(C::THREADS), C::SMEM_BYTES, st, a, b, c, d, M, N, K,
                   alpha, beta, Cm, ldc, group_m);
}

// pair configurations: bm = 256 (two CTAs), the A box is 128 rows, the B box BN/2 rows
#define F32CFG2(BN, BK, ST)                                                                                  \
    F32Cfg{"tf32x3_2sm_256x" #BN "x" #BK "_s" #ST, BN, BK, ST, Cfg2<BN, BK, ST>::SMEM_BYTES,                  \
           (const void *)sgemm_3xtf32_2sm_kernel<Cfg2<BN, BK, ST>>, launch_f32_pair<Cfg2<BN, BK, ST>>, 2}

static const F32Cfg k_f32_cfgs[] = {
    F32CFG(128, 32, 3),
    F32CFG(128, 16, 6),
    F32CFG(256, 32, 2),
    F32CFG(256, 16, 4),
    F32CFG2(256, 32, 3),
    F32CFG2(256, 16, 6),
};
static constexpr int kNumF32Cfgs = sizeof(k_f32_cfgs) / sizeof(k_f32_cfgs[0]);
static constexpr int kDefaultF32 = 0;   // tf32x3_128x128x32_s3
static constexpr int kWideF32 = 3;      // tf32x3_128x256x16_s4
static constexpr int kPairF32 = 4;      // tf32x3_2sm_256x256x32_s3 (measured best at 8192 / 16384)

struct Ws {
    float *buf = nullptr;
    size_t cap = 0;   // floats
};
static std::mutex g_mu;
static std::map<std::pair<int, cudaStream_t>, Ws> g_ws;
static std::map<int, bool> g_attr;   // (device * 64 + cfg) -> smem attribute set

static std::vector<std::pair<int, float *>> g_retired;   // (device, buffer) kept for captured graphs

// Per-(device, stream) split workspace.  As in gemm_f64.cu: growth retires the old buffer
// instead of freeing it (a CUDA graph captured from an earlier call may still use it); only
// gemm_workspace_release() frees.
static float *workspace(cudaStream_t st, size_t floats) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    Ws &w = g_ws[{dev, st}];
    if (w.cap < floats) {
        const size_t want = std::max(floats, w.cap + w.cap / 4);
        float *p = nullptr;
        if (cudaMalloc(&p, want * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        if (w.buf) g_retired.push_back({dev, w.buf});
        w.buf = p;
        w.cap = want;
    }
    return w.buf;
}

// frees the current device's FP32 workspace (the caller has synchronized the device)
void workspace_release_f32() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if (it->first.first == dev) {
            cudaFree(it->second.buf);
            it = g_ws.erase(it);
        } else {
            ++it;
        }
    }
    for (auto it = g_retired.begin(); it != g_retired.end();) {
        if (it->first == dev) {
            cudaFree(it->second);
            it = g_retired.erase(it);
        } else {
            ++it;
        }
    }
}

static bool overlaps(const void *p, int64_t rows, int64_t cols, int64_t ld, const void *q, int64_t qrows,
                     int64_t qcols, int64_t qld) {
    if (!p || !q || rows <= 0 || cols <= 0 || qrows <= 0 || qcols <= 0) return false;
    const char *p0 = (const char *)p, *p1 = p0 + ((rows - 1) * ld + cols) * 4;
    const char *q0 = (const char *)q, *q1 = q0 + ((qrows - 1) * qld + qcols) * 4;
    return p0 < q1 && q0 < p1;
}

static int impl(int64_t M, int64_t N, int64_t K, float alpha, const float *A, int64_t lda, const float *B,
                int64_t ldb, float beta, float *C, int64_t ldc, cudaStream_t st, int cfg_id = -1) {
    clear_error();
    if (M < 0 || N < 0 || K < 0)
        return set_error(GEMM_ERR_ARG, "M=%lld N=%lld K=%lld must be >= 0", (long long)M, (long long)N, (long long)K);
    const int64_t lim = (int64_t(1) << 31) - 4096;   // int32 tile arithmetic and TMA coordinates
    if (M > lim || N > lim || K > lim) return set_error(GEMM_ERR_UNSUPPORTED, "M, N, K must be < 2^31");
    if (lda < std::max<int64_t>(1, K)) return set_error(GEMM_ERR_ARG, "lda=%lld must be >= max(1,K)", (long long)lda);
    if (ldb < std::max<int64_t>(1, N)) return set_error(GEMM_ERR_ARG, "ldb=%lld must be >= max(1,N)", (long long)ldb);
    if (ldc < std::max<int64_t>(1, N)) return set_error(GEMM_ERR_ARG, "ldc=%lld must be >= max(1,N)", (long long)ldc);
    if (M == 0 || N == 0) return GEMM_OK;
    if (!C) return set_error(GEMM_ERR_ARG, "C is NULL with M*N > 0");
    if ((uintptr_t)C % 4) return set_error(GEMM_ERR_ARG, "C is not 4-byte aligned");
    const bool need_ab = (alpha != 0.0f && K > 0);
    if (need_ab) {
        if (!A) return set_error(GEMM_ERR_ARG, "A is NULL with alpha != 0, K > 0");
        if (!B) return set_error(GEMM_ERR_ARG, "B is NULL with alpha != 0, K > 0");
        if ((uintptr_t)A % 4 || (uintptr_t)B % 4) return set_error(GEMM_ERR_ARG, "A/B not 4-byte aligned");
        if (overlaps(C, M, N, ldc, A, M, K, lda)) return set_error(GEMM_ERR_ARG, "C overlaps A");
        if (overlaps(C, M, N, ldc, B, K, N, ldb)) return set_error(GEMM_ERR_ARG, "C overlaps B");
    }
    if (!need_ab) {
        if (beta == 1.0f) return GEMM_OK;
        const int64_t total = M * N;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        return cuda_check(launch_k(scale_f32_kernel, dim3(blocks), dim3(256), 0, st, (int)M, (int)N, beta, C, ldc),
                          "scale_f32_kernel launch");
    }
    if (cfg_id < -1 || cfg_id >= kNumF32Cfgs)
        return set_error(GEMM_ERR_ARG, "f32 cfg_id=%d out of range [-1, %d)", cfg_id, kNumF32Cfgs);
    // default: CTA-pair 256 x 256 tiles for large problems (least shared-memory operand
    // traffic per FLOP), 128 x 256 for medium, 128 x 128 when N is small
    const int pick = (M >= 512 && N >= 256) ? kPairF32 : (N > 128 ? kWideF32 : kDefaultF32);
    const F32Cfg &cf = k_f32_cfgs[cfg_id >= 0 ? cfg_id : pick];
    // split A and B into tf32 hi / lo in workspace, row pitch padded to 16 bytes
    const int64_t ka = (K + 3) & ~int64_t(3);
    const size_t a_sz = (size_t)M * ka, b_sz = (size_t)N * ka;   // A and B^T, both K-major
    float *ws = workspace(st, 2 * a_sz + 2 * b_sz + 64);
    if (!ws) return set_error(GEMM_ERR_ALLOC, "sgemm workspace of %zu bytes", (2 * a_sz + 2 * b_sz) * 4);
    float *Ah = ws, *Al = Ah + a_sz, *Bh = Al + a_sz, *Bl = Bh + b_sz;
    {
        const int64_t ta = M * K, tb = K * N;
        int rc = cuda_check(launch_k(split_tf32_kernel, dim3((unsigned)std::min<int64_t>((ta + 255) / 256, 148 * 32)),
                                     dim3(256), 0, st, A, lda, M, K, Ah, Al, ka),
                            "split_tf32_kernel launch");
        if (rc) return rc;
        (void)tb;
        dim3 tgrid((unsigned)((N + 31) / 32), (unsigned)((K + 31) / 32));
        rc = cuda_check(launch_k(split_tf32_t_kernel, tgrid, dim3(32, 8), 0, st, B, ldb, K, N, Bh, Bl, ka),
                        "split_tf32_t_kernel launch");
        if (rc) return rc;
    }
    CUtensorMap mAh, mAl, mBh, mBl;
    const int bbox = cf.ctas == 2 ? cf.bn / 2 : cf.bn;   // B^T rows per CTA
    int rc = make_tmap_f32(&mAh, Ah, M, K, ka, cf.bk, BM);
    if (!rc) rc = make_tmap_f32(&mAl, Al, M, K, ka, cf.bk, BM);
    if (!rc) rc = make_tmap_f32(&mBh, Bh, N, K, ka, cf.bk, bbox);
    if (!rc) rc = make_tmap_f32(&mBl, Bl, N, K, ka, cf.bk, bbox);
    if (rc) return rc;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const int key = dev * 64 + (int)(&cf - k_f32_cfgs);
        if (!g_attr[key]) {
            rc = cuda_check(cudaFuncSetAttribute(cf.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cf.smem),
                            "cudaFuncSetAttribute(sgemm)");
            if (rc) return rc;
            g_attr[key] = true;
        }
    }
    const int64_t bm = (int64_t)BM * cf.ctas;
    const int64_t tiles = ((M + bm - 1) / bm) * ((N + cf.bn - 1) / cf.bn) * cf.ctas;   // CTAs
    if (tiles > 0x7FFFFFFF) return set_error(GEMM_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)tiles);
    cf.launch(dim3((unsigned)tiles), st, mAh, mAl, mBh, mBl, (int)M, (int)N, (int)K, alpha, beta, C, ldc, 8);
    return cuda_check(cudaGetLastError(), "sgemm_3xtf32_kernel launch");
}

}  // namespace f32
}  // namespace dg

extern "C" {

int gemm_f32(int64_t M, int64_t N, int64_t K, float alpha, const float *A, int64_t lda, const float *B, int64_t ldb,
             float beta, float *C, int64_t ldc) {
    return dg::f32::impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (cudaStream_t)0);
}

int gemm_f32_stream(int64_t M, int64_t N, int64_t K, float alpha, const float *A, int64_t lda, const float *B,
                    int64_t ldb, float beta, float *C, int64_t ldc, void *stream) {
    return dg::f32::impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (cudaStream_t)stream);
}

int gemm_f32_cfg(int64_t M, int64_t N, int64_t K, float alpha, const float *A, int64_t lda, const float *B,
                 int64_t ldb, float beta, float *C, int64_t ldc, int cfg_id, void *stream) {
    return dg::f32::impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (cudaStream_t)stream, cfg_id);
}

int gemm_f32_num_cfgs(void) { return dg::f32::kNumF32Cfgs; }

int gemm_f32_cfg_name(int cfg_id, char *buf, int len) {
    dg::clear_error();
    if (cfg_id < 0 || cfg_id >= dg::f32::kNumF32Cfgs) return dg::set_error(GEMM_ERR_ARG, "f32 cfg_id out of range");
    if (!buf || len <= 0) return dg::set_error(GEMM_ERR_ARG, "buf is NULL or len <= 0");
    snprintf(buf, (size_t)len, "%s", dg::f32::k_f32_cfgs[cfg_id].name);
    return GEMM_OK;
}

}  // extern "C"
