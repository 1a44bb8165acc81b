// dgemm_kernels.cuh -- sm_100a FP64 GEMM kernels: C = alpha*A*B + beta*C, row-major.
//
// PAPER.md Eq. (1); tiled algorithm Fig. 2 P:102-107 and §2.1 P:131-133:
// "calculate one tile of the matrix C per Alpaka block ... Every element stores
// the partial result of alpha*A*B in element local memory".  The paper's tunables
// (tile size T and elements per thread, Listing 1) become the
// compile-time tile parameters of Cfg below:
//
//   BM x BN   CTA tile of C            (the paper's block tile t*T)
//   BK        k-depth of one pipeline stage (multiple of 16)
//   WM x WN   warp tile; E = WM*WN/32 accumulators per thread
//             (the paper's "elements per thread", its element layer)
//   STAGES    depth of the shared-memory ring (the paper's A/B tile cache, Eq. (5))
//
// B200 design:
// * a1 work division: one CTA per BM x BN tile of C, grouped ("swizzled") raster of
//   group_m tile rows so that CTAs resident together share A and B panels in L2.
// * a2 staging: A tile (BM x 16 doubles per k-group, 128-byte rows) and B tile
//   (16 x 16-double boxes) land in shared memory through TMA with the 128-byte
//   swizzle (16-byte chunk index ^= row & 7), driven by one producer warp and a
//   ring of full/empty mbarriers (tma kernel), or through cp.async into the same
//   swizzled layout (generic kernel, any alignment / leading dimension).
// * a3 tile MMA: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the only native FP64 MMA of
//   sm_100a; tcgen05 has no f64 kind).  Fragments are read with 16-byte LDS through
//   a k-permutation chosen so that, under the TMA 128-byte swizzle, both the A and
//   the B fragment loads are free of bank conflicts (see kperm_chunk below).
// * a4 epilogue: alpha once on the finished sum, beta*C read only when beta != 0,
//   4 contiguous doubles per thread -> one 256-bit STG per (m-block, n-pair).
#pragma once
#include <cstdint>
#include <cuda.h>

#include "ptx.cuh"

namespace dg {

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_ = 0>
struct Cfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
    static_assert(BM % WM == 0 && BN % WN == 0, "warp tiles must tile the CTA tile");
    static_assert(WM % 8 == 0 && WN % 16 == 0, "warp tile: m-blocks of 8, n-pairs of 16");
    static_assert(BK % 16 == 0, "BK is a multiple of the 16-wide k-permutation group");
    static_assert(BM <= 256, "TMA box rows <= 256");
    static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
    static constexpr int CONSUMER_WARPS = WARPS_M * WARPS_N;
    static constexpr int CONSUMER_THREADS = CONSUMER_WARPS * 32;
    static constexpr int MB = WM / 8;    // 8-row m-blocks per warp
    static constexpr int NP = WN / 16;   // 16-column n-pairs per warp (two 8-wide n-blocks each)
    static constexpr int KG = BK / 16;   // 16-deep k-groups per stage
    static constexpr int E = WM * WN / 32;
    // shared-memory layout of one stage: A sub-tiles [KG][BM][16], then B boxes [KG][BN/16][16][16]
    static constexpr uint32_t A_SUB = BM * 128;
    static constexpr uint32_t A_BYTES = KG * A_SUB;
    static constexpr uint32_t B_BOX = 16 * 128;
    static constexpr uint32_t B_KG = (BN / 16) * B_BOX;
    static constexpr uint32_t B_BYTES = KG * B_KG;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t BAR_BYTES = 2 * STAGES * 8;
    static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + BAR_BYTES + 1024;  // +1024: manual alignment
    // two CTAs per SM when shared memory allows it (227 KB per SM usable, ~1 KB reserved per CTA)
    // MINB_ > 0: the launch-bounds occupancy is forced (3 CTAs per SM for the E = 8 tiles, whose
    // one-per-SM register budget would otherwise stop at two)
    static constexpr int MINB = MINB_;
    static constexpr int MIN_BLOCKS = MINB_ > 0 ? MINB_ : (2 * (SMEM_BYTES + 1024) <= 228 * 1024) ? 2 : 1;
};

// k-permutation inside a 16-deep k-group.  A thread with MMA k-index t (= lane & 3)
// and half p in {0,1} owns the 16-byte chunk c(t,p) (two consecutive k) of each
// 128-byte row; MMA slice q = 2p+s uses real k = 2*c(t,p) + s.  (t,p) -> c is a
// bijection onto 0..7, so every k of the group is used exactly once per slice set.
// With the hardware 128-byte swizzle (physical chunk = chunk ^ (row & 7)):
//  * A loads (rows g = lane>>2, chunk c(t,p)) hit 8 distinct chunks per 8-lane phase
//    because c(t,p) >> 1 is distinct over t;
//  * B loads (row k = 2c+s, chunk g) hit 8 distinct chunks per phase because
//    c(t,p) & 3 is distinct over t.
__device__ __forceinline__ int kperm_chunk(int t, int p) { return t + 4 * ((t & 1) ^ p); }

__device__ __forceinline__ void lds_v2(uint32_t addr, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

// Per-thread constant offsets for fragment loads.
template <class C>
struct FragOffsets {
    uint32_t a[2];      // A: byte offset within a k-group sub-tile, for p = 0, 1 (includes warp row)
    uint32_t b[2][2];   // B: byte offset within a k-group, for (p, s) (includes warp n-pair base)
    __device__ __forceinline__ FragOffsets(int warp_m, int warp_n, int lane) {
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int c = kperm_chunk(t, p);
            a[p] = (uint32_t)((warp_m * C::WM + g) * 128 + ((c ^ g) << 4));
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int k = 2 * c + s;
                b[p][s] = (uint32_t)((warp_n * C::WN / 16) * C::B_BOX + k * 128 + ((g ^ (k & 7)) << 4));
            }
        }
    }
};

// A warp hands a ring slot back to the producer.  Its fragment loads of the slot are
// generic-proxy reads and the refill is an async-proxy (TMA) write, so every lane fences
// (fence.proxy.async: its prior shared-memory accesses are performed and ordered before
// async-proxy accesses) before lane 0 arrives on the slot's `empty` barrier.  Without the
// fence the arrive can overtake the warp's last LDS of the slot (ptxas places it before the
// stage's last DMMAs); measured: once the refill was issued by a warp other than the laggard,
// split-K results picked up k-steps from the next lap of the ring.
__device__ __forceinline__ void release_slot(uint64_t *empty_bar, int lane) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);
}

// One pipeline stage of the warp's register-blocked tile multiply (row a3).
template <class C>
__device__ __forceinline__ void mma_stage(uint32_t sA, uint32_t sB, const FragOffsets<C> &fo,
                                          double (&acc)[C::MB][C::NP][2][2]) {
#pragma unroll
    for (int kg = 0; kg < C::KG; ++kg) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            double a[C::MB][2];
            double b[C::NP][2][2];
#pragma unroll
            for (int mb = 0; mb < C::MB; ++mb)
                lds_v2(sA + kg * C::A_SUB + mb * 1024 + fo.a[p], a[mb][0], a[mb][1]);
#pragma unroll
            for (int np = 0; np < C::NP; ++np)
#pragma unroll
                for (int s = 0; s < 2; ++s)
                    lds_v2(sB + kg * C::B_KG + np * C::B_BOX + fo.b[p][s], b[np][s][0], b[np][s][1]);
#pragma unroll
            for (int s = 0; s < 2; ++s)
#pragma unroll
                for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
                    for (int np = 0; np < C::NP; ++np)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            dmma_m8n8k4(acc[mb][np][j][0], acc[mb][np][j][1], a[mb][s], b[np][s][j]);
        }
    }
}

// The same tile multiply split into "halves" (one k-group half p: 2 MMA slices) so that a
// caller can keep the next half's fragments in flight while the current half's DMMAs
// issue -- across the stage boundary too (cross-stage prefetch, XP kernels).
template <class C>
struct Frag {
    double a[C::MB][2];
    double b[C::NP][2][2];
};

template <class C>
__device__ __forceinline__ void load_half(uint32_t sA, uint32_t sB, int h, const FragOffsets<C> &fo, Frag<C> &f) {
    const int kg = h >> 1, p = h & 1;
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb) lds_v2(sA + kg * C::A_SUB + mb * 1024 + fo.a[p], f.a[mb][0], f.a[mb][1]);
#pragma unroll
    for (int np = 0; np < C::NP; ++np)
#pragma unroll
        for (int s = 0; s < 2; ++s)
            lds_v2(sB + kg * C::B_KG + np * C::B_BOX + fo.b[p][s], f.b[np][s][0], f.b[np][s][1]);
}

template <class C>
__device__ __forceinline__ void mma_half(const Frag<C> &f, double (&acc)[C::MB][C::NP][2][2]) {
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
            for (int np = 0; np < C::NP; ++np)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    dmma_m8n8k4(acc[mb][np][j][0], acc[mb][np][j][1], f.a[mb][s], f.b[np][s][j]);
}

// Epilogue (row a4): C = alpha*acc + beta*C, each C element read (beta != 0) and written once.
// Thread (g, t) of an (m-block, n-pair) owns row g and the 4 contiguous columns 4t..4t+3:
// acc[mb][np][j][i] is real column 4t + 2i + j of the n-pair; v = {acc[..][0][0],
// acc[..][1][0], acc[..][0][1], acc[..][1][1]} are columns col..col+3.
__device__ __forceinline__ void epilogue_quad(const double (&v)[4], int row, int col, int M, int N, double alpha,
                                              double beta, double *__restrict__ Cm, int64_t ldc, bool vec) {
    if (row >= M) return;
    double *crow = Cm + (int64_t)row * ldc;
    if (vec && col + 3 < N) {
        double o[4];
        if (beta != 0.0) {
            double c[4];
            ldg_v4(crow + col, c[0], c[1], c[2], c[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = fma(alpha, v[e], beta * c[e]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = alpha * v[e];
        }
        stg_v4(crow + col, o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (col + e < N) {
                const double o = (beta != 0.0) ? fma(alpha, v[e], beta * crow[col + e]) : alpha * v[e];
                crow[col + e] = o;
            }
        }
    }
}

template <class C>
__device__ __forceinline__ void epilogue(const double (&acc)[C::MB][C::NP][2][2], int row0, int col0, int lane,
                                         int M, int N, double alpha, double beta, double *__restrict__ Cm,
                                         int64_t ldc, bool vec) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb) {
#pragma unroll
        for (int np = 0; np < C::NP; ++np) {
            const double v[4] = {acc[mb][np][0][0], acc[mb][np][1][0], acc[mb][np][0][1], acc[mb][np][1][1]};
            epilogue_quad(v, row0 + mb * 8 + g, col0 + np * 16 + 4 * t, M, N, alpha, beta, Cm, ldc, vec);
        }
    }
}

// floor(a * b / c) for 0 <= a, b and 0 < c: a 32-bit division when the product fits (always,
// for k-step ranges), the 64-bit one only otherwise (a long software sequence; the per-CTA
// trace put the prologue at 0.65 us)
__device__ __forceinline__ int mul_div(int a, int b, int c) {
    const unsigned long long p = (unsigned long long)(unsigned)a * (unsigned)b;
    if (p <= 0xffffffffull) return (int)((unsigned)p / (unsigned)c);
    return (int)(p / (unsigned long long)c);
}

// Grouped raster (row a1): consecutive CTAs walk group_m tile-rows column by column.
__device__ __forceinline__ void tile_coords(int bid, int tiles_m, int tiles_n, int group_m, int &tm, int &tn) {
    const int per_group = group_m * tiles_n;
    const int group = bid / per_group;
    const int first_m = group * group_m;
    const int gsize = min(group_m, tiles_m - first_m);
    const int r = bid - group * per_group;
    tm = first_m + r % gsize;
    tn = r / gsize;
}

// ------------------------------------------------------------------------------
// TMA + mbarrier kernel.  No dedicated producer warp: a separate warp would push
// the per-SMSP warp count from 2 to 3 and cap registers at 168/thread (the 64x32
// warp tile needs ~200).  Lane 0 of warp 0 is the producer: at the top of k-step kt
// it waits until every consumer warp has released the slot read at kt-1 (empty
// mbarrier) and refills it with k-step kt-1+STAGES by TMA (full mbarrier,
// expect_tx).  STAGES-1 stages stay in flight ahead of the slowest warp.
template <class C>
__device__ __forceinline__ void tma_issue_stage(uint8_t *stage_ptr, const CUtensorMap *tmA, const CUtensorMap *tmB,
                                                uint64_t *full_bar, int m0, int n0, int kt, uint64_t pol,
                                                bool md = false) {
    mbar_arrive_expect_tx(full_bar, C::STAGE_BYTES);
    uint8_t *sA = stage_ptr;
    uint8_t *sB = stage_ptr + C::A_BYTES;
    if (md) {
        // multi-dimensional maps (K % 16 == 0, N % 16 == 0; host: make_tmap_a3 / make_tmap_b4):
        // A as (16 columns, rows, k-groups), box (16, BM, KG) -> smem [kg][row][16];
        // B as (16 columns, 16 rows, 16-column panels, k-groups), box (16, 16, BN/16, KG) ->
        // smem [kg][panel][row][16] -- the same swizzled layout the 2-D boxes fill, in 2
        // instructions per stage instead of KG * (1 + BN/16)
        tma_load_3d(sA, tmA, 0, m0, kt * C::KG, full_bar, pol);
        tma_load_4d(sB, tmB, 0, 0, n0 / 16, kt * C::KG, full_bar, pol);
        return;
    }
#pragma unroll
    for (int kg = 0; kg < C::KG; ++kg) {
        const int k = kt * C::BK + kg * 16;
        tma_load_2d(sA + kg * C::A_SUB, tmA, k, m0, full_bar, pol);
#pragma unroll
        for (int c = 0; c < C::BN / 16; ++c)
            tma_load_2d(sB + kg * C::B_KG + c * C::B_BOX, tmB, n0 + 16 * c, k, full_bar, pol);
    }
}

// Deterministic split-K (row a5, small shapes): gridDim.y = splits; split s of a tile
// multiplies k-steps [s*KT/S, (s+1)*KT/S) into a raw (unscaled) partial.  Every split
// stores its partial to the workspace; the CTA that arrives last on the tile's counter
// sums the S partials in the fixed order s = 0, 1, ..., S-1 and runs the epilogue, so
// the result does not depend on which CTA finishes last.  The counter is reset by that
// CTA, leaving the workspace ready for the next launch on the same stream.
struct SplitArgs {
    int splits;        // 1 = no split
    double *ws;        // [tiles][splits][E/4][warps][32][4] doubles
    int *counters;     // [tiles], zero between launches
};

template <class C>
__device__ __forceinline__ double *partial_slot(double *ws, int64_t slot, int warp, int lane) {
    constexpr int Q = C::E / 4;   // 256-bit groups per thread
    return ws + (slot * Q * C::CONSUMER_WARPS * 32 + (int64_t)warp * 32 + lane) * 4;
}

// Sum the nseg partial tiles slot_of(0), slot_of(1), ... into acc in that fixed order
// (deterministic).  Loads are batched -- PB partials x QC 256-bit groups, at most 32 doubles
// in flight per thread, so the E = 16 instances stay within 128 registers and E = 64 within
// 255 -- and a batch is issued before any of it is added: about nseg / PB L2 round trips
// per q-chunk instead of nseg.
template <class C, int PB_MAX = 32, class SlotOf>
__device__ __forceinline__ void sum_partials(double (&acc)[C::MB][C::NP][2][2], const double *ws, int nseg,
                                             SlotOf slot_of, int warp, int lane) {
    constexpr int Q = C::E / 4;
    constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;   // doubles between q groups
    // E = 16: 2 partials x 4 quads in flight; E = 8: 4 x 2, or 2 x 2 in the 3-CTA/SM instances
    // (64 registers: the four-partial batch alone held 32 doubles)
    constexpr int PB0 = C::E >= 32 ? 1 : C::MINB >= 3 ? 2 : 32 / C::E;
    constexpr int PB = PB0 < PB_MAX ? PB0 : PB_MAX;                   // partials in flight
    constexpr int QC = Q < 8 ? Q : 8;                                  // q groups in flight
    static_assert(Q % QC == 0, "q chunking");
    double *flat = &acc[0][0][0][0];
#pragma unroll
    for (int e = 0; e < C::E; ++e) flat[e] = 0.0;
    for (int t0 = 0; t0 < nseg; t0 += PB) {
#pragma unroll
        for (int q0 = 0; q0 < Q; q0 += QC) {
            double v[PB][QC][4];
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                if (t0 + u < nseg) {
                    const double *src =
                        partial_slot<C>(const_cast<double *>(ws), slot_of(t0 + u), warp, lane) + q0 * QSTRIDE;
#pragma unroll
                    for (int q = 0; q < QC; ++q)
                        asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                                     : "=d"(v[u][q][0]), "=d"(v[u][q][1]), "=d"(v[u][q][2]), "=d"(v[u][q][3])
                                     : "l"(src + q * QSTRIDE));
                }
            }
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                if (t0 + u < nseg) {
#pragma unroll
                    for (int q = 0; q < QC; ++q)
#pragma unroll
                        for (int e = 0; e < 4; ++e) flat[4 * (q0 + q) + e] += v[u][q][e];
                }
            }
        }
    }
}

// Deterministic reduction of the nseg partial sums of one tile (split-K slices or
// stream-K segments).  Partial `seg` goes to workspace slot (tile * stride + seg); the
// CTA arriving last on the tile's counter adds the nseg partials in segment order (so the
// result is independent of arrival order), resets the counter and returns true with the
// total in acc; the others return false.
template <class C>
__device__ __forceinline__ bool partial_reduce(double (&acc)[C::MB][C::NP][2][2], double *ws, int *counters,
                                               int64_t tile, int stride, int seg, int nseg, int warp, int lane) {
    constexpr int Q = C::E / 4;
    constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;   // doubles between q groups
    double *mine = partial_slot<C>(ws, tile * stride + seg, warp, lane);
    double *flat = &acc[0][0][0][0];
#pragma unroll
    for (int q = 0; q < Q; ++q) stg_v4(mine + q * QSTRIDE, flat[4 * q], flat[4 * q + 1], flat[4 * q + 2], flat[4 * q + 3]);
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        const int old = atomicAdd(&counters[tile], 1);
        s_last = (old == nseg - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    sum_partials<C>(acc, ws, nseg, [&](int t) { return tile * stride + t; }, warp, lane);
    if (threadIdx.x == 0) counters[tile] = 0;
    return true;
}

// Split-K finish, ordered by slice (returns true if this CTA runs the epilogue: no split, or the
// last slice).  Slices 0..S-2 store their raw partial, and thread 0 publishes it with one
// red.release on the tile's counter after a CTA barrier (the barrier orders every thread's
// stores before the release) -- then the CTA exits without waiting for anything.  Slice S-1
// keeps its own partial, waits (ld.acquire) until the counter reaches S-1, and adds
// partials 0..S-2 and then its own, i.e. (((0 + p0) + p1) + ...) + p_{S-1}: the order, hence
// the bits, of summing all S partials in slice order.  The last slice's wait relies on the
// block scheduler dispatching CTAs in linear order (slices 0..S-2 of a tile have lower
// linear indices than slice S-1, gridDim.y = S), as serial split-K schemes do; the previous
// scheme (every slice stores, the last to arrive on an atomic sums) made each CTA wait for
// its atomic's round trip and the reducer re-read its own partial (per-CTA traces).
template <class C>
__device__ __forceinline__ bool split_reduce(double (&acc)[C::MB][C::NP][2][2], const SplitArgs &sk, int tile,
                                             int s, int warp, int lane, uint32_t smem_base) {
    const int S = sk.splits;
    if (S <= 1) return true;
    if constexpr (C::E >= 32) {   // large warp tiles: the last-arriver scheme (no registers to spare)
        return partial_reduce<C>(acc, sk.ws, sk.counters, tile, S, s, S, warp, lane);
    }
    constexpr int Q = C::E / 4;
    constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;
    int *ctr = sk.counters + tile;
    double *flat = &acc[0][0][0][0];
    if (s < S - 1) {
        double *mine = partial_slot<C>(sk.ws, (int64_t)tile * S + s, warp, lane);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            stg_v4(mine + q * QSTRIDE, flat[4 * q], flat[4 * q + 1], flat[4 * q + 2], flat[4 * q + 3]);
        __syncthreads();
        if (threadIdx.x == 0) red_release_add(ctr, 1);
        return false;
    }
    // the last slice: park the own partial in the drained ring, wait for the others
    static_assert(C::STAGES * C::STAGE_BYTES >= (uint32_t)C::E * C::CONSUMER_THREADS * 8, "own partial fits");
    __syncthreads();   // every warp is done with the ring
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t a = smem_base + (uint32_t)(((q * C::CONSUMER_WARPS + warp) * 32 + lane) * 32);
        sts_v2(a, flat[4 * q], flat[4 * q + 1]);
        sts_v2(a + 16, flat[4 * q + 2], flat[4 * q + 3]);
    }
    if (threadIdx.x == 0)
        while (ld_acquire(ctr) < S - 1) __nanosleep(32);   // rarely taken: the siblings were dispatched first
    __syncthreads();   // thread 0's acquire orders the others' partials before every thread's loads
    sum_partials<C>(acc, sk.ws, S - 1, [&](int t) { return (int64_t)tile * S + t; }, warp, lane);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t a = smem_base + (uint32_t)(((q * C::CONSUMER_WARPS + warp) * 32 + lane) * 32);
        double v0, v1, v2, v3;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v0), "=d"(v1) : "r"(a));
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v2), "=d"(v3) : "r"(a + 16));
        flat[4 * q] += v0;
        flat[4 * q + 1] += v1;
        flat[4 * q + 2] += v2;
        flat[4 * q + 3] += v3;
    }
    if (threadIdx.x == 0) *ctr = 0;   // ready for the next launch on this stream
    return true;
}

// Cluster split-K (SPLIT == 2, row a5): the S = gridDim.y slices of a tile run as one thread-
// block cluster (1, S, 1).  After its k-range each CTA writes its raw partial into its own
// shared memory (the drained ring), the cluster synchronises, and CTA s reduces the 256-bit
// accumulator groups q = s, s + S, ... of every thread: it reads group q of the same thread
// from the S CTAs through distributed shared memory in slice order 0..S-1 -- the order, and so
// the bits, of the global-memory split-K with the same S -- and stores those C quads.  No
// global partials, no counters, no last-arriver: the reduction is spread evenly over the
// cluster's CTAs.  A second cluster barrier keeps every CTA's shared memory alive until the
// others have read it.
template <class C>
__device__ __forceinline__ void cluster_reduce_epilogue(double (&acc)[C::MB][C::NP][2][2], uint32_t part, int warp,
                                                        int lane, int row0, int col0, int M, int N, double alpha,
                                                        double beta, double *__restrict__ Cm, int64_t ldc, bool vec) {
    constexpr int Q = C::E / 4;
    static_assert(C::STAGES * C::STAGE_BYTES >= (uint32_t)C::E * C::CONSUMER_THREADS * 8, "partial fits the ring");
    const double *flat = &acc[0][0][0][0];
    // partial layout [q][warp][lane][4 doubles]: a warp's 32 lanes write 1 KB contiguously
    __syncthreads();   // every warp has finished reading the ring's last stage
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t a = part + (uint32_t)(((q * C::CONSUMER_WARPS + warp) * 32 + lane) * 32);
        sts_v2(a, flat[4 * q], flat[4 * q + 1]);
        sts_v2(a + 16, flat[4 * q + 2], flat[4 * q + 3]);
    }
    dsm_sync();
    const int S = (int)gridDim.y;   // cluster size
    const int me = (int)dsm_rank();
    for (int q = me; q < Q; q += S) {
        const uint32_t a = part + (uint32_t)(((q * C::CONSUMER_WARPS + warp) * 32 + lane) * 32);
        double x[4] = {0.0, 0.0, 0.0, 0.0};
        for (int s = 0; s < S; ++s) {   // slice order
            const uint32_t r = dsm_map(a, (uint32_t)s);
            double v0, v1, v2, v3;
            dsm_ld_v2(r, v0, v1);
            dsm_ld_v2(r + 16, v2, v3);
            x[0] += v0;
            x[1] += v1;
            x[2] += v2;
            x[3] += v3;
        }
        const int mb = q / C::NP, np = q - mb * C::NP;
        const double w[4] = {x[0], x[2], x[1], x[3]};   // (j,i) = (0,0), (1,0), (0,1), (1,1)
        epilogue_quad(w, row0 + mb * 8, col0 + np * 16, M, N, alpha, beta, Cm, ldc, vec);
    }
    dsm_sync();
}

// SPLIT = false instantiations carry no split-K code (the reduction's registers would
// otherwise raise the 256x64/64x32 kernel from 199 to 255 registers).
// XP = true: cross-stage fragment prefetch -- the first half of stage i+1 is loaded (after
// its full-barrier wait) before the last half of stage i is multiplied, so the DMMA pipe
// does not drain at stage boundaries.
// ROT > 1: the refill of k-step i is issued by lane 0 of warp i % ROT instead of always by
// warp 0, spreading the producer's per-k-step instructions over ROT warps (and so over the
// SM's sub-partitions); the ring protocol is unchanged.
template <class C, int SPLIT, bool XP, int ROT = 1>
__global__ void __launch_bounds__(C::CONSUMER_THREADS, C::MIN_BLOCKS)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                     int N, int K, double alpha, double beta, double *__restrict__ Cm, int64_t ldc, int vec,
                     int group_m, SplitArgs sk) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(base_ptr + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;
    DG_TRACE_AT(0);

    const int tiles_m = (M + C::BM - 1) / C::BM, tiles_n = (N + C::BN - 1) / C::BN;
    int tm, tn;
    tile_coords(blockIdx.x, tiles_m, tiles_n, group_m, tm, tn);
    const int m0 = tm * C::BM, n0 = tn * C::BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KT = (K + C::BK - 1) / C::BK;
    const int split = SPLIT ? (int)blockIdx.y : 0;
    const int nsplit = SPLIT == 2 ? (int)gridDim.y : (SPLIT ? sk.splits : 1);
    const int kt0 = mul_div(split, KT, nsplit);
    const int NK = mul_div(split + 1, KT, nsplit) - kt0;   // k-steps of this CTA
    const bool producer = (threadIdx.x == 0);
    const bool md = (vec & 2) != 0;   // stage A / B with the 3-D / 4-D tensor maps
    constexpr int R = ROT < C::CONSUMER_WARPS ? ROT : C::CONSUMER_WARPS;   // warps sharing the refills
    uint64_t pol = 0;

    if (producer) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CONSUMER_WARPS);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (R > 1 ? lane == 0 : producer) pol = l2_policy_evict_normal();
    griddep_wait();
    DG_TRACE_AT(1);
    griddep_launch();
    if (producer) {
        for (int s = 0; s < C::STAGES && s < NK; ++s) {
            tma_issue_stage<C>(base_ptr + s * C::STAGE_BYTES, &tmA, &tmB, &full[s], m0, n0, kt0 + s, pol, md);
#ifdef DG_TRACE
            if (s == 0) DG_TRACE_AT(5);   // the first stage's TMA issued
#endif
        }
    }
    __syncthreads();

    const int warp_m = warp / C::WARPS_N, warp_n = warp % C::WARPS_N;
    const FragOffsets<C> fo(warp_m, warp_n, lane);
    double acc[C::MB][C::NP][2][2];
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
        for (int np = 0; np < C::NP; ++np)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[mb][np][j][0] = acc[mb][np][j][1] = 0.0;

    if constexpr (!XP) {
        for (int i = 0; i < NK; ++i) {
            const int s = i % C::STAGES;
            const bool refill = R > 1 ? (lane == 0 && warp == i % R) : producer;
            if (refill && i > 0) {
                const int in = i - 1 + C::STAGES;   // refill the slot released at i-1
                if (in < NK) {
                    const int sp = (i - 1) % C::STAGES;
                    mbar_wait(&empty[sp], ((i - 1) / C::STAGES) & 1);
                    tma_issue_stage<C>(base_ptr + sp * C::STAGE_BYTES, &tmA, &tmB, &full[sp], m0, n0, kt0 + in,
                                       pol, md);
                }
            }
            if (R > 1) __syncwarp();   // the refilling lane rejoins before the warp-wide mma.sync
            mbar_wait(&full[s], (i / C::STAGES) & 1);
#ifdef DG_TRACE
            if (i == 0) DG_TRACE_AT(2);
#endif
            const uint32_t sA = base + s * C::STAGE_BYTES;
            mma_stage<C>(sA, sA + C::A_BYTES, fo, acc);
            release_slot(&empty[s], lane);
        }
    } else {
        constexpr int H = 2 * C::KG;   // halves per stage (even: half 0 of every stage uses f[0])
        Frag<C> f[2];
        if (NK > 0) {
            mbar_wait(&full[0], 0);
            load_half<C>(base, base + C::A_BYTES, 0, fo, f[0]);
        }
        for (int i = 0; i < NK; ++i) {
            const int s = i % C::STAGES;
            const bool refill = R > 1 ? (lane == 0 && warp == i % R) : producer;
            if (refill && i > 0) {
                const int in = i - 1 + C::STAGES;
                if (in < NK) {
                    const int sp = (i - 1) % C::STAGES;
                    mbar_wait(&empty[sp], ((i - 1) / C::STAGES) & 1);
                    tma_issue_stage<C>(base_ptr + sp * C::STAGE_BYTES, &tmA, &tmB, &full[sp], m0, n0, kt0 + in,
                                       pol, md);
                }
            }
            if (R > 1) __syncwarp();   // the refilling lane rejoins before the warp-wide mma.sync
            const uint32_t sA = base + s * C::STAGE_BYTES;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (h + 1 < H) {
                    load_half<C>(sA, sA + C::A_BYTES, h + 1, fo, f[(h + 1) & 1]);
                } else {
                    // every fragment of slot s has been requested: hand the slot back before
                    // the next stage's loads are issued, so the release fence waits only
                    // for this slot's last half (needed by the DMMAs below anyway)
                    release_slot(&empty[s], lane);
                    if (i + 1 < NK) {
                        const int s1 = (i + 1) % C::STAGES;
                        mbar_wait(&full[s1], ((i + 1) / C::STAGES) & 1);
                        const uint32_t sA1 = base + s1 * C::STAGE_BYTES;
                        load_half<C>(sA1, sA1 + C::A_BYTES, 0, fo, f[0]);
                    }
                }
                mma_half<C>(f[h & 1], acc);
            }
        }
    }
    DG_TRACE_AT(3);
#ifdef DG_TRACE
    DG_TRACE_SLOT(7, (unsigned long long)dg_smid());
#endif
    if constexpr (SPLIT == 2) {
        if (gridDim.y > 1) {
            cluster_reduce_epilogue<C>(acc, base, warp, lane, m0 + warp_m * C::WM + (lane >> 2),
                                       n0 + warp_n * C::WN + 4 * (lane & 3), M, N, alpha, beta, Cm, ldc, (vec & 1) != 0);
            DG_TRACE_AT(6);
            return;
        }
    } else if constexpr (SPLIT == 1) {
        if (!split_reduce<C>(acc, sk, blockIdx.x, split, warp, lane, base)) {
            DG_TRACE_AT(6);
            return;
        }
    }
    DG_TRACE_AT(4);
    epilogue<C>(acc, m0 + warp_m * C::WM, n0 + warp_n * C::WN, lane, M, N, alpha, beta, Cm, ldc, (vec & 1) != 0);
    DG_TRACE_AT(6);
#ifdef DG_TRACE
    DG_TRACE_SLOT(7, (unsigned long long)dg_smid() | (1ull << 32));
#endif
}

// ------------------------------------------------------------------------------
// Stream-K kernel (row a5): a persistent grid of G CTAs (SMs x resident CTAs per SM)
// shares the U = tiles x KT k-steps evenly: CTA g runs global k-steps [g*U/G, (g+1)*U/G),
// crossing tile boundaries, so no SM idles in a partial last wave.  A tile covered by
// one CTA gets the plain epilogue; a tile cut by CTA boundaries is finished by
// partial_reduce (deterministic segment order).  The TMA producer streams k-steps in
// global order, so the smem ring stays full across tile boundaries.
__device__ __forceinline__ int64_t sk_bound(int64_t g, int64_t U, int64_t G) { return g * U / G; }
// number of g in [0, G] with floor(g*U/G) <= x
__device__ __forceinline__ int64_t sk_count_le(int64_t x, int64_t U, int64_t G) {
    const int64_t c = ((x + 1) * G + U - 1) / U;   // ceil((x+1) G / U)
    return c > G + 1 ? G + 1 : c;
}

template <class C>
__device__ __forceinline__ bool streamk_reduce(double (&acc)[C::MB][C::NP][2][2], double *ws, int *counters,
                                               int tile, int my_slot, int t0, int before, int nseg, int U, int G,
                                               int warp, int lane) {
    constexpr int Q = C::E / 4;
    constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;
    double *mine = partial_slot<C>(ws, my_slot, warp, lane);
    double *flat = &acc[0][0][0][0];
#pragma unroll
    for (int q = 0; q < Q; ++q) stg_v4(mine + q * QSTRIDE, flat[4 * q], flat[4 * q + 1], flat[4 * q + 2], flat[4 * q + 3]);
    __threadfence();
    __syncthreads();
    __shared__ int s_last_sk;
    if (threadIdx.x == 0) s_last_sk = (atomicAdd(&counters[tile], 1) == nseg - 1);
    __syncthreads();
    if (!s_last_sk) return false;
    __threadfence();
    // segment order = k order: segment j of the tile comes from CTA before - 1 + j
    sum_partials<C, 1>(acc, ws, nseg, [&](int j) {
        const int gj = before - 1 + j;
        return (int64_t)(2 * gj + (sk_bound(gj, U, G) >= t0 ? 0 : 1));
    }, warp, lane);
    if (threadIdx.x == 0) counters[tile] = 0;
    return true;
}

template <class C>
__global__ void __launch_bounds__(C::CONSUMER_THREADS, C::MIN_BLOCKS)
    dgemm_streamk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int N, int K, double alpha, double beta, double *__restrict__ Cm, int64_t ldc, int vec,
                         int group_m, double *ws, int *counters) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(base_ptr + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;
    DG_TRACE_AT(0);

    const int tiles_m = (M + C::BM - 1) / C::BM, tiles_n = (N + C::BN - 1) / C::BN;
    // 32-bit k-step bookkeeping (the host guarantees U = tiles * KT < 2^31) keeps the
    // 64x32-warp-tile instance free of register spills
    const int KT = (K + C::BK - 1) / C::BK;
    const int U = tiles_m * tiles_n * KT, G = gridDim.x, g = blockIdx.x;
    const int u0 = (int)sk_bound(g, U, G), u1 = (int)sk_bound(g + 1, U, G);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = (threadIdx.x == 0);
    // stateless refills rotated over R warps (as in dgemm_tma_kernel): local k-step l is
    // global unit u0 + l
    constexpr int R = 4 < C::CONSUMER_WARPS ? 4 : C::CONSUMER_WARPS;
    // the L2 policy is created once per refilling lane, not per refill (createpolicy sits on the
    // refilling warp's path, ahead of its DMMAs)
    const uint64_t pol = (lane == 0 && warp < R) ? l2_policy_evict_normal() : 0;
    auto issue_at = [&](int slot, int l) {
        const int u = u0 + l;
        const int t = u / KT;
        int tm, tn;
        tile_coords(t, tiles_m, tiles_n, group_m, tm, tn);
        tma_issue_stage<C>(base_ptr + slot * C::STAGE_BYTES, &tmA, &tmB, &full[slot], tm * C::BM, tn * C::BN,
                           u - t * KT, pol, (vec & 2) != 0);
    };
    const int nloc = u1 - u0;   // k-steps of this CTA

    if (producer) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CONSUMER_WARPS);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    DG_TRACE_AT(1);
    griddep_launch();
    if (producer) {
        for (int s = 0; s < C::STAGES && s < nloc; ++s) issue_at(s, s);
    }
    __syncthreads();

    const int warp_m = warp / C::WARPS_N, warp_n = warp % C::WARPS_N;
    const FragOffsets<C> fo(warp_m, warp_n, lane);
    double acc[C::MB][C::NP][2][2];
    int li = 0;                 // local k-step index
    int stage = 0, phase = 0;   // ring position of li
    int tile = u0 / KT;
    int kb = u0 - tile * KT;
    while (li < nloc) {
        const int ke = (u1 - tile * KT) < KT ? (u1 - tile * KT) : KT;
#pragma unroll
        for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
            for (int np = 0; np < C::NP; ++np)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[mb][np][j][0] = acc[mb][np][j][1] = 0.0;
        for (int k = kb; k < ke; ++k, ++li) {
            if (lane == 0 && warp == li % R && li > 0 && li - 1 + C::STAGES < nloc) {
                // refill the slot released at li-1 (the one before `stage`)
                const int sp = stage == 0 ? C::STAGES - 1 : stage - 1;
                const int pp = stage == 0 ? phase ^ 1 : phase;
                mbar_wait(&empty[sp], (uint32_t)pp);
                issue_at(sp, li - 1 + C::STAGES);
            }
            __syncwarp();   // the refilling lane rejoins before the warp-wide mma.sync
            mbar_wait(&full[stage], (uint32_t)phase);
#ifdef DG_TRACE
            if (li == 0) DG_TRACE_AT(2);
#endif
            const uint32_t sA = base + stage * C::STAGE_BYTES;
            mma_stage<C>(sA, sA + C::A_BYTES, fo, acc);
            release_slot(&empty[stage], lane);
            if (++stage == C::STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        // segments of this tile: CTA boundaries strictly inside (tile*KT, (tile+1)*KT)
        const int t0 = tile * KT;
        const int before = (int)sk_count_le(t0, U, G);                 // boundaries <= t0
        const int nseg = (int)sk_count_le(t0 + KT - 1, U, G) - before + 1;
        int tm, tn;
        tile_coords(tile, tiles_m, tiles_n, group_m, tm, tn);
        bool do_epi = true;
#ifdef DG_TRACE
        if (t0 + kb == u0) DG_TRACE_AT(3);                      // first tile of this CTA
        if (li >= nloc) DG_TRACE_AT(5);                         // last tile
#endif
        if (nseg > 1) {
            // Partial of CTA g goes to workspace slot 2g (its first unit) or 2g+1 (its last
            // unit); segment j of the tile comes from CTA g_j = before - 1 + j.
            const int my_slot = 2 * g + ((t0 + kb) == u0 ? 0 : 1);
            do_epi = streamk_reduce<C>(acc, ws, counters, tile, my_slot, t0, before, nseg, U, G, warp, lane);
        }
        if (do_epi)
            epilogue<C>(acc, tm * C::BM + warp_m * C::WM, tn * C::BN + warp_n * C::WN, lane, M, N, alpha, beta, Cm,
                        ldc, (vec & 1) != 0);
#ifdef DG_TRACE
        if (t0 + kb == u0) DG_TRACE_AT(4);
#endif
        ++tile;
        kb = 0;
    }
    DG_TRACE_AT(6);
#ifdef DG_TRACE
    DG_TRACE_SLOT(7, (unsigned long long)dg_smid() | ((unsigned long long)(tile - u0 / KT) << 32));
#endif
}

// ------------------------------------------------------------------------------
// Hybrid schedule (row a5, large shapes).  The T tiles split into W*G data-parallel tiles
// (W = floor(T/G) full waves of G = SMs x resident CTAs; run by the plain XP kernel, one
// tile per CTA) and a tail of T - W*G < G tiles, which alone would leave most SMs idle in
// a partial last wave.  The tail's Ut = tail*KT k-steps are shared stream-K style by gsk
// CTAs of dgemm_sktail_kernel (gsk >= tail, so a CTA's range spans at most two tiles).  A
// tail segment that is a whole tile gets the plain epilogue; any other stores its raw
// partial to workspace slot 2g+j (j = segment 0/1 of CTA g), and
// dgemm_hybrid_fixup_kernel sums each cut tile's partials in k order and runs the epilogue.
// (A persistent kernel that also ran the full waves was measured 1-3 % slower: CTAs that
// pick up tiles at different times fall out of k-lockstep, and the L2 working set of a
// wave -- shared A/B k-slices -- grows; DRAM reads rose from 6.4 to 7.5 GB at 8192^3.)
struct HybArgs {
    int tile0;      // first tail tile (= W*G)
    int gsk;        // CTAs sharing the tail
    double *ws;     // [2*gsk][E/4][warps][32][4] partials
};

template <class C>
__global__ void __launch_bounds__(C::CONSUMER_THREADS, C::MIN_BLOCKS)
    dgemm_sktail_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                        int N, int K, double alpha, double beta, double *__restrict__ Cm, int64_t ldc, int vec,
                        int group_m, HybArgs hy) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(base_ptr + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;

    const int tiles_m = (M + C::BM - 1) / C::BM, tiles_n = (N + C::BN - 1) / C::BN;
    const int KT = (K + C::BK - 1) / C::BK;
    const int g = blockIdx.x;
    // this CTA's range [u0, u1) of tail k-steps (host: tiles * KT < 2^31)
    const int64_t Ut = (int64_t)(tiles_m * tiles_n - hy.tile0) * KT;
    const int u0 = (int)((int64_t)g * Ut / hy.gsk), u1 = (int)((int64_t)(g + 1) * Ut / hy.gsk);
    if (u1 <= u0) return;
    const int ta = u0 / KT;                       // first (tail-local) tile
    const int nseg = (u1 - 1) / KT - ta + 1;      // 1 or 2
    const int total = u1 - u0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = (threadIdx.x == 0);
    // refills rotate over R warps as in dgemm_tma_kernel; a refill is stateless: local
    // k-step l of this CTA is tail unit u0 + l, in tile ta or ta + 1 (a range spans <= 2)
    constexpr int R = 4 < C::CONSUMER_WARPS ? 4 : C::CONSUMER_WARPS;
    const uint64_t pol = (lane == 0 && warp < R) ? l2_policy_evict_normal() : 0;   // once per refilling lane
    auto issue_at = [&](int slot, int l) {
        const int u = u0 + l;
        const int t = u >= (ta + 1) * KT ? ta + 1 : ta;
        int tm, tn;
        tile_coords(hy.tile0 + t, tiles_m, tiles_n, group_m, tm, tn);
        tma_issue_stage<C>(base_ptr + slot * C::STAGE_BYTES, &tmA, &tmB, &full[slot], tm * C::BM, tn * C::BN,
                           u - t * KT, pol, (vec & 2) != 0);
    };

    if (producer) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CONSUMER_WARPS);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    griddep_wait();
    griddep_launch();
    if (producer) {
        for (int s = 0; s < C::STAGES && s < total; ++s) issue_at(s, s);
    }
    __syncthreads();

    const int warp_m = warp / C::WARPS_N, warp_n = warp % C::WARPS_N;
    const FragOffsets<C> fo(warp_m, warp_n, lane);
    constexpr int H = 2 * C::KG;
    constexpr bool kXP = C::E >= 64;   // as in dgemm_tma_kernel: XP pays only for E = 64
    double acc[C::MB][C::NP][2][2];
    int it = 0;
    int stage = 0, phase = 0;
    for (int j = 0; j < nseg; ++j) {
        const int t = ta + j;
        const int kb = j == 0 ? u0 - t * KT : 0;
        const int ke = (u1 - t * KT) < KT ? (u1 - t * KT) : KT;
        const int NK = ke - kb;
#pragma unroll
        for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
            for (int np = 0; np < C::NP; ++np)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) acc[mb][np][jj][0] = acc[mb][np][jj][1] = 0.0;
        Frag<C> f[2];
        if constexpr (kXP) {
            mbar_wait(&full[stage], (uint32_t)phase);
            load_half<C>(base + stage * C::STAGE_BYTES, base + stage * C::STAGE_BYTES + C::A_BYTES, 0, fo, f[0]);
        }
        for (int i = 0; i < NK; ++i, ++it) {
            if (lane == 0 && warp == it % R && it > 0 && it - 1 + C::STAGES < total) {
                const int sp = stage == 0 ? C::STAGES - 1 : stage - 1;   // slot released at it-1
                const int pp = stage == 0 ? phase ^ 1 : phase;
                mbar_wait(&empty[sp], (uint32_t)pp);
                issue_at(sp, it - 1 + C::STAGES);
            }
            __syncwarp();   // the refilling lane rejoins before the warp-wide mma.sync
            const uint32_t sA = base + stage * C::STAGE_BYTES;
            const int s1 = stage + 1 == C::STAGES ? 0 : stage + 1;
            const int p1 = stage + 1 == C::STAGES ? phase ^ 1 : phase;
            if constexpr (kXP) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    if (h + 1 < H) {
                        load_half<C>(sA, sA + C::A_BYTES, h + 1, fo, f[(h + 1) & 1]);
                    } else {
                        release_slot(&empty[stage], lane);   // as in dgemm_tma_kernel (XP)
                        if (i + 1 < NK) {   // cross-stage prefetch inside the segment
                            mbar_wait(&full[s1], (uint32_t)p1);
                            const uint32_t sA1 = base + s1 * C::STAGE_BYTES;
                            load_half<C>(sA1, sA1 + C::A_BYTES, 0, fo, f[0]);
                        }
                    }
                    mma_half<C>(f[h & 1], acc);
                }
            } else {
                mbar_wait(&full[stage], (uint32_t)phase);
                mma_stage<C>(sA, sA + C::A_BYTES, fo, acc);
                release_slot(&empty[stage], lane);
            }
            stage = s1;
            phase = p1;
        }
        if (kb == 0 && ke == KT) {   // the whole tile: plain epilogue
            int tm, tn;
            tile_coords(hy.tile0 + t, tiles_m, tiles_n, group_m, tm, tn);
            epilogue<C>(acc, tm * C::BM + warp_m * C::WM, tn * C::BN + warp_n * C::WN, lane, M, N, alpha, beta, Cm,
                        ldc, (vec & 1) != 0);
        } else {
            constexpr int Q = C::E / 4;
            constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;
            double *mine = partial_slot<C>(hy.ws, 2 * g + j, warp, lane);
            const double *flat = &acc[0][0][0][0];
#pragma unroll
            for (int q = 0; q < Q; ++q)
                stg_v4(mine + q * QSTRIDE, flat[4 * q], flat[4 * q + 1], flat[4 * q + 2], flat[4 * q + 3]);
        }
    }
}

constexpr int kFixQ = 4;   // quads per fix-up CTA (grid.y = MB*NP / FixQ<C>), fewer for E = 8 tiles
template <class C>
constexpr int FixQ = (C::MB * C::NP) < kFixQ ? (C::MB * C::NP) : kFixQ;

// Tail fix-up: one CTA per (tail tile, FixQ<C> quads); a tile cut between CTAs gets the sum of its
// partials in k order (CTA jlo's segment first), then the plain epilogue.
template <class C>
__global__ void __launch_bounds__(C::CONSUMER_THREADS, 1)
    dgemm_hybrid_fixup_kernel(int M, int N, int K, double alpha, double beta, double *__restrict__ Cm, int64_t ldc,
                              int vec, int group_m, int tdp, int gsk, const double *__restrict__ ws) {
    griddep_wait();
    griddep_launch();
    const int tiles_m = (M + C::BM - 1) / C::BM, tiles_n = (N + C::BN - 1) / C::BN;
    const int KT = (K + C::BK - 1) / C::BK;
    const int64_t Ut = (int64_t)(tiles_m * tiles_n - tdp) * KT;
    const int b = blockIdx.x;
    const int64_t t0 = (int64_t)b * KT;
    const int jlo = (int)sk_count_le(t0, Ut, gsk) - 1;             // CTA holding k-step t0
    const int jhi = (int)sk_count_le(t0 + KT - 1, Ut, gsk) - 1;    // CTA holding the last k-step
    if (jlo == jhi) return;   // one CTA covered the whole tile: epilogue already done
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warp_m = warp / C::WARPS_N, warp_n = warp % C::WARPS_N;
    constexpr int64_t QSTRIDE = (int64_t)C::CONSUMER_WARPS * 32 * 4;
    int tm, tn;
    tile_coords(tdp + b, tiles_m, tiles_n, group_m, tm, tn);
    const int row0 = tm * C::BM + warp_m * C::WM + (lane >> 2);
    const int col0 = tn * C::BN + warp_n * C::WN + 4 * (lane & 3);
    // quad q = mb * NP + np holds flat accumulators 4q..4q+3 = acc[mb][np][j][i] (j major).
    // blockIdx.y selects FixQ<C> quads; their FixQ<C> loads per partial are issued together so
    // the sum costs ~nseg memory round trips, not nseg * quads.
    const int qb = blockIdx.y * FixQ<C>;
    double x[FixQ<C>][4];
#pragma unroll
    for (int u = 0; u < FixQ<C>; ++u) x[u][0] = x[u][1] = x[u][2] = x[u][3] = 0.0;
    for (int j = jlo; j <= jhi; ++j) {
        const int slot = 2 * j + (sk_bound(j, Ut, gsk) >= t0 ? 0 : 1);
        const double *src = partial_slot<C>(const_cast<double *>(ws), slot, warp, lane) + qb * QSTRIDE;
        double v[FixQ<C>][4];
#pragma unroll
        for (int u = 0; u < FixQ<C>; ++u)
            asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                         : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                         : "l"(src + u * QSTRIDE));
#pragma unroll
        for (int u = 0; u < FixQ<C>; ++u)
#pragma unroll
            for (int e = 0; e < 4; ++e) x[u][e] += v[u][e];
    }
#pragma unroll
    for (int u = 0; u < FixQ<C>; ++u) {
        const int q = qb + u;
        const int mb = q / C::NP, np = q - mb * C::NP;
        const double w[4] = {x[u][0], x[u][2], x[u][1], x[u][3]};   // (j,i) = (0,0), (1,0), (0,1), (1,1)
        epilogue_quad(w, row0 + mb * 8, col0 + np * 16, M, N, alpha, beta, Cm, ldc, (vec & 1) != 0);
    }
}

// ------------------------------------------------------------------------------
// Generic kernel: any 8-byte-aligned pointers and leading dimensions.  All warps
// stage tiles with 8-byte cp.async (zero-filled outside the matrix) into the same
// swizzled layout, STAGES-deep ring with cp.async groups.
template <class C>
__device__ __forceinline__ void generic_load_stage(uint32_t sA, uint32_t sB, const double *__restrict__ A,
                                                   int64_t lda, const double *__restrict__ B, int64_t ldb,
                                                   int M, int N, int K, int m0, int n0, int k0) {
    const int tid = threadIdx.x;
    for (int idx = tid; idx < C::BM * C::BK; idx += C::CONSUMER_THREADS) {
        const int r = idx / C::BK, k = idx % C::BK;
        const int gm = m0 + r, gk = k0 + k;
        const bool ok = gm < M && gk < K;
        const double *src = ok ? A + (int64_t)gm * lda + gk : A;
        const uint32_t dst = sA + (k >> 4) * C::A_SUB + r * 128 + ((((k & 15) >> 1) ^ (r & 7)) << 4) + (k & 1) * 8;
        cp_async_8(dst, src, ok);
    }
    for (int idx = tid; idx < C::BK * C::BN; idx += C::CONSUMER_THREADS) {
        const int k = idx / C::BN, n = idx % C::BN;
        const int gk = k0 + k, gn = n0 + n;
        const bool ok = gk < K && gn < N;
        const double *src = ok ? B + (int64_t)gk * ldb + gn : B;
        const int kk = k & 15, nn = n & 15;
        const uint32_t dst = sB + (k >> 4) * C::B_KG + (n >> 4) * C::B_BOX + kk * 128 +
                             ((((nn >> 1) ^ (kk & 7))) << 4) + (nn & 1) * 8;
        cp_async_8(dst, src, ok);
    }
}

template <class C>
__global__ void __launch_bounds__(C::CONSUMER_THREADS, 1)
    dgemm_generic_kernel(const double *__restrict__ A, int64_t lda, const double *__restrict__ B, int64_t ldb,
                         int M, int N, int K, double alpha, double beta, double *__restrict__ Cm, int64_t ldc,
                         int vec, int group_m) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;

    const int tiles_m = (M + C::BM - 1) / C::BM, tiles_n = (N + C::BN - 1) / C::BN;
    int tm, tn;
    tile_coords(blockIdx.x, tiles_m, tiles_n, group_m, tm, tn);
    const int m0 = tm * C::BM, n0 = tn * C::BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KT = (K + C::BK - 1) / C::BK;
    griddep_wait();
    griddep_launch();

#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
        if (s < KT) {
            const uint32_t sA = base + s * C::STAGE_BYTES;
            generic_load_stage<C>(sA, sA + C::A_BYTES, A, lda, B, ldb, M, N, K, m0, n0, s * C::BK);
        }
        cp_async_commit();
    }

    const int warp_m = warp / C::WARPS_N, warp_n = warp % C::WARPS_N;
    const FragOffsets<C> fo(warp_m, warp_n, lane);
    double acc[C::MB][C::NP][2][2];
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
        for (int np = 0; np < C::NP; ++np)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[mb][np][j][0] = acc[mb][np][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<C::STAGES - 2>();
        __syncthreads();
        const int kn = kt + C::STAGES - 1;
        if (kn < KT) {
            const uint32_t sA = base + (kn % C::STAGES) * C::STAGE_BYTES;
            generic_load_stage<C>(sA, sA + C::A_BYTES, A, lda, B, ldb, M, N, K, m0, n0, kn * C::BK);
        }
        cp_async_commit();
        const uint32_t sA = base + (kt % C::STAGES) * C::STAGE_BYTES;
        mma_stage<C>(sA, sA + C::A_BYTES, fo, acc);
    }
    cp_async_wait<0>();
    epilogue<C>(acc, m0 + warp_m * C::WM, n0 + warp_n * C::WN, lane, M, N, alpha, beta, Cm, ldc, (vec & 1) != 0);
}

}  // namespace dg
