// ptx.cuh -- thin inline-PTX wrappers for sm_100a used by the DGEMM kernels.
//
// Nothing here is GEMM arithmetic except dmma_m8n8k4 (the FP64 tensor-pipe
// instruction, SASS DMMA.8x8x4).  Everything else is data movement and
// synchronisation: mbarriers, TMA (cp.async.bulk.tensor -> SASS UTMALDG),
// cp.async (LDGSTS) and 256-bit global vector access (LDG/STG.E.ENL2.256).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace dg {

// ---- optional per-CTA timeline (instrumented builds only: build.py --trace, -DDG_TRACE) ----
// Each CTA writes 8 u64 at trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8]: globaltimer (ns)
// at the points the kernels mark with DG_TRACE_AT(slot), and in slot 7 the SM id.  The
// pointer is per translation unit and set by launch_k before each launch.  Product builds
// compile all of this away.
#ifdef DG_TRACE
static __device__ unsigned long long *dg_trace_buf;
static void *dg_trace_last = reinterpret_cast<void *>(~uintptr_t(0));   // host copy of dg_trace_buf
__device__ __forceinline__ unsigned long long dg_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned dg_smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;\n" : "=r"(r));
    return r;
}
#define DG_TRACE_SLOT(slot, val)                                                                     \
    do {                                                                                             \
        if (threadIdx.x == 0 && dg_trace_buf)                                                        \
            dg_trace_buf[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (slot)] = (val);         \
    } while (0)
#define DG_TRACE_AT(slot) DG_TRACE_SLOT(slot, dg_gtimer())
#else
#define DG_TRACE_SLOT(slot, val) ((void)0)
#define DG_TRACE_AT(slot) ((void)0)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- FP64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col) --------------------
// Fragment ownership (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t,
//   a = A[g][t], b = B[t][g], {d0, d1} = D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ---- mbarrier ------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- thread-block clusters / distributed shared memory (cluster split-K) -------------------
__device__ __forceinline__ uint32_t dsm_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// every thread of every CTA of the cluster: release this CTA's prior shared-memory writes,
// acquire the other CTAs'
__device__ __forceinline__ void dsm_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// the address of the same shared-memory location in cluster CTA `rank`
__device__ __forceinline__ uint32_t dsm_map(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void dsm_ld_v2(uint32_t cluster_addr, double &x, double &y) {
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t addr, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

// ---- gpu-scope release / acquire on a global counter (ordered split-K) -----------------------
__device__ __forceinline__ void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ---- programmatic dependent launch (PDL) -------------------------------------------
// The host launches every GEMM kernel with programmatic stream serialization, so a kernel
// may become resident while the previous kernel in the stream is still draining.  Each
// kernel sets up its shared-memory state, then griddep_wait() blocks until the previous
// grid has completed and its memory is visible -- before the first global access -- and
// griddep_launch() lets the next kernel start its own setup early (it still waits in turn).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ---- TMA ------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2-D tiled load: coordinates are (innermost = column, row) in elements.
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// 3-D / 4-D tiled loads (one instruction for a whole stage of A, resp. B; see
// dgemm_kernels.cuh tma_issue_stage): coordinates innermost first.
__device__ __forceinline__ void tma_load_3d(void *smem_dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *smem_dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// ---- cp.async (LDGSTS), 8-byte granules with zero-fill ----------------------------
__device__ __forceinline__ void cp_async_8(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- 256-bit global vector access (sm_100) -----------------------------------------
__device__ __forceinline__ void ldg_v4(const double *p, double &a, double &b, double &c, double &d) {
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p));
}
__device__ __forceinline__ void stg_v4(double *p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}

}  // namespace dg
