// host_api.cu -- gemm_f64_host: the end-to-end call on HOST buffers.
//
// The paper times "the run of the algorithm without copy operations to device
// memory"; this entry point is the opposite view, the whole job a user
// with host data sees, with the copies overlapped with the DMMA kernel (three
// streams: h2d, compute, d2h; schedule below).  Per-entry arithmetic is that of
// gemm_f64 on the whole matrix: blocks of C only change which CTA computes an
// entry, and split-K is disabled here so every block uses the same k-order chain.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/gemm_f64.h"
#include "internal.h"

namespace dg {

struct HostPool {
    double *dA = nullptr, *dB = nullptr, *dC = nullptr;
    size_t nA = 0, nB = 0, nC = 0;   // capacities in doubles
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_out;
};

static std::mutex g_pool_mu;
static std::map<int, HostPool> g_pools;

static int ensure(double **p, size_t *cap, size_t need) {
    if (*cap >= need) return GEMM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (need == 0) return GEMM_OK;
    if (cudaMalloc(p, need * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GEMM_ERR_ALLOC, "cudaMalloc of %zu bytes failed", need * sizeof(double));
    }
    *cap = need;
    return GEMM_OK;
}

static int ensure_events(std::vector<cudaEvent_t> &v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t e;
        int rc = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        if (rc) return rc;
        v.push_back(e);
    }
    return GEMM_OK;
}

// Schedule (all copies from the caller's host buffers into packed device buffers):
//   h2d : A rows [0, R0), then B in column panels, then A row panels 1.. (and C0 rows
//         alongside the A rows when beta != 0)
//   comp: row panel 0 is multiplied column block by column block as the B panels land
//         (R0 is sized so that this work covers the whole B transfer:
//         R0 ~ 4 * compute_rate / h2d_bandwidth rows, independent of N and K), then
//         each later row panel as soon as its A rows land; the last row panel is again
//         computed in column blocks so that its device->host copy overlaps
//   d2h : every finished block / panel of C
// Exposed copy time is the first A rows + the first B panel and the last C block.
static int host_impl(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
                     int64_t ldb, double beta, double *C, int64_t ldc) {
    clear_error();
    int rc = validate(M, N, K, alpha, A, lda, B, ldb, C, ldc);
    if (rc) return rc;
    if (M == 0 || N == 0) return GEMM_OK;
    const bool need_ab = (alpha != 0.0 && K > 0);
    const bool need_c_in = (beta != 0.0);
    if (!need_ab && beta == 1.0) return GEMM_OK;

    int dev = 0;
    if ((rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice"))) return rc;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    HostPool &P = g_pools[dev];
    if (!P.h2d) {
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking), "stream"))) return rc;
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking), "stream"))) return rc;
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking), "stream"))) return rc;
    }
    // device copies are packed: ld = row length
    const int64_t Kp = std::max<int64_t>(1, K);
    if ((rc = ensure(&P.dA, &P.nA, need_ab ? (size_t)M * K : 0))) return rc;
    if ((rc = ensure(&P.dB, &P.nB, need_ab ? (size_t)K * N : 0))) return rc;
    if ((rc = ensure(&P.dC, &P.nC, (size_t)M * N))) return rc;

    // ---- geometry
    const double flops = 2.0 * (double)M * (double)N * (double)K;
    const bool tiny = !need_ab || flops < 2e10;      // < ~1 ms of GPU work: one shot
    int64_t R0 = M, Rp = M, cb = N;                  // first panel rows, later panel rows, column block
    if (!tiny) {
        // R0 ~ 4 * compute rate / H2D bandwidth rows keeps the GPU busy while B streams in;
        // 2304 = 9 rows of 256-row tiles: with 2048-column blocks (32 tiles of 64) a block is
        // 288 tiles = 1.95 waves of 148 SMs (2560 rows gave 320 tiles = 2.16 waves).
        R0 = std::min<int64_t>(M, 2304);
        Rp = 2048;
        cb = std::max<int64_t>(512, ((N + 7) / 8 + 63) / 64 * 64);   // <= 8 column blocks
    }
    const int64_t ncb = (N + cb - 1) / cb;
    const int64_t nrest = (M > R0) ? (M - R0 + Rp - 1) / Rp : 0;
    // events: one per column block of panel 0, one per later panel, one per column block
    // of the last panel (h2d_done / comp_done each use at most this many)
    const size_t nev = (size_t)(2 * ncb + nrest + 8);
    if ((rc = ensure_events(P.ev_in, nev))) return rc;
    if ((rc = ensure_events(P.ev_out, nev))) return rc;

    auto h2d_rows = [&](double *dst, int64_t dld, const double *src, int64_t sld, int64_t cols, int64_t rows,
                        const char *what) {
        return cuda_check(cudaMemcpy2DAsync(dst, dld * 8, src, sld * 8, cols * 8, rows, cudaMemcpyHostToDevice, P.h2d),
                          what);
    };
    auto d2h_block = [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc) {
        return cuda_check(cudaMemcpy2DAsync(C + r0 * ldc + c0, ldc * 8, P.dC + r0 * N + c0, N * 8, nc * 8, nr,
                                            cudaMemcpyDeviceToHost, P.d2h),
                          "D2H C block");
    };
    auto run = [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc) {
        return gemm_impl(nr, nc, need_ab ? K : 0, need_ab ? alpha : 0.0, P.dA + r0 * K, Kp, P.dB + c0, N, beta,
                         P.dC + r0 * N + c0, N, -1, P.comp, /*force_splits=*/1);
    };
    size_t ei = 0, eo = 0;
    auto h2d_done = [&]() -> int {   // compute stream waits for everything copied so far
        if (ei >= P.ev_in.size()) return set_error(GEMM_ERR_CUDA, "internal: h2d event pool exhausted");
        int r = cuda_check(cudaEventRecord(P.ev_in[ei], P.h2d), "event");
        if (!r) r = cuda_check(cudaStreamWaitEvent(P.comp, P.ev_in[ei], 0), "wait");
        ++ei;
        return r;
    };
    auto comp_done = [&]() -> int {  // d2h stream waits for everything computed so far
        if (eo >= P.ev_out.size()) return set_error(GEMM_ERR_CUDA, "internal: d2h event pool exhausted");
        int r = cuda_check(cudaEventRecord(P.ev_out[eo], P.comp), "event");
        if (!r) r = cuda_check(cudaStreamWaitEvent(P.d2h, P.ev_out[eo], 0), "wait");
        ++eo;
        return r;
    };

    // ---- row panel 0: A rows and C0 rows first, then B column blocks, each followed by its GEMM block
    if (need_ab && (rc = h2d_rows(P.dA, K, A, lda, K, R0, "H2D A panel"))) return rc;
    if (need_c_in && (rc = h2d_rows(P.dC, N, C, ldc, N, R0, "H2D C panel"))) return rc;
    for (int64_t j = 0; j < ncb; ++j) {
        const int64_t c0 = j * cb, nc = std::min(N, c0 + cb) - c0;
        if (need_ab && (rc = cuda_check(cudaMemcpy2DAsync(P.dB + c0, N * 8, B + c0, ldb * 8, nc * 8, K,
                                                          cudaMemcpyHostToDevice, P.h2d),
                                        "H2D B panel")))
            return rc;
        if ((rc = h2d_done())) return rc;
        if ((rc = run(0, R0, c0, nc))) return rc;
        if ((rc = comp_done())) return rc;
        if ((rc = d2h_block(0, R0, c0, nc))) return rc;
    }
    // ---- later row panels
    for (int64_t p = 0; p < nrest; ++p) {
        const int64_t r0 = R0 + p * Rp, nr = std::min(M, r0 + Rp) - r0;
        if (need_ab && (rc = h2d_rows(P.dA + r0 * K, K, A + r0 * lda, lda, K, nr, "H2D A panel"))) return rc;
        if (need_c_in && (rc = h2d_rows(P.dC + r0 * N, N, C + r0 * ldc, ldc, N, nr, "H2D C panel"))) return rc;
        if ((rc = h2d_done())) return rc;
        // the last panel in 2 column blocks: the final D2H overlaps the first one (narrower
        // blocks shorten the exposed copy but fall into partial waves, measured slower)
        const bool last = (p == nrest - 1);
        const int64_t lcb = last ? std::max<int64_t>(512, ((N + 1) / 2 + 63) / 64 * 64) : N;
        const int64_t nlcb = (N + lcb - 1) / lcb;
        for (int64_t j = 0; j < nlcb; ++j) {
            const int64_t c0 = j * lcb, nc = std::min(N, c0 + lcb) - c0;
            if ((rc = run(r0, nr, c0, nc))) return rc;
            if ((rc = comp_done())) return rc;
            if ((rc = d2h_block(r0, nr, c0, nc))) return rc;
        }
    }
    return cuda_check(cudaStreamSynchronize(P.d2h), "gemm_f64_host synchronize");
}

}  // namespace dg

using namespace dg;

extern "C" {

int gemm_f64_host(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
                  int64_t ldb, double beta, double *C, int64_t ldc) {
    return host_impl(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

int gemm_host_pool_release(void) {
    clear_error();
    int dev = 0;
    int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it == g_pools.end()) return GEMM_OK;
    HostPool &P = it->second;
    cudaDeviceSynchronize();
    cudaFree(P.dA);
    cudaFree(P.dB);
    cudaFree(P.dC);
    for (auto e : P.ev_in) cudaEventDestroy(e);
    for (auto e : P.ev_out) cudaEventDestroy(e);
    if (P.h2d) cudaStreamDestroy(P.h2d);
    if (P.comp) cudaStreamDestroy(P.comp);
    if (P.d2h) cudaStreamDestroy(P.d2h);
    g_pools.erase(it);
    return GEMM_OK;
}

}  // extern "C"
