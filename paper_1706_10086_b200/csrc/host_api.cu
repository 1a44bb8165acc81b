// host_api.cu -- gemm_f64_host: the end-to-end call on HOST buffers.
//
// The paper times "the run of the algorithm without copy operations to device
// memory"; this entry point is the opposite view, the whole job a user
// with host data sees.  Copies are overlapped with the DMMA kernel by row
// panels: B goes first (every panel needs all of it), then for each panel p of
// rows the A rows (and C rows when beta != 0) travel host->device on the h2d
// stream, the compute stream multiplies panel p once its rows landed, and the
// d2h stream returns panel p while panel p+1 computes.  Per-entry arithmetic
// is that of gemm_f64 on the whole matrix (row panels do not change it).
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
    if ((rc = ensure(&P.dA, &P.nA, need_ab ? (size_t)M * K : 0))) return rc;
    if ((rc = ensure(&P.dB, &P.nB, need_ab ? (size_t)K * N : 0))) return rc;
    if ((rc = ensure(&P.dC, &P.nC, (size_t)M * N))) return rc;

    // Panel size: at least two waves of 128x128 tiles per panel, at most 8 panels.
    const int64_t tiles_n = (N + 127) / 128;
    int64_t min_rows = ((2 * 148 + tiles_n - 1) / tiles_n) * 128;
    int64_t npan = std::max<int64_t>(1, std::min<int64_t>(8, M / std::max<int64_t>(min_rows, 1)));
    int64_t rows_per = ((M + npan - 1) / npan + 127) / 128 * 128;
    npan = (M + rows_per - 1) / rows_per;
    if ((rc = ensure_events(P.ev_in, (size_t)npan))) return rc;
    if ((rc = ensure_events(P.ev_out, (size_t)npan))) return rc;

    if (need_ab) {
        if ((rc = cuda_check(cudaMemcpy2DAsync(P.dB, N * 8, B, ldb * 8, N * 8, K, cudaMemcpyHostToDevice, P.h2d),
                             "H2D B")))
            return rc;
    }
    for (int64_t p = 0; p < npan; ++p) {
        const int64_t r0 = p * rows_per, r1 = std::min(M, r0 + rows_per), nr = r1 - r0;
        if (need_ab &&
            (rc = cuda_check(cudaMemcpy2DAsync(P.dA + r0 * K, K * 8, A + r0 * lda, lda * 8, K * 8, nr,
                                               cudaMemcpyHostToDevice, P.h2d),
                             "H2D A panel")))
            return rc;
        if (need_c_in &&
            (rc = cuda_check(cudaMemcpy2DAsync(P.dC + r0 * N, N * 8, C + r0 * ldc, ldc * 8, N * 8, nr,
                                               cudaMemcpyHostToDevice, P.h2d),
                             "H2D C panel")))
            return rc;
        if ((rc = cuda_check(cudaEventRecord(P.ev_in[p], P.h2d), "event"))) return rc;
        if ((rc = cuda_check(cudaStreamWaitEvent(P.comp, P.ev_in[p], 0), "wait"))) return rc;
        rc = gemm_impl(nr, N, need_ab ? K : 0, need_ab ? alpha : 0.0, P.dA + r0 * K, std::max<int64_t>(1, K), P.dB,
                       N, beta, P.dC + r0 * N, N, -1, P.comp);
        if (rc) return rc;
        if ((rc = cuda_check(cudaEventRecord(P.ev_out[p], P.comp), "event"))) return rc;
        if ((rc = cuda_check(cudaStreamWaitEvent(P.d2h, P.ev_out[p], 0), "wait"))) return rc;
        if ((rc = cuda_check(cudaMemcpy2DAsync(C + r0 * ldc, ldc * 8, P.dC + r0 * N, N * 8, N * 8, nr,
                                               cudaMemcpyDeviceToHost, P.d2h),
                             "D2H C panel")))
            return rc;
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
