// sharded.cu -- row-block-sharded multi-GPU GEMM; one process per GPU.
//
// C = alpha*A*B + beta*C partitioned by rows of C: rank r owns A[r0:r1, :] and
// C[r0:r1, :], r0 = floor(r*M/P).  Every rank needs all of B, which is the one
// exchange step: an NCCL broadcast over NVLink 5 / NVSwitch.  The paper itself has
// no communication (Alpaka "does not abstract the inter-node communication").
//
// bcast_chunks == 1: broadcast B in place, then the local GEMM (serial).
// bcast_chunks  > 1: B is split into column panels; the root packs panel j into a
//   library workspace (copy engine), panel j is broadcast on the comm stream while
//   panel j-1 is multiplied on the caller's stream (C[:, panel] with ldb = panel
//   width).  Per-entry arithmetic is unchanged -> bitwise equal to chunks == 1.
//   Non-root B buffers receive the unpacked panels at the end.
// Both paths launch without split-K (force_splits = 1) so the per-entry k-order chain
// is the same for any panel width and any number of ranks.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "../../include/gemm_f64.h"
#include "internal.h"

namespace dg {

struct Comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1, dev = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> ev;
    double *ws = nullptr;
    size_t ws_cap = 0;
    cudaEvent_t ws_free = nullptr;   // recorded after the last reader of ws (previous call)
    bool ws_free_valid = false;
};

static int nccl_check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return GEMM_OK;
    return set_error(GEMM_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

static int ensure_events(Comm *c, size_t n) {
    while (c->ev.size() < n) {
        cudaEvent_t e;
        int rc = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        if (rc) return rc;
        c->ev.push_back(e);
    }
    return GEMM_OK;
}

}  // namespace dg

using namespace dg;

extern "C" {

int gemm_comm_unique_id(unsigned char id_out[128]) {
    clear_error();
    if (!id_out) return set_error(GEMM_ERR_ARG, "id_out is NULL");
    ncclUniqueId id;
    int rc = nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    if (rc) return rc;
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
    for (int i = 0; i < 128; ++i) id_out[i] = (unsigned char)id.internal[i];
    return GEMM_OK;
}

int gemm_comm_init(void **comm_out, int nranks, const unsigned char id[128], int rank) {
    clear_error();
    if (!comm_out) return set_error(GEMM_ERR_ARG, "comm_out is NULL");
    if (!id) return set_error(GEMM_ERR_ARG, "id is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(GEMM_ERR_ARG, "rank=%d / nranks=%d invalid", rank, nranks);
    Comm *c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    int rc = cuda_check(cudaGetDevice(&c->dev), "cudaGetDevice");
    if (!rc) rc = cuda_check(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking), "stream");
    if (!rc) {
        ncclUniqueId uid;
        for (int i = 0; i < 128; ++i) uid.internal[i] = (char)id[i];
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.blocking = 1;
        // GEMM_NCCL_MAX_CTAS caps the CTAs NCCL's kernels take (the SMs a concurrent panel
        // broadcast steals from the GEMM with bcast_chunks > 1); unset = NCCL's default
        if (const char *e = std::getenv("GEMM_NCCL_MAX_CTAS")) {
            const int v = std::atoi(e);
            if (v > 0) cfg.maxCTAs = v;
        }
        rc = nccl_check(ncclCommInitRankConfig(&c->nccl, nranks, uid, rank, &cfg), "ncclCommInitRankConfig");
    }
    if (rc) {
        if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
        delete c;
        return rc;
    }
    *comm_out = c;
    return GEMM_OK;
}

int gemm_comm_destroy(void *comm) {
    clear_error();
    if (!comm) return GEMM_OK;
    Comm *c = static_cast<Comm *>(comm);
    int rc = GEMM_OK;
    if (c->nccl) rc = nccl_check(ncclCommDestroy(c->nccl), "ncclCommDestroy");
    for (auto e : c->ev) cudaEventDestroy(e);
    if (c->ws_free) cudaEventDestroy(c->ws_free);
    if (c->ws) cudaFree(c->ws);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    delete c;
    return rc;
}

int gemm_comm_info(void *comm, int *nranks, int *rank) {
    clear_error();
    if (!comm || !nranks || !rank) return set_error(GEMM_ERR_ARG, "comm / nranks / rank is NULL");
    Comm *c = static_cast<Comm *>(comm);
    int rc = nccl_check(ncclCommCount(c->nccl, nranks), "ncclCommCount");
    if (!rc) rc = nccl_check(ncclCommUserRank(c->nccl, rank), "ncclCommUserRank");
    return rc;
}

int gemm_bcast_f64(double *buf, int64_t count, int root, void *comm, void *stream) {
    clear_error();
    if (!comm) return set_error(GEMM_ERR_ARG, "comm is NULL");
    Comm *c = static_cast<Comm *>(comm);
    if (count < 0) return set_error(GEMM_ERR_ARG, "count=%lld < 0", (long long)count);
    if (root < 0 || root >= c->nranks) return set_error(GEMM_ERR_ARG, "root=%d out of range", root);
    if (count == 0) return GEMM_OK;
    if (!buf) return set_error(GEMM_ERR_ARG, "buf is NULL");
    return nccl_check(ncclBroadcast(buf, buf, (size_t)count, ncclDouble, root, c->nccl, (cudaStream_t)stream),
                      "ncclBroadcast");
}

int gemm_f64_sharded(int64_t M_local, int64_t N, int64_t K, double alpha, const double *A_local, int64_t lda,
                     double *B, int64_t ldb, double beta, double *C_local, int64_t ldc, void *comm, int root,
                     int bcast_chunks, void *stream_) {
    clear_error();
    if (!comm) return set_error(GEMM_ERR_ARG, "comm is NULL");
    Comm *c = static_cast<Comm *>(comm);
    cudaStream_t st = (cudaStream_t)stream_;
    if (root < 0 || root >= c->nranks) return set_error(GEMM_ERR_ARG, "root=%d out of range [0,%d)", root, c->nranks);
    if (bcast_chunks < 1) return set_error(GEMM_ERR_ARG, "bcast_chunks=%d must be >= 1", bcast_chunks);
    if (N < 0 || K < 0) return set_error(GEMM_ERR_ARG, "N=%lld K=%lld must be >= 0", (long long)N, (long long)K);
    if (K > 0 && N > 0 && ldb != N)
        return set_error(GEMM_ERR_UNSUPPORTED, "sharded GEMM needs contiguous B (ldb=%lld != N=%lld)",
                         (long long)ldb, (long long)N);
    int rc = validate(M_local, N, K, alpha, A_local, lda, B, std::max<int64_t>(ldb, 1), C_local, ldc);
    if (rc) return rc;
    const bool need_b = (alpha != 0.0 && K > 0 && N > 0);
    if (!need_b) return gemm_impl(M_local, N, K, alpha, A_local, lda, B, ldb, beta, C_local, ldc, -1, st);
    if (!B) return set_error(GEMM_ERR_ARG, "B is NULL");

    int nch = (int)std::min<int64_t>(bcast_chunks, std::max<int64_t>(1, N / 64));
    if (nch == 1) {
        rc = nccl_check(ncclBroadcast(B, B, (size_t)(K * N), ncclDouble, root, c->nccl, st), "ncclBroadcast(B)");
        if (rc) return rc;
        return gemm_impl(M_local, N, K, alpha, A_local, lda, B, ldb, beta, C_local, ldc, -1, st, 1);
    }

    // ---- column-panel pipeline ----
    if (!c->ws_free &&
        (rc = cuda_check(cudaEventCreateWithFlags(&c->ws_free, cudaEventDisableTiming), "cudaEventCreate")))
        return rc;
    if (c->ws_cap < (size_t)(K * N)) {
        // the previous call's GEMMs (on whatever stream it used) may still read the old panels
        if (c->ws_free_valid && (rc = cuda_check(cudaEventSynchronize(c->ws_free), "cudaEventSynchronize")))
            return rc;
        if (c->ws) cudaFree(c->ws);
        c->ws = nullptr;
        c->ws_cap = 0;
        if (cudaMalloc(&c->ws, (size_t)(K * N) * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            return set_error(GEMM_ERR_ALLOC, "sharded workspace of %lld bytes", (long long)(K * N * 8));
        }
        c->ws_cap = (size_t)(K * N);
    }
    if ((rc = ensure_events(c, (size_t)nch + 2))) return rc;
    // panel widths: multiples of 16 columns except the last
    const int64_t w = ((N + nch - 1) / nch + 15) / 16 * 16;
    nch = (int)((N + w - 1) / w);
    const bool is_root = (c->rank == root);
    // comm stream starts after prior work on the caller's stream (B / C may be written there)
    // and after the previous call's last GEMM, which read the panels it is about to overwrite
    if ((rc = cuda_check(cudaEventRecord(c->ev[nch], st), "event"))) return rc;
    if ((rc = cuda_check(cudaStreamWaitEvent(c->comm_stream, c->ev[nch], 0), "wait"))) return rc;
    if (c->ws_free_valid && (rc = cuda_check(cudaStreamWaitEvent(c->comm_stream, c->ws_free, 0), "wait")))
        return rc;
    for (int j = 0; j < nch; ++j) {
        const int64_t n0 = j * w, nw = std::min(N, n0 + w) - n0;
        double *panel = c->ws + K * n0;   // packed K x nw
        if (is_root &&
            (rc = cuda_check(cudaMemcpy2DAsync(panel, nw * 8, B + n0, ldb * 8, nw * 8, K, cudaMemcpyDeviceToDevice,
                                               c->comm_stream),
                             "pack panel")))
            return rc;
        if ((rc = nccl_check(ncclBroadcast(panel, panel, (size_t)(K * nw), ncclDouble, root, c->nccl, c->comm_stream),
                             "ncclBroadcast(panel)")))
            return rc;
        if ((rc = cuda_check(cudaEventRecord(c->ev[j], c->comm_stream), "event"))) return rc;
        if ((rc = cuda_check(cudaStreamWaitEvent(st, c->ev[j], 0), "wait"))) return rc;
        rc = gemm_impl(M_local, nw, K, alpha, A_local, lda, panel, nw, beta, C_local + n0, ldc, -1, st, 1);
        if (rc) return rc;
    }
    if (!is_root) {   // leave the broadcast B in the caller's buffer, as the contract says
        for (int j = 0; j < nch; ++j) {
            const int64_t n0 = j * w, nw = std::min(N, n0 + w) - n0;
            if ((rc = cuda_check(cudaMemcpy2DAsync(B + n0, ldb * 8, c->ws + K * n0, nw * 8, nw * 8, K,
                                                   cudaMemcpyDeviceToDevice, c->comm_stream),
                                 "unpack panel")))
                return rc;
        }
    }
    if ((rc = cuda_check(cudaEventRecord(c->ev[nch + 1], c->comm_stream), "event"))) return rc;
    if ((rc = cuda_check(cudaStreamWaitEvent(st, c->ev[nch + 1], 0), "wait"))) return rc;
    // every reader of the panels (this call's GEMMs and the unpack) is ordered before this point
    if ((rc = cuda_check(cudaEventRecord(c->ws_free, st), "event"))) return rc;
    c->ws_free_valid = true;
    return GEMM_OK;
}

}  // extern "C"
