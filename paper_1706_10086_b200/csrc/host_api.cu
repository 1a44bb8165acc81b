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
#include <string>
#include <tuple>
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
//   h2d : A rows [0, Ra), B column block 0, A rows [Ra, R0), B column blocks 1.., then the
//         A row panels (and C0 rows alongside the A rows when beta != 0)
//   comp: row panel 0 (R0 rows) is multiplied column block by column block as the B
//         blocks land -- block 0 first on rows [0, Ra) so the GPU starts after a short
//         copy; R0 is sized so a block's GEMM outlasts the next block's copy
//         (R0 >= 4 * compute_rate / h2d_bandwidth rows, independent of N and K); then the
//         later row panels, each as soon as its A rows land; the last panel is thin
//         (256 rows, 2 column blocks) so the final device->host copy is short
//   d2h : every finished block / panel of C
// Block widths and panel heights are chosen so that each GEMM's 256x64 tile count falls
// just below a multiple of the SM count (little partial-wave waste).  The geometry was
// chosen with a copy/compute simulation calibrated on measured PCIe and GEMM rates
// (DESIGN.md §e2e): 16384^3 264 -> 255 ms.  Round 2: the same simulation runs here per shape
// (plan_geometry) and replaces the rule's geometry when a coarse grid finds one > 1 % faster.
namespace {
constexpr double kRate = 36.6e12;   // FP64 DMMA GEMM rate (FLOP/s)
constexpr double kH2D = 55e9;       // pinned H2D bandwidth (B/s), PCIe 5 x16
constexpr int kTm = 256, kTn = 64;  // tile of the large-shape kernel

// tile count t = r * c falls in a wave as fully as possible: efficiency t / (S * ceil(t / S))
double wave_eff(int64_t t, int S) { return (double)t / ((double)S * (double)((t + S - 1) / S)); }

int64_t best_factor(int64_t fixed, int64_t lo, int64_t hi, int S) {
    int64_t best = lo;
    double be = -1.0;
    for (int64_t x = lo; x <= hi; ++x) {
        const double e = wave_eff(fixed * x, S);
        if (e > be + 1e-9) {
            be = e;
            best = x;
        }
    }
    return best;
}

// Block geometry of the schedule above (rows / columns).
struct Geo {
    int64_t R0, Ra, cb0, cb, Rp, Rlast;
    int nlast;
};

// Copy/compute simulation of the schedule (tools/e2e_sim.py --r02 is the same model): three
// in-order streams; a GEMM block starts when its copies have landed and the previous block is
// done, and takes ceil(tiles / (2 SMs)) waves of 64x64 tiles at the calibrated per-CTA rate
// (16384^3: 222 waves in 237.7 ms) + fixed costs; copies run at the measured pinned PCIe rates.
// Predicted 251.1 ms at 16384^3 (measured 250.8-252.0) and 38.7 ms for config 4 (38.5).
constexpr double kRateCta = 64.0 * 64.0 * 16384.0 * 2.0 / (237.7e-3 / 222.0);
constexpr double kD2H = 53e9;

double sim_gemm(int64_t m, int64_t n, int64_t K, int S) {
    const int64_t tiles = ((m + 63) / 64) * ((n + 63) / 64);
    return (double)((tiles + 2 * S - 1) / (2 * S)) * (64.0 * 64.0 * (double)K * 2.0 / kRateCta + 3e-6) + 4e-6;
}

double simulate(int64_t M, int64_t N, int64_t K, bool c_in, const Geo &g, int S) {
    double th = 0.0, tc = 0.0, td = 0.0;
    auto h2d = [&](double bytes) { th += bytes / kH2D; return th; };
    auto block = [&](double ready, int64_t nr, int64_t nc) {
        tc = std::max(tc, ready) + sim_gemm(nr, nc, K, S);
        td = std::max(td, tc) + 8.0 * (double)nr * (double)nc / kD2H;
    };
    const double row_bytes = 8.0 * (double)(K + (c_in ? N : 0));
    const int64_t R0 = std::min(M, g.R0), Ra = std::min(R0, g.Ra);
    double ready = h2d(row_bytes * (double)Ra);
    bool first = true;
    for (int64_t c0 = 0; c0 < N;) {
        const int64_t nc = std::min(N - c0, first ? g.cb0 : g.cb);
        ready = h2d(8.0 * (double)K * (double)nc);
        if (first && Ra < R0) {
            block(ready, Ra, nc);
            ready = h2d(row_bytes * (double)(R0 - Ra));
            block(ready, R0 - Ra, nc);
        } else {
            block(ready, R0, nc);
        }
        first = false;
        c0 += nc;
    }
    for (int64_t r0 = R0; r0 < M;) {
        const int64_t rem = M - r0;
        const int64_t nr = (rem <= g.Rlast || g.Rlast == 0) ? rem : (rem <= g.Rlast + g.Rp ? rem - g.Rlast : g.Rp);
        ready = h2d(row_bytes * (double)nr);
        const bool last = (r0 + nr >= M);
        const int64_t lcb = last ? std::max<int64_t>(kTn, ((N + g.nlast - 1) / g.nlast + kTn - 1) / kTn * kTn) : N;
        for (int64_t c0 = 0; c0 < N; c0 += lcb) block(ready, nr, std::min(N, c0 + lcb) - c0);
        r0 += nr;
    }
    return std::max(tc, td);
}

// The geometry for this shape: the wave-fill rule's (round 1), unless a coarse grid of
// alternatives simulates more than 1 % faster -- e.g. config 4 (32768 x 4096 x 4096), where the
// rule's 5888-row panels leave the device->host copies of C unoverlapped (38.7 -> 34.0 ms
// predicted).  Cached per shape; the search costs ~1 ms once.
Geo plan_geometry(int64_t M, int64_t N, int64_t K, bool c_in, int S, const Geo &rule) {
    static std::mutex mu;
    static std::map<std::tuple<int64_t, int64_t, int64_t, bool, int>, Geo> cache;
    const auto key = std::make_tuple(M, N, K, c_in, S);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    Geo best = rule;
    const double t_rule = simulate(M, N, K, c_in, rule, S);
    double t_best = t_rule;
    for (int64_t r0 : {16, 32, 48})
        for (int64_t ra : {4, 12, 16})
            for (int64_t cbt : {16, 24})
                for (int64_t rp : {16, 32, 48, 60, 92})
                    for (int64_t rl : {2, 4})
                        for (int nl : {1, 2}) {
                            const Geo g{64 * r0, 64 * ra, 64 * 16, 64 * cbt, 64 * rp, 64 * rl, nl};
                            const double t = simulate(M, N, K, c_in, g, S);
                            if (t < t_best) {
                                t_best = t;
                                best = g;
                            }
                        }
    if (t_best > 0.99 * t_rule) best = rule;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() > 256) cache.clear();
    cache[key] = best;
    return best;
}
// The block geometry of one gemm_f64_host call: one shot for tiny problems (< ~1 ms of GPU
// work), else the wave-fill rule's geometry or the simulated search's (plan_geometry).
Geo host_geometry(int64_t M, int64_t N, int64_t K, bool need_ab, bool need_c_in, int S) {
    const double flops = 2.0 * (double)M * (double)N * (double)K;
    if (!need_ab || flops < 2e10) return Geo{M, M, N, N, M, 0, 1};
    const int64_t tn_all = (N + kTn - 1) / kTn;
    const int64_t r_bal = (int64_t)(4.0 * kRate / kH2D / kTm) + 1;          // 11 tile rows
    const int64_t r0 = best_factor(std::min<int64_t>(tn_all, 24), r_bal, r_bal + 2, S);
    const int64_t R0 = std::min<int64_t>(M, r0 * kTm);
    const int64_t cbt = best_factor(r0, 16, 32, S);                          // 24 at S = 148
    const Geo rule{R0, std::min<int64_t>(R0, 3 * kTm), std::min<int64_t>(N, 16 * kTn), std::min<int64_t>(N, cbt * kTn),
                   best_factor(tn_all, 8, 24, S) * kTm /* 15 x 256 at N = 16384 */, kTm, N >= 2 * 512 ? 2 : 1};
    Geo g = plan_geometry(M, N, K, need_c_in, S, rule);
    g.R0 = std::min(M, g.R0);
    g.Ra = std::min(g.R0, g.Ra);
    g.cb0 = std::min(N, g.cb0);
    g.cb = std::min(N, g.cb);
    return g;
}
}  // namespace

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
    int S = 148;
    cudaDeviceGetAttribute(&S, cudaDevAttrMultiProcessorCount, dev);
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
    const Geo geo = host_geometry(M, N, K, need_ab, need_c_in, S);
    const int64_t R0 = geo.R0, Ra = geo.Ra, Rp = geo.Rp, Rlast = geo.Rlast, cb0 = geo.cb0, cb = geo.cb;
    const int64_t nlast = geo.nlast;
    // column blocks of panel 0: cb0, then cb each
    std::vector<std::pair<int64_t, int64_t>> cols;
    for (int64_t c0 = 0; c0 < N;) {
        const int64_t w = std::min(N - c0, cols.empty() ? cb0 : cb);
        cols.push_back({c0, w});
        c0 += w;
    }
    // later row panels: Rp rows each, the last one Rlast rows (thin: short final D2H)
    std::vector<std::pair<int64_t, int64_t>> rows;
    for (int64_t r0 = R0; r0 < M;) {
        const int64_t rem = M - r0;
        const int64_t nr = (rem <= Rlast || Rlast == 0) ? rem : (rem <= Rlast + Rp ? rem - Rlast : Rp);
        rows.push_back({r0, nr});
        r0 += nr;
    }
    const size_t nev = cols.size() + 2 + rows.size() * (size_t)(nlast + 1) + 8;
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

    // ---- row panel 0
    auto h2d_a = [&](int64_t r0, int64_t nr) -> int {
        int r = GEMM_OK;
        if (need_ab) r = h2d_rows(P.dA + r0 * K, K, A + r0 * lda, lda, K, nr, "H2D A rows");
        if (!r && need_c_in) r = h2d_rows(P.dC + r0 * N, N, C + r0 * ldc, ldc, N, nr, "H2D C rows");
        return r;
    };
    auto h2d_b = [&](int64_t c0, int64_t nc) -> int {
        if (!need_ab) return GEMM_OK;
        return cuda_check(cudaMemcpy2DAsync(P.dB + c0, N * 8, B + c0, ldb * 8, nc * 8, K, cudaMemcpyHostToDevice, P.h2d),
                          "H2D B block");
    };
    auto block = [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc) -> int {
        int r = run(r0, nr, c0, nc);
        if (!r) r = comp_done();
        if (!r) r = d2h_block(r0, nr, c0, nc);
        return r;
    };
    // Everything from here on enqueues asynchronous work that reads A, B, C (host memory the
    // caller may free once we return): on any error the three streams are drained before the
    // first error is returned, so the call stays synchronous on its error paths too.
    auto enqueue = [&]() -> int {
    int rc = GEMM_OK;
    if ((rc = h2d_a(0, Ra))) return rc;
    for (size_t j = 0; j < cols.size(); ++j) {
        const int64_t c0 = cols[j].first, nc = cols[j].second;
        if ((rc = h2d_b(c0, nc))) return rc;
        if ((rc = h2d_done())) return rc;
        if (j == 0 && Ra < R0) {   // block 0 on the first Ra rows while the rest of panel 0's A lands
            if ((rc = block(0, Ra, c0, nc))) return rc;
            if ((rc = h2d_a(Ra, R0 - Ra))) return rc;
            if ((rc = h2d_done())) return rc;
            if ((rc = block(Ra, R0 - Ra, c0, nc))) return rc;
        } else {
            if ((rc = block(0, R0, c0, nc))) return rc;
        }
    }
    // ---- later row panels
    for (size_t p = 0; p < rows.size(); ++p) {
        const int64_t r0 = rows[p].first, nr = rows[p].second;
        if ((rc = h2d_a(r0, nr))) return rc;
        if ((rc = h2d_done())) return rc;
        const bool last = (p + 1 == rows.size());
        const int64_t lcb = last ? std::max<int64_t>(kTn, ((N + nlast - 1) / nlast + kTn - 1) / kTn * kTn) : N;
        for (int64_t c0 = 0; c0 < N; c0 += lcb)
            if ((rc = block(r0, nr, c0, std::min(N, c0 + lcb) - c0))) return rc;
    }
    return GEMM_OK;
    };
    if ((rc = enqueue())) {
        const std::string first = last_error();
        cudaStreamSynchronize(P.h2d);
        cudaStreamSynchronize(P.comp);
        cudaStreamSynchronize(P.d2h);
        cudaGetLastError();
        return set_error(rc, "%s", first.c_str());
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

int gemm_host_plan(int64_t M, int64_t N, int64_t K, int beta_nonzero, int num_sms, int64_t geometry[7],
                   double *sim_seconds) {
    clear_error();
    if (M < 0 || N < 0 || K < 0) return set_error(GEMM_ERR_ARG, "negative shape");
    if (!geometry) return set_error(GEMM_ERR_ARG, "geometry is NULL");
    int S = num_sms;
    if (S <= 0) {
        int dev = 0;
        int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        if (!rc) rc = cuda_check(cudaDeviceGetAttribute(&S, cudaDevAttrMultiProcessorCount, dev), "SM count");
        if (rc) return rc;
    }
    const Geo g = host_geometry(M, N, K, M > 0 && N > 0 && K > 0, beta_nonzero != 0, S);
    const int64_t v[7] = {g.R0, g.Ra, g.cb0, g.cb, g.Rp, g.Rlast, g.nlast};
    for (int i = 0; i < 7; ++i) geometry[i] = v[i];
    if (sim_seconds) *sim_seconds = simulate(M, N, K, beta_nonzero != 0, g, S);
    return GEMM_OK;
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
