// aux.cu -- input synthesis and FP64 peak microbenchmarks (no GEMM arithmetic).
//
// gemm_fill_f64: the device twin of synth/__init__.py's counter-based generator
// (SplitMix64 finaliser at a logical (row, col) index); tests check the two bitwise.
// gemm_peak_probe: DMMA.8x8x4 / DFMA throughput loops that calibrate the FP64 roof
// (Eq. (8), P(f,o,n) = f*o*n: clock x FLOP/clk/SM x SMs).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/gemm_f64.h"
#include "internal.h"
#include "ptx.cuh"

namespace dg {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

static uint64_t host_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void fill_kernel(int mode, uint64_t base, int64_t cols, int64_t row0, int64_t nrows, double *X,
                            int64_t ldx) {
    const int64_t total = nrows * cols;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cols, j = idx - r * cols;
        const int64_t i = row0 + r;
        double v;
        if (mode == 3) {
            v = 1.0;
        } else if (mode == 4) {
            v = (i == j) ? 1.0 : 0.0;
        } else if (mode == 5) {
            v = 0.0;
        } else {
            const uint64_t ctr = (uint64_t)i * (uint64_t)cols + (uint64_t)j + 1ull;
            const uint64_t bits = mix64(base + ctr * 0x9E3779B97F4A7C15ull) >> 11;
            if (mode == 0)
                v = 2.0 * ((double)bits * 0x1.0p-53) - 1.0;
            else if (mode == 1)
                v = (double)((int64_t)(bits % 513ull) - 256) / 256.0;
            else
                v = (double)((int64_t)(bits % 17ull) - 8);
        }
        X[r * ldx + j] = v;
    }
}

// 8 independent accumulator chains per warp; each round = 8 DMMA.8x8x4.
__global__ void dmma_probe_kernel(int64_t iters, double *out, int64_t *cycles) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    const long long t0 = clock64();
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_m8n8k4(c[i][0], c[i][1], a, b);
    }
    const long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    // one value per block: keeps the chains live without a reduction
    if (threadIdx.x == 0) {
        out[blockIdx.x] = s;
        if (blockIdx.x == 0 && cycles) cycles[0] = t1 - t0;
    }
}

__global__ void dfma_probe_kernel(int64_t iters, double *out, int64_t *cycles) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i * 1e-3;
    const long long t0 = clock64();
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
    }
    const long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (threadIdx.x == 0) {
        out[blockIdx.x] = s;
        if (blockIdx.x == 0 && cycles) cycles[0] = t1 - t0;
    }
}

}  // namespace dg

using namespace dg;

extern "C" {

int gemm_fill_f64(int mode, uint64_t seed, int mat, int64_t rows, int64_t cols, int64_t row0, int64_t nrows,
                  double *X, int64_t ldx, void *stream) {
    clear_error();
    if (mode < 0 || mode > 5) return set_error(GEMM_ERR_ARG, "mode=%d not in 0..5", mode);
    if (rows < 0 || cols < 0 || row0 < 0 || nrows < 0 || row0 + nrows > rows)
        return set_error(GEMM_ERR_ARG, "row slab [%lld,%lld) outside [0,%lld) or negative cols", (long long)row0,
                         (long long)(row0 + nrows), (long long)rows);
    if (nrows == 0 || cols == 0) return GEMM_OK;
    if (!X) return set_error(GEMM_ERR_ARG, "X is NULL");
    if (ldx < cols) return set_error(GEMM_ERR_ARG, "ldx=%lld < cols=%lld", (long long)ldx, (long long)cols);
    const uint64_t base = host_mix64(seed * 0x9E3779B97F4A7C15ull + (uint64_t)(mat + 1) * 0xD1B54A32D192ED03ull);
    const int64_t total = nrows * cols;
    const int threads = 256;
    const int blocks = (int)((total + threads - 1) / threads < 148 * 32 ? (total + threads - 1) / threads : 148 * 32);
    fill_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(mode, base, cols, row0, nrows, X, ldx);
    return cuda_check(cudaGetLastError(), "fill_kernel launch");
}

int gemm_peak_probe(int kind, int blocks, int warps, int64_t iters, double *out, int64_t *cycles_out,
                    void *stream) {
    clear_error();
    if (kind != 0 && kind != 1) return set_error(GEMM_ERR_ARG, "kind=%d must be 0 (DMMA) or 1 (DFMA)", kind);
    if (blocks <= 0 || warps <= 0 || warps > 32 || iters <= 0 || !out)
        return set_error(GEMM_ERR_ARG, "bad probe arguments (blocks=%d warps=%d iters=%lld out=%p)", blocks, warps,
                         (long long)iters, (void *)out);
    if (kind == 0)
        dmma_probe_kernel<<<blocks, warps * 32, 0, (cudaStream_t)stream>>>(iters, out, cycles_out);
    else
        dfma_probe_kernel<<<blocks, warps * 32, 0, (cudaStream_t)stream>>>(iters, out, cycles_out);
    return cuda_check(cudaGetLastError(), "peak probe launch");
}

}  // extern "C"
