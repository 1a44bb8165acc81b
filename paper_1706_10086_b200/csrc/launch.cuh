// launch.cuh -- kernel launch with programmatic dependent launch (PDL), shared by the FP64
// and FP32 translation units.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

#include "ptx.cuh"

namespace dg {

#ifdef DG_TRACE
void *trace_device_ptr();   // gemm_f64.cu: the buffer gemm_trace_set() registered (or NULL)
#endif

// Every GEMM kernel is launched with programmatic stream serialization (PDL): it may become
// resident while the previous kernel of the stream drains and waits for it in-kernel
// (griddep_wait in ptx.cuh) before touching global memory.  GEMM_PDL=0 in the environment
// launches them the classic way (A/B measurements).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("GEMM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
#ifdef DG_TRACE
    // only when the registered buffer changed, so back-to-back traced launches keep their
    // programmatic-dependent-launch overlap (no copy node between them)
    void *tp = trace_device_ptr();
    if (tp != dg_trace_last) {   // both per translation unit, like dg_trace_buf
        cudaMemcpyToSymbolAsync(dg_trace_buf, &tp, sizeof(tp), 0, cudaMemcpyHostToDevice, st);
        dg_trace_last = tp;
    }
#endif
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// The same with a thread-block cluster of (cx, cy, 1) CTAs (cluster split-K).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                    unsigned cx, unsigned cy, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cx;
    attr[0].val.clusterDim.y = cy;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
#ifdef DG_TRACE
    void *tp = trace_device_ptr();
    if (tp != dg_trace_last) {
        cudaMemcpyToSymbolAsync(dg_trace_buf, &tp, sizeof(tp), 0, cudaMemcpyHostToDevice, st);
        dg_trace_last = tp;
    }
#endif
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dg
