// host_util.h -- host-side helpers for the C ABI entry points.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <utility>

#include "specdec.h"

namespace specdec {

int record_cuda_error(cudaError_t e);  // stores the message, returns SPECDEC_ERR_CUDA
int device_sm_count();                 // SMs of the current device (cached per device)

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int dtype_size(int dtype) {
    switch (dtype) {
        case SPECDEC_F32: return 4;
        case SPECDEC_F16: return 2;
        case SPECDEC_BF16: return 2;
        default: return 0;
    }
}

inline int check_launch() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPECDEC_OK : record_cuda_error(e);
}

bool pdl_enabled();  // SPECDEC_PDL (default on), unless suppressed on this thread
void pdl_suppress(bool on);             // nestable: launches on this thread without PDL
int annotate_error(int rc, const char *where);  // prefixes the last CUDA error message
void ensure_carveout(const void *fn);   // SPECDEC_CARVEOUT: one shared-memory carveout for all kernels

// Launch with the programmatic-stream-serialization attribute (PDL) when enabled; the
// kernels call pdl_wait() before reading anything a predecessor may write.
template <typename... KArgs, typename... Args>
int launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
             Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    ensure_carveout(reinterpret_cast<const void *>(kernel));
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    return e == cudaSuccess ? SPECDEC_OK : record_cuda_error(e);
}

}  // namespace specdec
