// internal.h -- launchers shared between the kernel TUs and the C ABI (capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace miso_b200 {

cudaError_t launch_optimize(const double* speeds, const uint32_t* offsets, uint64_t n,
                            uint8_t* cand, double* obj, uint64_t en0, uint64_t en1,
                            cudaStream_t stream);

}  // namespace miso_b200
