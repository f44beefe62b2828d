// Launch interface of the multi-heap batch (kernels_many.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rxg {

struct ManyDev {
    const uint8_t* tables = nullptr;
    const uint64_t* table_off = nullptr;
    const uint32_t* meta = nullptr;
    const uint8_t* text = nullptr;
    const uint64_t* str_off = nullptr;
};

cudaError_t launch_many(const ManyDev& d, uint64_t n_patterns, uint64_t n_strings, uint32_t sep, uint8_t* results,
                        uint32_t max_table_bytes, int device, cudaStream_t st);

}  // namespace rxg
