// Launch interface for the single-string engines.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "launch.hpp"

namespace rxg {

cudaError_t launch_seq(const DevTable& t, const uint8_t* text, uint64_t len, int32_t* accept, cudaStream_t st);

}  // namespace rxg
