// Launch interface of the chunk-parallel single-string walk (kernels_chunked.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "launch.hpp"
#include "lines_tma.hpp"

namespace rxg {

size_t chunked_scratch_bytes(uint64_t len, uint32_t chunk);
uint32_t chunked_auto_chunk(const DevTable& t, uint64_t len, int device);

// scratch: chunked_scratch_bytes(len, chunk) device bytes. repairs: device u64 (nullable).
// entry: table state the string starts in (kStartState = the start state);
// exit_state (device, nullable) receives the table state after the string.
constexpr uint32_t kStartState = 0xFFFFFFFFu;
cudaError_t launch_chunked(const DevTable& t, const uint8_t* text, uint64_t len, uint32_t chunk, uint32_t lookback,
                           void* scratch, int32_t* accept, unsigned long long* repairs, int device, cudaStream_t st,
                           uint32_t entry = kStartState, uint32_t* exit_state = nullptr);

// TMA-staged variant (tables from make_chunk_tma_table; d_img = device copy of t.lo).
uint32_t chunked_tma_auto_chunk(const LtTable& t, uint64_t len, int device);
size_t chunked_tma_scratch_bytes(uint64_t len, uint32_t chunk);
cudaError_t launch_chunked_tma(const LtTable& t, const void* d_img, const uint8_t* text, uint64_t len, uint32_t chunk,
                               uint32_t lookback, void* scratch, int32_t* accept, unsigned long long* repairs,
                               CountSlot cs, int device, cudaStream_t st, uint32_t entry = kStartState,
                               uint32_t* exit_state = nullptr);

}  // namespace rxg
