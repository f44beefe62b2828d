// Device UTF-8 validation with decode_utf8's error positions (utf8.cpp:16-46).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rxg {

// atomicMin(*first_bad, base + i) for the first byte i of [text, text+len) at
// which rx::decode_utf8 would throw, decoding every string of the buffer
// separately: strings end at `delim` (0..127; -1 = none) and/or every
// `stride` bytes (0 = none). *first_bad is not written when the buffer is
// valid, so the caller initialises it (UINT64_MAX).
cudaError_t launch_utf8_check(const uint8_t* text, uint64_t len, int32_t delim, uint32_t stride, uint64_t base,
                              unsigned long long* first_bad, int device, cudaStream_t st);

}  // namespace rxg
