// Host-side launch interface between the C ABI (capi.cu) and the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rxg {

// Device-resident shared-memory image plus the scalar offsets the kernels need.
struct DevTable {
    const void* img = nullptr;   // device copy of KTable::img
    uint32_t img_bytes = 0;
    bool cls = false;
    int esize = 2;
    uint32_t row_bytes = 0;
    uint32_t cls_off = 0;
    uint32_t ncols = 0;
    uint32_t start = 0, dead = 0, skip = 0, acc_shift = 0, tail_delta = 0;
    uint32_t term_acc = 0, term_rej = 0, delim_col = 0;
};

struct LaunchStats {
    uint32_t kernels = 0;   // kernels launched by the last call
};

// K2, delimited batch. `count` (device u64) is accumulated (caller zeroes it).
// `results` (device, one byte per line) and `line_base` are optional.
cudaError_t launch_lines(const DevTable& t, const uint8_t* text, uint64_t len, uint8_t delim,
                         uint32_t chunk, unsigned long long* count, uint8_t* results,
                         unsigned long long* scratch, size_t scratch_bytes, cudaStream_t st,
                         LaunchStats* ls);

// Chunk (bytes per chain) that gives one wave of resident chains over len.
uint32_t lines_auto_chunk(const DevTable& t, uint64_t len);

// Bytes of scratch launch_lines needs when results != nullptr.
size_t lines_scratch_bytes(uint64_t len, uint32_t chunk);

// K2, fixed-stride batch: strings text[i*stride, (i+1)*stride), i < n.
cudaError_t launch_fixed(const DevTable& t, const uint8_t* text, uint64_t n, uint32_t stride,
                         unsigned long long* count, uint8_t* results, cudaStream_t st, LaunchStats* ls);

// Same, on a raw-byte u16 table image whose entries were rebased by +0x400
// (absolute shared addresses; stride must be a multiple of 16).
cudaError_t launch_fixed_abs(const DevTable& t_abs, const uint8_t* text, uint64_t n, uint32_t stride,
                             unsigned long long* count, uint8_t* results, cudaStream_t st, LaunchStats* ls);

int device_sm_count(int device);

// Per-(heap, stream) completion slot in device memory, all zero when idle:
// [0] count accumulator, [1] CTA ticket, [2] aux (chunk engine: ~first wrong
// range). Kernels add their counts to [0]; the last CTA to finish publishes
// the total to the caller's counter (overwrite, or add when accumulating)
// and zeroes the slot again, so no memset launch precedes a call. Launches
// that share a slot are ordered by their stream.
struct CountSlot {
    unsigned long long* p = nullptr;
    bool accumulate = false;
    unsigned int* seam = nullptr;   // chunked engine: zeroed seam counters of this stream
};

// Fixed stride on the TMA data path (stride a multiple of 32; the absolute
// raw-byte u16 table plus a 144 KB ring must fit shared memory).
bool fixed_tma_fits(uint32_t img_bytes, uint32_t stride, int smem_limit);
// *n_done = strings handled (stride 32 leaves the last n % 4 to the caller).
cudaError_t launch_fixed_tma(const DevTable& t_abs, const uint8_t* text, uint64_t n, uint32_t stride,
                             unsigned long long* count, uint8_t* results, CountSlot cs, int device, cudaStream_t st,
                             uint64_t* n_done);

// Stream-ordered store of 0 or ~0 to one u64 (counters, tickets).
cudaError_t write_u64(void* dst, uint64_t value, cudaStream_t st);

}  // namespace rxg
