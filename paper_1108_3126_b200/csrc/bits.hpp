// K2b on the TMA data path (kernels_bits_tma.cu): tables and launch API.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "launch.hpp"
#include "program.hpp"

namespace rxg {

constexpr int32_t kBitsMaxWords = 16;                 // position set per lane: 511 positions + A
constexpr uint32_t kBitsMaxTableBytes = 96 * 1024;    // shared-memory image budget

// Bitset step tables in the kernel's bit order (positions 0..n_pos-1, the
// accept bit A at bit 32*WT - 1), for one delimiter (-1: fixed stride).
// WT <= 4: one row per byte [M, D] (M = the positions the byte matches,
//   D = all ones on the delimiter), then (T_g, R_g) of groups g >= 2 as
//   broadcast rows; regs = SH, E0, T_0, R_0, T_1, R_1 (kept in registers;
//   SH = positions whose follow is the next position, T_g = positions whose
//   residual follow row is R_g).
// WT 8, 16: one row per byte [M, D, pad]; then SH, E0 and (T_g, R_g) for
//   every group, read as shared-memory broadcasts.
struct BitsTables {
    bool ok = false;
    int32_t WT = 0, G = 0, GR = 2;
    uint32_t row_words = 0, xt_row_words = 0;
    std::vector<uint32_t> img, regs;
    uint32_t cmap_off = 0, xt_off = 0, xg_off = 0;   // byte offsets in img
};

BitsTables make_bits_tables(const Program& p, int32_t delim);

// Device copies (owned by the heap).
struct BitsImage {
    BitsTables t;
    const void* d_img = nullptr;
    const uint32_t* d_regs = nullptr;
};

// delimiter >= 0: lines; < 0: strings at `stride`. scratch: bits_scratch_bytes
// (results in line mode only; else may be null).
size_t bits_scratch_bytes(uint64_t len, uint32_t chunk, bool lines, bool results);
uint32_t bits_chunk(const BitsImage& b, uint64_t len, int32_t delimiter, uint32_t stride, uint32_t chunk);
cudaError_t launch_bits(const BitsImage& b, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                        uint32_t chunk, unsigned long long* count, uint8_t* results, void* scratch,
                        size_t scratch_bytes, CountSlot cs, cudaStream_t st);

}  // namespace rxg
