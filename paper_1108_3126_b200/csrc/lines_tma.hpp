// TMA-staged line kernel: constants, shared-memory layout and launch API.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "launch.hpp"
#include "program.hpp"

namespace rxg {

constexpr uint32_t kLtSmemBase = 0x400;           // dynamic shared window start (1 KB reserved)
constexpr uint32_t kLtAccAddr = 0x8000;           // START_A row: the only main-loop row with bit 15
constexpr uint32_t kLtColBytes = 4;               // column stride: byte b of a row -> bank (row + b) mod 32
constexpr uint32_t kLtRowBytes = 256 * kLtColBytes;

// Host-built absolute-address layout of one line table (+ stage ring).
// Two layouts:
//   direct (cls = false): rows of 256 u16 entries at 4-byte column stride,
//     entries and states are absolute shared addresses, START_A = 0x8000;
//   class  (cls = true):  rows indexed by byte class, entries and states are
//     row indices, a 256-entry u32 class map holds the absolute address of
//     each byte's column in row 0 (addr = row * row_bytes + cmap[b]), and
//     START_A is row 2^acc_shift (tail copies and TERM rows above it).
struct LtTable {
    bool ok = false;                 // false if the DFA is too large for this layout
    bool cls = false;
    uint32_t row_bytes = 0, cmap_addr = 0, acc_shift = 15;
    uint32_t hole_lo = 0, hole_hi = 0;   // unused rows inside the table (class layout): stage slots go here
    uint32_t acc_off = 0;                // plain (chunk) tables: byte offset of a row's accept flag
    uint32_t col_bytes = kLtColBytes;    // direct layouts: column stride (entry for byte b at row + col_bytes*b)
    uint32_t range_x = 0, range_k = 0;   // class layout with range-clamped columns: column = min(b ^ x, k) (k = 0: class map)
    // packed layout (chunk tables, DFA <= kLtPackedMaxStates): one u32 per byte holding the
    // whole transition function, 5-bit fields next*5 at bit 5*state, replicated per lane
    // (word for byte b, lane l at 0x400 + 128 b + 4 l); states are 5*state, acc_mask bit i = accept(i)
    bool packed = false;
    uint32_t acc_mask = 0;
    // packed chunk tables: states of the automaton when a byte permutes two or
    // more of them (input runs of it never synchronise a lookback guess, e.g.
    // (aaa)* over a's): the engine then computes every range's transfer
    // function directly instead of guessing entries first; 0 = guess
    uint32_t fn_states = 0;
    std::vector<uint8_t> lo, hi;     // images of [lo_addr, +lo) main rows and [hi_addr, +hi) upper rows
    uint32_t lo_addr = 0, hi_addr = 0;
    uint32_t lo_bytes = 0, hi_bytes = 0;
    uint32_t start = 0, skip = 0, void_row = 0, tail_delta = 0, term_acc = 0, term_rej = 0;
    uint32_t smem_table_end = 0;     // end of the table regions (stage ring placed at launch)
    // device copies
    void* d_lo = nullptr;
    void* d_hi = nullptr;
};

// freq: (S+2) x 256 state-by-byte visit counts of a sample (lt_sample_freq);
// null = default bank placement.
LtTable make_lines_tma_table(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq = nullptr,
                             bool force_class = false);
std::vector<double> lt_sample_freq(const Program& p, const Dfa& d, uint8_t delim, const uint8_t* sample, uint64_t len);
// Shortest lookback in {16, 32, 64} whose guess (walk the k bytes before a
// position from the start state) is the true state at >= 99.9% of the
// sample's positions: the chunk engine's default for this pattern.
uint32_t lt_sync_lookback(const Program& p, const Dfa& d, const uint8_t* sample, uint64_t len);
// Same for one long string (no delimiter): S x 256 counts.
std::vector<double> lt_sample_freq_plain(const Program& p, const Dfa& d, const uint8_t* sample, uint64_t len);

// Plain table (no delimiter) for the chunk-parallel single-string kernel:
// direct layout (accept flag in the high half of column 0) for small DFAs,
// class layout (accept flag in an extra column) otherwise. freq: S x 256
// state-by-byte counts of a sample (nullable). Rows start at 0x400; the
// stage ring goes after smem_table_end.
LtTable make_chunk_tma_table(const Program& p, const Dfa& d, const std::vector<double>* freq = nullptr);

// Row pairing + bank placement of the direct layouts (see lines_tma_table.cpp).
struct RowPlacement {
    std::vector<uint32_t> pair, half;   // per row: its group and 2-byte slot in the group
    std::vector<uint32_t> pair_off;     // per group: bank offset (words mod 32)
    uint32_t npairs = 0;                // groups
    uint32_t col_bytes = kLtColBytes;
};
uint32_t lt_choose_col_bytes(const std::vector<double>* freq, uint32_t nrows);
RowPlacement lt_place_groups(const std::vector<double>* freq, uint32_t nrows, uint32_t col_bytes, bool group_rows);

// Host emulation of the table walk, for CPU tests.
uint32_t lt_step(const LtTable& t, uint32_t s, uint8_t byte);
// Same for the plain (chunk) tables; lt_chunk_accept: accept bit of a table state.
uint32_t lt_chunk_step(const LtTable& t, uint32_t s, uint8_t byte);
bool lt_chunk_accept(const LtTable& t, uint32_t s);
inline uint32_t lt_count(const LtTable& t, uint32_t s) { return s >> t.acc_shift; }

// Largest DFA the direct layouts take (rows of 256 columns, absolute u16
// addresses below 64 KB: two rows per column word for lines, one for the
// single-string table); bigger ones use the class layout.
constexpr int32_t kLtDirectMaxStates = 52;
constexpr int32_t kLtChunkDirectMaxStates = 56;
constexpr int32_t kLtPackedMaxStates = 6;

// chunk = bytes per range (multiple of lines_tma_slice()), 0 = one wave of ranges.
cudaError_t launch_lines_tma(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                             unsigned long long* count, CountSlot cs, cudaStream_t st);
uint32_t lines_tma_slice();

// Per-line results on the same kernel: a delimiter count per range, an
// exclusive scan (the line index of each range's first line), then the walk
// writes results[line] at every delimiter of an owned line and for its tail.
// chunk must be the effective one (lines_tma_chunk); scratch on device.
uint32_t lines_tma_chunk(const LtTable& t, uint64_t len, uint32_t chunk);
size_t lines_tma_results_scratch(uint64_t len, uint32_t chunk);
cudaError_t launch_lines_tma_results(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim,
                                     uint32_t chunk, unsigned long long* count, uint8_t* results, void* scratch,
                                     size_t scratch_bytes, CountSlot cs, cudaStream_t st);

}  // namespace rxg
