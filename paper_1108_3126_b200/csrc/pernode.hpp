// Launch interface of the thread-per-node engines (kernels_pernode.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rxg {

// Heap table in SoA form for the literal §8 protocol (device pointers).
struct RoundsTables {
    const uint8_t* kind = nullptr;
    const uint32_t* sym = nullptr;
    const int32_t* left = nullptr;
    const int32_t* right = nullptr;
    const int32_t* knode = nullptr;
    int32_t n = 0;
};

// Position-form bitset tables for K1 (device pointers).
struct PernodeTables {
    const uint8_t* cls = nullptr;
    const uint32_t* cmask = nullptr;
    const uint32_t* shift = nullptr;
    const uint32_t* has_group = nullptr;
    const int32_t* group = nullptr;
    const uint32_t* rows = nullptr;
    const uint32_t* trig = nullptr;
    const uint32_t* init = nullptr;
    int32_t W = 0, n_bits = 0, n_groups = 0, n_classes = 0;
};

constexpr int32_t kRoundsMaxNodes = 32 * 1024;   // one CTA of 1024 threads, <= 32 nodes each

// stats (device, 4 x u64, nullable): claims, rounds, macro steps, max claims per node per step.
// trace (device, zeroed, nullable): per symbol the next schedule as (N+1)-bit rows, bit N = null.
// enqueued (device u64, nullable): rx::LockstepStats.enqueued of the same
// string (every macro step's claims but the end-of-input step's);
// schedule (device, len + 1 x u32, nullable): ParStats.schedule_sizes.
cudaError_t launch_rounds(const RoundsTables& t, const uint8_t* text, uint64_t len, int32_t* accept,
                          unsigned long long* stats, uint32_t* trace, cudaStream_t st,
                          unsigned long long* enqueued = nullptr, uint32_t* schedule = nullptr);

// One par_task (single >= 0) or one run_rounds (single < 0) on caller-held
// ParState arrays in device memory: c, n (int64 x N), claims (u32 x N),
// flags {more_c, any_n, accept_pending, accept_next}; *launches = rounds.
cudaError_t launch_par(const RoundsTables& t, long long* c, long long* n, uint32_t* claims, int* flags, long long tt,
                       uint32_t symbol, int32_t single, unsigned long long* launches, cudaStream_t st);

// Segmented K1 (long strings across SMs): device scratch for up to
// max_segs segments of W words (pernode_seg_scratch_bytes), changed = 3
// zeroed round counters (16 bytes; zero again when the launch completes).
struct PernodeSegScratch {
    uint32_t* entry = nullptr;     // max_segs x W
    uint32_t* exits = nullptr;     // 2 x max_segs x W
    unsigned int* changed = nullptr;
    uint64_t max_segs = 0;
};
constexpr uint64_t kPernodeSegMin = 1ull << 20;   // strings at least this long are segmented
constexpr uint32_t kPernodeLookback = 1024;       // bytes walked from E0 to guess a segment's entry
constexpr uint64_t kPernodeMaxSegs = 8192;
inline size_t pernode_seg_scratch_bytes(int32_t W) { return 3 * kPernodeMaxSegs * static_cast<size_t>(W) * 4 + 64; }

// every > 0: E after every `every` symbols into checkpoints ((len/every) x W words; one warp).
// ss (nullable): strings >= kPernodeSegMin without checkpoints run as segments (cooperative launch).
cudaError_t launch_pernode(const PernodeTables& t, const uint8_t* text, uint64_t len, uint32_t every,
                           uint32_t* checkpoints, int32_t* accept, cudaStream_t st,
                           const PernodeSegScratch* ss = nullptr);

// K2b: warp-per-line bitset batch (line mode). scratch: lines_bitset_scratch_bytes(len).
size_t lines_bitset_scratch_bytes(uint64_t len);
cudaError_t launch_lines_bitset(const PernodeTables& t, const uint8_t* text, uint64_t len, uint8_t delim,
                                unsigned long long* count, uint8_t* results, void* scratch, size_t scratch_bytes,
                                int device, cudaStream_t st);

}  // namespace rxg
