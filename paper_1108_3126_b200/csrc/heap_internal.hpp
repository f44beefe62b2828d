// Internal definition of the rxg_heap handle (include/rxg.h) and the host
// helpers shared by capi.cu (single device) and multi.cu (communicators and
// the persistent multi-device handle). Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rxg.h"
#include "launch.hpp"
#include "bits.hpp"
#include "lines_tma.hpp"
#include "pernode.hpp"
#include "program.hpp"
#include "tables.hpp"

namespace rxg {

// A TMA table image published to launches. Never mutated after publication:
// a retune (rxg_heap_tune) builds a new one and swaps the shared_ptr under
// rxg_heap::mu; launches copy the shared_ptr under the same lock, so a
// launch never reads a half-replaced table. The device copies are owned by
// the heap (rxg_heap::allocs) and freed only when the heap is destroyed, so
// a kernel still running on a replaced image (or a CUDA graph captured
// earlier) keeps valid memory.
struct ChunkImage {
    LtTable lt;
    const void* d = nullptr;   // device copy of lt.lo
};

struct TableSlot {
    KTable host;
    DevTable dev;
    std::shared_ptr<const LtTable> lt;        // TMA line layout (delimited slots; null or !ok if it does not fit)
    DevTable abs;                             // plain slot: entries rebased to absolute shared addresses
    bool has_abs = false;
    std::shared_ptr<const ChunkImage> chunk;  // plain slot: TMA chunk-parallel layout (null or !lt.ok if it does not fit)
};

constexpr int32_t kMaxDfaStates = 16384;

// Occurrences of byte d in p[0, n): eight bytes per step, exact (a byte of
// x ^ d is zero iff bit 7 of ((y & 0x7f) + 0x7f) | y is clear).
inline uint64_t count_byte(const uint8_t* p, size_t n, uint8_t d) {
    constexpr uint64_t lo7 = 0x7f7f7f7f7f7f7f7full, ones = 0x0101010101010101ull;
    const uint64_t pat = ones * d;
    uint64_t total = 0;
    size_t i = 0;
    while (i + 8 <= n) {
        uint64_t acc = 0;   // per-byte hit counts, at most 255 steps before they are summed
        const size_t stop = std::min(n & ~size_t(7), i + 8 * 255);
        for (; i < stop; i += 8) {
            uint64_t x;
            std::memcpy(&x, p + i, 8);
            x ^= pat;
            acc += (~(((x & lo7) + lo7) | x) >> 7) & ones;
        }
        acc = (acc & 0x00ff00ff00ff00ffull) + ((acc >> 8) & 0x00ff00ff00ff00ffull);
        total += (acc * 0x0001000100010001ull) >> 48;
    }
    for (; i < n; ++i) total += p[i] == d;
    return total;
}

// A few host threads that copy one buffer in parallel (pageable input into
// pinned staging: one thread's memcpy runs far below the PCIe link), counting
// a delimiter byte on the way (the per-string results' offsets) while the
// bytes are in cache; with dst null they only count.
class HostCopyPool {
public:
    explicit HostCopyPool(unsigned n) : n_(n ? n : 1) {
        for (unsigned k = 0; k < n_; ++k) threads_.emplace_back([this, k] { loop(k); });
    }
    ~HostCopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            quit_ = true;
        }
        go_.notify_all();
        for (auto& t : threads_) t.join();
    }
    // Returns the number of `delim` bytes in src[0, n) (0 when delim < 0).
    uint64_t copy(void* dst, const void* src, size_t n, int delim = -1) {
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = static_cast<uint8_t*>(dst);
        src_ = static_cast<const uint8_t*>(src);
        len_ = n;
        delim_ = delim;
        hits_ = 0;
        pending_ = n_;
        ++gen_;
        go_.notify_all();
        done_.wait(lk, [&] { return pending_ == 0; });
        return hits_;
    }

private:
    void loop(unsigned k) {
        uint64_t seen = 0;
        for (;;) {
            uint8_t* d;
            const uint8_t* s;
            size_t n;
            int delim;
            {
                std::unique_lock<std::mutex> lk(mu_);
                go_.wait(lk, [&] { return quit_ || gen_ != seen; });
                if (quit_) return;
                seen = gen_;
                d = dst_;
                s = src_;
                n = len_;
                delim = delim_;
            }
            const size_t part = (n / n_ + 4095) & ~size_t(4095);
            const size_t lo = std::min(n, part * k), hi = std::min(n, lo + part);
            uint64_t hits = 0;
            constexpr size_t kSub = 256u << 10;   // copy, then count from cache
            for (size_t at = lo; at < hi; at += kSub) {
                const size_t m = std::min(kSub, hi - at);
                if (d) std::memcpy(d + at, s + at, m);
                if (delim >= 0) hits += count_byte((d ? d : s) + at, m, static_cast<uint8_t>(delim));
            }
            std::lock_guard<std::mutex> lk(mu_);
            hits_ += hits;
            if (--pending_ == 0) done_.notify_all();
        }
    }
    unsigned n_;
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable go_, done_;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool quit_ = false;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t len_ = 0;
    int delim_ = -1;
    uint64_t hits_ = 0;
};

}  // namespace rxg

struct rxg_heap {
    int device = -1;
    rxg::Program prog;
    bool dfa_ok = false;
    bool tma_ok = true;     // the dynamic shared window starts at 0x400 (the TMA layouts' absolute addresses)
    int32_t dfa_sets = 0;   // states before minimisation
    uint32_t lookback = 64; // chunk engine lookback (rxg_heap_tune with delimiter -1 shortens it)
    rxg::Dfa dfa;
    int smem_limit = 0;
    std::mutex mu;          // guards everything below that is created lazily or replaced
    std::mutex host_mu;     // host-buffer calls share the staging buffers and streams
    std::unique_ptr<rxg::TableSlot> plain;
    std::map<int, std::unique_ptr<rxg::TableSlot>> lines;
    std::map<int, std::vector<double>> line_freq;   // sampled state x byte counts per delimiter (rxg_heap_tune)
    // device allocations of table images and retired stream scratch: freed with the heap
    std::vector<void*> allocs;
    // staging for host-buffer calls
    uint8_t* d_stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    // pageable host input: pinned staging pieces, filled by a few host threads
    uint8_t* h_pin[2] = {nullptr, nullptr};
    size_t pin_bytes = 0;
    std::unique_ptr<rxg::HostCopyPool> copier;
    // per-string results of host-buffer calls: a device and a pinned slot per
    // pipeline stage (piece k's results cross while piece k+1 is matched)
    uint8_t* d_rres[2] = {nullptr, nullptr};
    uint8_t* h_rres[2] = {nullptr, nullptr};
    size_t rres_bytes[2] = {0, 0};   // grow-only, sized by the strings a piece holds
    unsigned long long* d_count = nullptr;
    int32_t* d_accept = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    // lazily built tables of the thread-per-node engines
    void* d_rounds = nullptr;
    rxg::RoundsTables rounds;
    void* d_pernode = nullptr;
    rxg::PernodeTables pernode;
    // K2b tables on the TMA path per delimiter (-1: fixed stride); a null entry: not supported
    std::map<int, std::shared_ptr<const rxg::BitsImage>> bits;
    // Per stream, keyed by cudaStreamGetId (so cudaStreamPerThread from two
    // threads gives two keys): the CountSlot (launch.hpp, zero when idle), the
    // chunked engine's seam arrival counters (zero when idle, grow-only) and
    // its scratch (guesses, exits, checkpoints; grow-only).
    std::map<unsigned long long, unsigned long long*> slots;
    std::map<unsigned long long, std::pair<unsigned int*, size_t>> seams;
    std::map<unsigned long long, std::pair<void*, size_t>> scratch;

    ~rxg_heap();
};

namespace rxg {
namespace detail {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
void set_launches(int n);
int launches();

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int need_device(rxg_heap* h, bool dfa = true);

// A heap for `device` with the program, memoized step and tuning of `proto`
// (built once on the host, uploaded per device).
int clone_heap(const rxg_heap* proto, int device, rxg_heap** out);
// Copy proto's sampled placement for `delimiter` into h and rebuild h's tables.
int adopt_tuning(rxg_heap* h, const rxg_heap* proto, int32_t delimiter);

// Batch on device buffers with engine selection; zero_count = overwrite the
// count (false: accumulate).
int batch_any(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride, int engine,
              unsigned long long* d_count, uint8_t* d_results, cudaStream_t st, bool zero_count);

// The pipelined host-buffer path (pieces of 64 MiB: copy k+1 while matching k).
// On return (RXG_OK) the stream is idle, h->d_count holds the count, and the
// results / utf8 check are in host memory; *count (nullable) is read back.
int host_batch(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* count,
               uint8_t* results, uint64_t* utf8_first_bad);

uint64_t count_strings(const uint8_t* text, uint64_t lo, uint64_t hi, int32_t delimiter, uint32_t stride);

}  // namespace detail
}  // namespace rxg
