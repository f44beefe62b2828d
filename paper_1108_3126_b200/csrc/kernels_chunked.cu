// Chunk-parallel walk of one long string (RXG_ENGINE_CHUNKED).
//
// The memoized step is a deterministic transition function, so a string can
// be cut into P ranges that are walked concurrently if each range knows its
// entry state. Phase 1 guesses it: range j first walks the `lookback` bytes
// before its start from the start state (for patterns whose state is fixed
// by a bounded suffix of the input, e.g. (a|b)*abb or a keyword union, the
// guess is exact), then walks its own bytes, recording the entry guess g[j],
// the exit state e[j] and the state every kMid bytes.
// Phase 2 (one warp, in order) repairs the chain of entry states: range j is
// exact iff its entry equals the exact exit of range j-1. On a mismatch the
// range is re-walked from the exact entry until its state meets the recorded
// trajectory at a kMid checkpoint (from there on both walks coincide), or to
// its end. The result is exact for every pattern; only the amount of phase 2
// work depends on how quickly the automaton forgets its past.
#include <cstdint>

#include "chunked.hpp"

namespace rxg {

namespace {

constexpr uint32_t kMid = 64;   // trajectory checkpoint period (bytes)

struct ChunkArgs {
    const uint8_t* text;
    uint64_t len;
    uint32_t chunk;      // bytes per range (multiple of kMid)
    uint32_t lookback;
    uint64_t nranges;
    const uint4* img;
    uint32_t img_words;
    uint32_t cls_off, start, dead, acc_col;
    uint32_t* g;         // nranges
    uint32_t* e;         // nranges
    uint32_t* mid;       // nranges x (chunk / kMid)
    int32_t* accept;
    uint32_t entry;                // table state the string starts in
    uint32_t* exit_state;          // nullable: table state after the string
    unsigned long long* repairs;   // ranges re-walked (instrumentation, nullable)
    unsigned int* ticket;          // zeroed before the walk: CTAs finished
    unsigned long long* first_bad; // set to ~0 before the walk: first range whose entry guess is wrong
};

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

template <typename E, bool CLS>
__device__ __forceinline__ uint32_t step(const uint8_t* sm, uint32_t cls_off, uint32_t s, uint32_t b) {
    const uint32_t col = CLS ? static_cast<uint32_t>(sm[cls_off + b]) : b;
    return *reinterpret_cast<const E*>(sm + s + col * static_cast<uint32_t>(sizeof(E)));
}

template <typename E, bool CLS>
__device__ uint32_t walk(const ChunkArgs& a, const uint8_t* sm, uint32_t s, uint64_t lo, uint64_t hi) {
    uint64_t p = lo;
    for (; p < hi && (p & 15); ++p) s = step<E, CLS>(sm, a.cls_off, s, a.text[p]);
    for (; p + 16 <= hi; p += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + p));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) s = step<E, CLS>(sm, a.cls_off, s, (word_of(v, w) >> (8 * k)) & 0xFFu);
    }
    for (; p < hi; ++p) s = step<E, CLS>(sm, a.cls_off, s, a.text[p]);
    return s;
}

__device__ __forceinline__ void load_table(uint8_t* sm, const uint4* img, uint32_t words) {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = img[i];
    __syncthreads();
}

template <typename E, bool CLS>
__global__ void __launch_bounds__(256) k_chunk_walk(const __grid_constant__ ChunkArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    load_table(sm, a.img, a.img_words);
    const uint32_t per = a.chunk / kMid;
    const uint32_t lane = threadIdx.x & 31;
    // whole warps iterate together (ranges j = base + tid), so the boundary
    // j-1 -> j is checked from registers for every lane but lane 0
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < a.nranges; base += stride) {
        const uint64_t j = base + threadIdx.x;
        const bool live = j < a.nranges;
        uint32_t s = a.entry, guess = a.entry;
        if (live) {
            const uint64_t c0 = j * a.chunk;
            const uint64_t c1 = min(c0 + a.chunk, a.len);
            if (j > 0) s = walk<E, CLS>(a, sm, a.start, c0 > a.lookback ? c0 - a.lookback : 0, c0);
            guess = s;
            a.g[j] = s;
            uint32_t* mid = a.mid + j * per;
            uint32_t k = 0;
            for (uint64_t p = c0; p < c1; p += kMid, ++k) {
                s = walk<E, CLS>(a, sm, s, p, min(p + kMid, c1));
                mid[k] = s;
            }
            a.e[j] = s;
        }
        const uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, s, 1);
        const uint32_t bad = __reduce_min_sync(0xFFFFFFFFu, live && lane > 0 && guess != prev ? lane : ~0u);
        if (lane == 0 && bad != ~0u) atomicMin(a.first_bad, j + bad);
    }
    // The last CTA to finish checks every range boundary in parallel, so the
    // in-order repair pass only starts where a guess was actually wrong.
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    unsigned long long bad = ~0ull;   // the warp-boundary ranges (j = 32, 64, ...) are left
    for (uint64_t j = 32 * (1 + static_cast<uint64_t>(threadIdx.x)); j < a.nranges; j += 32ull * blockDim.x)
        if (a.g[j] != a.e[j - 1]) {
            bad = j;
            break;
        }
    if (bad != ~0ull) atomicMin(a.first_bad, bad);
}

// Phase 2: one warp repairs the entry states in order; lane 0 walks, the warp
// scans for the next mismatch 32 ranges at a time.
template <typename E, bool CLS>
__global__ void __launch_bounds__(32) k_chunk_fix(const __grid_constant__ ChunkArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    load_table(sm, a.img, a.img_words);
    const uint32_t lane = threadIdx.x;
    const uint32_t per = a.chunk / kMid;
    unsigned long long repairs = 0;
    const unsigned long long fb = *a.first_bad;
    // ranges before the first wrong guess chain exactly (range 0 starts at the true start)
    uint32_t exact = a.nranges == 0 ? a.entry : (fb == ~0ull ? a.e[a.nranges - 1] : a.e[fb - 1]);
    for (uint64_t base = fb == ~0ull ? a.nranges : fb; base < a.nranges; base += 32) {
        // ranges base..base+31: find mismatches in order; after a repair the
        // exact exit may change, so re-scan from the repaired range.
        uint64_t j = base;
        while (j < a.nranges && j < base + 32) {
            const uint64_t jj = j + lane;
            const bool ok_lane = jj >= a.nranges || jj >= base + 32 ||
                                 (jj == j ? a.g[jj] == exact : a.g[jj] == a.e[jj - 1]);
            const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok_lane);
            if (!bad) {
                const uint64_t last = min(base + 32, a.nranges) - 1;
                exact = a.e[last];
                j = last + 1;
                break;
            }
            const uint64_t r = j + (__ffs(bad) - 1);
            const uint32_t entry = r == j ? exact : a.e[r - 1];
            // re-walk range r from its exact entry until it meets the recorded trajectory
            uint32_t s = entry;
            if (lane == 0) {
                const uint64_t c0 = r * a.chunk, c1 = min(c0 + a.chunk, a.len);
                uint32_t* mid = a.mid + r * per;
                uint32_t k = 0;
                for (uint64_t p = c0; p < c1; p += kMid, ++k) {
                    s = walk<E, CLS>(a, sm, s, p, min(p + kMid, c1));
                    if (s == mid[k]) {   // trajectories coincide from here on
                        s = a.e[r];
                        break;
                    }
                    mid[k] = s;
                }
                a.g[r] = entry;
                a.e[r] = s;
                ++repairs;
            }
            __syncwarp();
            exact = __shfl_sync(0xFFFFFFFFu, s, 0);
            j = r + 1;
        }
    }
    if (lane == 0) {
        *a.accept = static_cast<int32_t>(*reinterpret_cast<const E*>(sm + exact + a.acc_col));
        if (a.exit_state) *a.exit_state = exact;
        if (a.repairs) *a.repairs = repairs;
    }
}

template <typename E, bool CLS>
cudaError_t run(const DevTable& t, const ChunkArgs& a, int device, cudaStream_t st) {
    const uint32_t smem = t.img_bytes;
    cudaError_t e = cudaFuncSetAttribute(k_chunk_walk<E, CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_chunk_fix<E, CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chunk_walk<E, CLS>, 256, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * device_sm_count(device);
    const uint64_t want = (a.nranges + 255) / 256;
    const int grid = static_cast<int>(want < cap ? (want ? want : 1) : cap);
    k_chunk_walk<E, CLS><<<grid, 256, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_chunk_fix<E, CLS><<<1, 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

size_t chunked_scratch_bytes(uint64_t len, uint32_t chunk) {
    const uint64_t n = (len + chunk - 1) / chunk;
    return 16 + (2 * n + n * (chunk / kMid)) * sizeof(uint32_t) + 64;
}

uint32_t chunked_auto_chunk(const DevTable& t, uint64_t len, int device) {
    // about one range per resident thread (256-thread CTAs, occupancy by the table size)
    const uint64_t per_sm_threads = t.img_bytes > 100 * 1024 ? 256 : (t.img_bytes > 50 * 1024 ? 768 : 2048);
    const uint64_t ranges = per_sm_threads * static_cast<uint64_t>(device_sm_count(device));
    uint64_t c = (len + ranges - 1) / ranges;
    c = (c + kMid - 1) / kMid * kMid;
    if (c < 4 * kMid) c = 4 * kMid;
    return static_cast<uint32_t>(c);
}

cudaError_t launch_chunked(const DevTable& t, const uint8_t* text, uint64_t len, uint32_t chunk, uint32_t lookback,
                           void* scratch, int32_t* accept, unsigned long long* repairs, int device, cudaStream_t st,
                           uint32_t entry, uint32_t* exit_state) {
    ChunkArgs a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    a.lookback = lookback;
    a.nranges = (len + chunk - 1) / chunk;
    a.img = static_cast<const uint4*>(t.img);
    a.img_words = t.img_bytes / 16;
    a.cls_off = t.cls_off;
    a.start = t.start;
    a.entry = entry == kStartState ? t.start : entry;
    a.exit_state = exit_state;
    a.dead = t.dead;
    a.acc_col = t.ncols * static_cast<uint32_t>(t.esize);
    a.ticket = static_cast<unsigned int*>(scratch);
    a.first_bad = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(scratch) + 8);
    uint32_t* sc = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + 16);
    a.g = sc;
    a.e = sc + a.nranges;
    a.mid = sc + 2 * a.nranges;
    a.accept = accept;
    a.repairs = repairs;
    if (chunk == 0 || chunk % kMid) return cudaErrorInvalidValue;
    {
        cudaError_t e = write_u64(scratch, 0, st);   // ticket
        if (e == cudaSuccess) e = write_u64(static_cast<uint8_t*>(scratch) + 8, ~0ull, st);   // first_bad
        if (e != cudaSuccess) return e;
    }
    if (t.esize == 2) return t.cls ? run<uint16_t, true>(t, a, device, st) : run<uint16_t, false>(t, a, device, st);
    return t.cls ? run<uint32_t, true>(t, a, device, st) : run<uint32_t, false>(t, a, device, st);
}

}  // namespace rxg
