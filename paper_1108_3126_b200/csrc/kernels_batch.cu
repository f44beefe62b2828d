// K2 — batched lockstep over many strings.
//
// Each thread advances K independent "chains". A chain is a fixed byte
// range of the input (delimited mode) or one string (fixed-stride mode). The
// memoized lockstep step lives in shared memory (tables.hpp): one LDS per
// input byte moves a string from E_i to E_{i+1}, i.e. one reference macro
// step step_char(evolve(S), a) (proj/src/lockstep.cpp:77-80).
//
// Delimited mode ownership rule: a chain owns the lines that START inside
// its range. It enters its range in SKIP state unless the previous byte is a
// delimiter, swallows the foreign line tail, and at its range end finishes
// its last line by walking the "tail copy" of the table, whose delimiter
// column drops into absorbing TERM rows. Every line is therefore matched by
// exactly one chain, and every input byte is read by the chain that owns it
// plus (for line tails) the one before it.
#include <cub/device/device_scan.cuh>

#include "launch.hpp"

namespace rxg {

namespace {

constexpr int kBlock = 256;

struct LinesArgs {
    const uint8_t* text;
    uint64_t len;
    uint64_t nchunks;
    uint32_t chunk;
    uint32_t img_words;   // 16-byte words of the table image
    const uint4* img;
    uint32_t cls_off;
    uint32_t start, skip, acc_shift, tail_delta, term_acc;
    uint32_t delim;
    unsigned long long* count;
    uint8_t* results;
    const unsigned long long* line_base;
};

struct FixedArgs {
    const uint8_t* text;
    uint64_t n;
    uint32_t stride;
    uint32_t img_words;
    const uint4* img;
    uint32_t cls_off;
    uint32_t start;
    uint32_t acc_col;   // byte offset of the accept column inside a row
    unsigned long long* count;
    uint8_t* results;
};

__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// One memoized lockstep step: row offset s, input byte b -> next row offset.
template <typename E, bool CLS>
__device__ __forceinline__ uint32_t step(const uint8_t* sm, uint32_t cls_off, uint32_t s, uint32_t b) {
    const uint32_t col = CLS ? static_cast<uint32_t>(sm[cls_off + b]) : b;
    return *reinterpret_cast<const E*>(sm + s + col * static_cast<uint32_t>(sizeof(E)));
}

__device__ __forceinline__ void load_table(uint8_t* sm, const uint4* img, uint32_t words) {
    uint4* dst = reinterpret_cast<uint4*>(sm);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = img[i];
    __syncthreads();
}

// Finish the line that straddles a chain's range end: walk the tail copy of
// the table from `pos` (16-aligned) until the first delimiter parks the
// string in a TERM row, or the buffer ends (then feed a virtual delimiter,
// the std::getline rule for a final unterminated line).
template <typename E, bool CLS>
__device__ uint32_t finish_line(const LinesArgs& a, const uint8_t* sm, uint32_t s, uint64_t pos) {
    while (pos < a.len) {
        if (pos + 16 <= a.len) {
            const uint4 v = ldg16(a.text + pos);
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k) s = step<E, CLS>(sm, a.cls_off, s, (word_of(v, w) >> (8 * k)) & 0xFFu);
            pos += 16;
        } else {
            for (; pos < a.len; ++pos) s = step<E, CLS>(sm, a.cls_off, s, a.text[pos]);
        }
        if (s >= a.term_acc) return s;
    }
    return step<E, CLS>(sm, a.cls_off, s, a.delim);
}

template <typename E, bool CLS, bool RES>
__device__ void chain_slow(const LinesArgs& a, const uint8_t* sm, uint64_t c, uint32_t& cnt) {
    const uint64_t c0 = c * a.chunk;
    const uint64_t c1 = min(c0 + a.chunk, a.len);
    uint32_t s = (c0 == 0 || a.text[c0 - 1] == a.delim) ? a.start : a.skip;
    unsigned long long line = RES ? a.line_base[c] : 0ull;
    uint32_t last = 0;
    for (uint64_t pos = c0; pos < c1; ++pos) {
        const uint32_t b = a.text[pos];
        const uint32_t prev = s;
        s = step<E, CLS>(sm, a.cls_off, s, b);
        if (RES) {
            if (b == a.delim) {
                if (prev != a.skip) a.results[line] = static_cast<uint8_t>(s >> a.acc_shift);
                ++line;
            }
        }
        cnt += s >> a.acc_shift;
        last = b;
    }
    if (s != a.skip && last != a.delim) {
        s = finish_line<E, CLS>(a, sm, s + a.tail_delta, c1);
        const uint32_t ok = s == a.term_acc;
        if (RES) a.results[line] = static_cast<uint8_t>(ok);
        cnt += ok;
    }
}

template <typename E, bool CLS, int K, bool RES>
__global__ void __launch_bounds__(kBlock) k_lines(const __grid_constant__ LinesArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    load_table(sm, a.img, a.img_words);
    uint32_t cnt = 0;
    const uint64_t groups = (a.nchunks + K - 1) / K;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += nthreads) {
        const uint64_t first = g * K;
        if ((first + K) * a.chunk > a.len) {
            for (int j = 0; j < K; ++j)
                if (first + j < a.nchunks) chain_slow<E, CLS, RES>(a, sm, first + j, cnt);
            continue;
        }
        const uint8_t* base = a.text + first * a.chunk;
        uint32_t s[K];
        unsigned long long line[K];
        uint4 cur[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint64_t c0 = (first + j) * a.chunk;
            s[j] = (c0 == 0 || a.text[c0 - 1] == a.delim) ? a.start : a.skip;
            line[j] = RES ? a.line_base[first + j] : 0ull;
            cur[j] = ldg16(base + static_cast<uint64_t>(j) * a.chunk);
        }
        const uint32_t nblk = a.chunk / 16;
        for (uint32_t i = 0; i < nblk; ++i) {
            uint4 nxt[K];
            if (i + 1 < nblk) {
#pragma unroll
                for (int j = 0; j < K; ++j) nxt[j] = ldg16(base + static_cast<uint64_t>(j) * a.chunk + (i + 1) * 16u);
            }
#pragma unroll
            for (int w = 0; w < 4; ++w) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const uint32_t b = (word_of(cur[j], w) >> (8 * k)) & 0xFFu;
                        const uint32_t prev = s[j];
                        s[j] = step<E, CLS>(sm, a.cls_off, prev, b);
                        if (RES) {
                            if (b == a.delim) {
                                if (prev != a.skip) a.results[line[j]] = static_cast<uint8_t>(s[j] >> a.acc_shift);
                                ++line[j];
                            }
                        }
                        cnt += s[j] >> a.acc_shift;
                    }
                }
            }
            if (i + 1 < nblk) {
#pragma unroll
                for (int j = 0; j < K; ++j) cur[j] = nxt[j];
            }
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint32_t last = cur[j].w >> 24;
            if (s[j] != a.skip && last != a.delim) {
                const uint32_t t = finish_line<E, CLS>(a, sm, s[j] + a.tail_delta, (first + j + 1) * a.chunk);
                const uint32_t ok = t == a.term_acc;
                if (RES) a.results[line[j]] = static_cast<uint8_t>(ok);
                cnt += ok;
            }
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.count, static_cast<unsigned long long>(cnt));
}

// Delimiters per chunk (results mode: global line index of each chunk's first line).
__global__ void __launch_bounds__(kBlock) k_count_delims(const uint8_t* __restrict__ text, uint64_t len,
                                                          uint32_t chunk, uint64_t nchunks, uint32_t delim,
                                                          unsigned long long* __restrict__ out) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint64_t c0 = c * chunk, c1 = min(c0 + chunk, len);
    const uint32_t d4 = delim * 0x01010101u;
    uint32_t n = 0;
    uint64_t pos = c0;
    for (; pos + 16 <= c1; pos += 16) {
        const uint4 v = ldg16(text + pos);
        n += __popc(__vcmpeq4(v.x, d4)) + __popc(__vcmpeq4(v.y, d4)) + __popc(__vcmpeq4(v.z, d4)) +
             __popc(__vcmpeq4(v.w, d4));
    }
    n /= 8;
    for (; pos < c1; ++pos) n += text[pos] == delim;
    out[c] = n;
}

// Fixed-stride strings: few large CTAs (one table copy per SM, not per 256
// threads: the table can be as large as a small input), 4 strings per thread.
constexpr int kFixedBlock = 1024;
constexpr int kFixedChains = 4;

template <typename E, bool CLS, int K, bool RES>
__global__ void __launch_bounds__(kFixedBlock) k_fixed(const __grid_constant__ FixedArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    load_table(sm, a.img, a.img_words);
    uint32_t cnt = 0;
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool vec = (a.stride % 16u) == 0;
    for (uint64_t base = 0; base < a.n; base += T * K) {
        uint32_t s[K];
        bool live[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            live[j] = base + j * T + tid < a.n;
            s[j] = a.start;
        }
        if (vec) {
            const uint32_t nblk = a.stride / 16;
            uint32_t i = 0;
            // two 16-byte blocks of every string in flight before the dependent walk
            for (; i + 2 <= nblk; i += 2) {
                uint4 v[K][2];
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (live[j]) {
                        const uint8_t* p = a.text + (base + j * T + tid) * a.stride + i * 16u;
                        v[j][0] = ldg16(p);
                        v[j][1] = ldg16(p + 16);
                    }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int w = 0; w < 4; ++w)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
#pragma unroll
                            for (int j = 0; j < K; ++j)
                                if (live[j]) s[j] = step<E, CLS>(sm, a.cls_off, s[j], (word_of(v[j][h], w) >> (8 * k)) & 0xFFu);
            }
            for (; i < nblk; ++i) {
                uint4 v[K];
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (live[j]) v[j] = ldg16(a.text + (base + j * T + tid) * a.stride + i * 16u);
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            if (live[j]) s[j] = step<E, CLS>(sm, a.cls_off, s[j], (word_of(v[j], w) >> (8 * k)) & 0xFFu);
            }
        } else {
            for (uint32_t i = 0; i < a.stride; ++i)
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (live[j]) s[j] = step<E, CLS>(sm, a.cls_off, s[j], a.text[(base + j * T + tid) * a.stride + i]);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (!live[j]) continue;
            const uint32_t ok = *reinterpret_cast<const E*>(sm + s[j] + a.acc_col);
            if (RES) a.results[base + j * T + tid] = static_cast<uint8_t>(ok);
            cnt += ok;
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.count, static_cast<unsigned long long>(cnt));
}

template <typename Kern>
int grid_for(Kern kern, uint32_t smem, uint64_t work_threads, int device) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * static_cast<uint64_t>(device_sm_count(device));
    const uint64_t want = (work_threads + kBlock - 1) / kBlock;
    return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

template <typename E, bool CLS, int K, bool RES>
cudaError_t run_lines(const DevTable& t, const LinesArgs& a, cudaStream_t st) {
    auto kern = k_lines<E, CLS, K, RES>;
    const uint32_t smem = t.img_bytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    const int grid = grid_for(kern, smem, (a.nchunks + K - 1) / K, dev);
    kern<<<grid, kBlock, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename E, bool CLS, int K, bool RES>
cudaError_t run_fixed(const DevTable& t, const FixedArgs& a, cudaStream_t st) {
    auto kern = k_fixed<E, CLS, K, RES>;
    const uint32_t smem = t.img_bytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFixedBlock, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * device_sm_count(dev);
    const uint64_t want = (a.n + static_cast<uint64_t>(kFixedBlock) * K - 1) / (static_cast<uint64_t>(kFixedBlock) * K);
    const int grid = static_cast<int>(want < cap ? (want ? want : 1) : cap);
    kern<<<grid, kFixedBlock, smem, st>>>(a);
    return cudaGetLastError();
}

constexpr int kChains = 2;

template <bool RES>
cudaError_t dispatch_lines(const DevTable& t, const LinesArgs& a, cudaStream_t st) {
    if (t.esize == 2) {
        return t.cls ? run_lines<uint16_t, true, kChains, RES>(t, a, st) : run_lines<uint16_t, false, kChains, RES>(t, a, st);
    }
    return t.cls ? run_lines<uint32_t, true, kChains, RES>(t, a, st) : run_lines<uint32_t, false, kChains, RES>(t, a, st);
}

template <bool RES>
cudaError_t dispatch_fixed(const DevTable& t, const FixedArgs& a, cudaStream_t st) {
    constexpr int K = kFixedChains;
    if (t.esize == 2) {
        return t.cls ? run_fixed<uint16_t, true, K, RES>(t, a, st) : run_fixed<uint16_t, false, K, RES>(t, a, st);
    }
    return t.cls ? run_fixed<uint32_t, true, K, RES>(t, a, st) : run_fixed<uint32_t, false, K, RES>(t, a, st);
}

template <typename E, bool CLS>
int lines_per_sm(uint32_t smem) {
    int per_sm = 0;
    cudaFuncSetAttribute(k_lines<E, CLS, kChains, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lines<E, CLS, kChains, false>, kBlock, smem);
    return per_sm < 1 ? 1 : per_sm;
}

}  // namespace

uint32_t lines_auto_chunk(const DevTable& t, uint64_t len) {
    int per_sm;
    if (t.esize == 2) per_sm = t.cls ? lines_per_sm<uint16_t, true>(t.img_bytes) : lines_per_sm<uint16_t, false>(t.img_bytes);
    else per_sm = t.cls ? lines_per_sm<uint32_t, true>(t.img_bytes) : lines_per_sm<uint32_t, false>(t.img_bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    // One wave: every resident chain gets one equal byte range, so line tails
    // and SKIP prefixes stay a small fraction of a range.
    const uint64_t chains = static_cast<uint64_t>(per_sm) * device_sm_count(dev) * kBlock * kChains;
    uint64_t c = (len + chains - 1) / chains;
    c = (c + 15) & ~uint64_t(15);
    if (c < 256) c = 256;
    if (c > (1u << 20)) c = 1u << 20;
    return static_cast<uint32_t>(c);
}

cudaError_t write_u64(void* dst, uint64_t value, cudaStream_t st) {
    // (cuStreamWriteValue64 measured slower than the memset kernel on B200:
    // config (b) 21.5 vs 18.5 us per step)
    if (value != 0 && value != ~0ull) return cudaErrorInvalidValue;
    return cudaMemsetAsync(dst, value ? 0xFF : 0, sizeof(uint64_t), st);
}

int device_sm_count(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cached[device] = n > 0 ? n : 148;
    }
    return cached[device];
}

size_t lines_scratch_bytes(uint64_t len, uint32_t chunk) {
    const uint64_t nchunks = (len + chunk - 1) / chunk;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<int64_t>(nchunks));
    return 2 * nchunks * sizeof(unsigned long long) + temp + 256;
}

cudaError_t launch_lines(const DevTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                         unsigned long long* count, uint8_t* results, unsigned long long* scratch,
                         size_t scratch_bytes, cudaStream_t st, LaunchStats* ls) {
    if (ls) ls->kernels = 0;
    if (len == 0) return cudaSuccess;
    LinesArgs a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    a.nchunks = (len + chunk - 1) / chunk;
    a.img = static_cast<const uint4*>(t.img);
    a.img_words = t.img_bytes / 16;
    a.cls_off = t.cls_off;
    a.start = t.start;
    a.skip = t.skip;
    a.acc_shift = t.acc_shift;
    a.tail_delta = t.tail_delta;
    a.term_acc = t.term_acc;
    a.delim = delim;
    a.count = count;
    if (!results) {
        if (ls) ls->kernels = 1;
        return dispatch_lines<false>(t, a, st);
    }
    if (!scratch || scratch_bytes < lines_scratch_bytes(len, chunk)) return cudaErrorInvalidValue;
    unsigned long long* per_chunk = scratch;
    unsigned long long* base = scratch + a.nchunks;
    void* temp = reinterpret_cast<uint8_t*>(base + a.nchunks);
    size_t temp_bytes = scratch_bytes - 2 * a.nchunks * sizeof(unsigned long long);
    const unsigned blocks = static_cast<unsigned>((a.nchunks + kBlock - 1) / kBlock);
    k_count_delims<<<blocks, kBlock, 0, st>>>(text, len, chunk, a.nchunks, delim, per_chunk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, per_chunk, base, static_cast<int64_t>(a.nchunks), st);
    if (e != cudaSuccess) return e;
    a.results = results;
    a.line_base = base;
    if (ls) ls->kernels = 3;
    return dispatch_lines<true>(t, a, st);
}

cudaError_t launch_fixed(const DevTable& t, const uint8_t* text, uint64_t n, uint32_t stride,
                         unsigned long long* count, uint8_t* results, cudaStream_t st, LaunchStats* ls) {
    if (ls) ls->kernels = 0;
    if (n == 0) return cudaSuccess;
    FixedArgs a{};
    a.text = text;
    a.n = n;
    a.stride = stride;
    a.img = static_cast<const uint4*>(t.img);
    a.img_words = t.img_bytes / 16;
    a.cls_off = t.cls_off;
    a.start = t.start;
    a.acc_col = t.ncols * static_cast<uint32_t>(t.esize);
    a.count = count;
    a.results = results;
    if (ls) ls->kernels = 1;
    return results ? dispatch_fixed<true>(t, a, st) : dispatch_fixed<false>(t, a, st);
}

}  // namespace rxg

// ── fixed stride, absolute-address variant ─────────────────────────────────
//
// Same walk as k_fixed, for raw-byte u16 tables (DFA <= ~120 states) whose
// entries were rebased to absolute shared addresses (+0x400) on the host:
// per byte PRMT + IMAD + LDS, no predication (lanes past the end walk string
// 0 and are not counted), 4 strings per thread, both 16-byte blocks of a
// 32-byte string loaded before the walk.
namespace rxg {

namespace {

constexpr uint32_t kAbsBase = 0x400;

struct FixedAbsArgs {
    const uint8_t* text;
    uint64_t n;
    uint32_t stride;   // multiple of 16
    uint32_t img_words;
    const uint4* img;
    uint32_t start;    // absolute
    uint32_t acc_col;  // byte offset of the accept column
    unsigned long long* count;
    uint8_t* results;
};

__device__ __forceinline__ uint32_t tab16(uint32_t addr) {
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

template <int K, bool RES>
__global__ void __launch_bounds__(1024) k_fixed_abs(const __grid_constant__ FixedAbsArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kAbsBase) __trap();
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    // warp slots interleave the CTAs (a warp's 32 strings stay consecutive, so its
    // loads coalesce): the partial last pass spreads over every SM, not the first few
    const uint64_t tid = (static_cast<uint64_t>(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31);
    const uint32_t nblk = a.stride / 16;
    // first 32 bytes of the K strings of a pass (lanes past the end read string 0)
    auto fetch = [&](uint64_t base, uint4 (&v)[K][2]) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint64_t idx = base + j * T + tid;
            const uint8_t* p = a.text + (idx < a.n ? idx : 0) * a.stride;
            v[j][0] = __ldg(reinterpret_cast<const uint4*>(p));
            v[j][1] = nblk > 1 ? __ldg(reinterpret_cast<const uint4*>(p + 16)) : make_uint4(0, 0, 0, 0);
        }
    };
    // the first pass's input is in flight while the table is copied in
    uint4 nxt[K][2];
    fetch(0, nxt);
    for (uint32_t i = threadIdx.x; i < a.img_words; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = a.img[i];
    __syncthreads();
    uint32_t cnt = 0;
    auto walk = [&](uint32_t (&s)[K], const uint4 (&v)[K][2], int halves) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h >= halves) break;
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const uint32_t word = w == 0 ? v[j][h].x : (w == 1 ? v[j][h].y : (w == 2 ? v[j][h].z : v[j][h].w));
                        s[j] = tab16(__dp4a(word, 2u << (8 * k), s[j]));   // s + 2 * byte k
                    }
        }
    };
    for (uint64_t base = 0; base < a.n; base += T * K) {
        uint4 cur[K][2];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            cur[j][0] = nxt[j][0];
            cur[j][1] = nxt[j][1];
        }
        if (base + T * K < a.n) fetch(base + T * K, nxt);   // next pass in flight during this one
        uint32_t s[K];
#pragma unroll
        for (int j = 0; j < K; ++j) s[j] = a.start;
        walk(s, cur, nblk > 1 ? 2 : 1);
        for (uint32_t i = 2; i < nblk; i += 2) {   // strings longer than 32 bytes
            uint4 v[K][2];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const uint64_t idx = base + j * T + tid;
                const uint8_t* p = a.text + (idx < a.n ? idx : 0) * a.stride + i * 16u;
                v[j][0] = __ldg(reinterpret_cast<const uint4*>(p));
                v[j][1] = i + 1 < nblk ? __ldg(reinterpret_cast<const uint4*>(p + 16)) : make_uint4(0, 0, 0, 0);
            }
            walk(s, v, i + 1 < nblk ? 2 : 1);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint64_t idx = base + j * T + tid;
            if (idx >= a.n) continue;
            const uint32_t ok = tab16(s[j] + a.acc_col);
            if (RES) a.results[idx] = static_cast<uint8_t>(ok);
            cnt += ok;
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.count, static_cast<unsigned long long>(cnt));
}

template <int K, bool RES>
cudaError_t run_fixed_abs(const FixedAbsArgs& a, uint32_t smem, cudaStream_t st) {
    auto kern = k_fixed_abs<K, RES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1024, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * device_sm_count(dev);
    const uint64_t want = (a.n + 1024ull * K - 1) / (1024ull * K);
    const int grid = static_cast<int>(want < cap ? (want ? want : 1) : cap);
    kern<<<grid, 1024, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fixed_abs(const DevTable& t, const uint8_t* text, uint64_t n, uint32_t stride,
                             unsigned long long* count, uint8_t* results, cudaStream_t st, LaunchStats* ls) {
    if (ls) ls->kernels = 0;
    if (n == 0) return cudaSuccess;
    if (t.cls || t.esize != 2 || stride % 16) return cudaErrorInvalidValue;
    FixedAbsArgs a{};
    a.text = text;
    a.n = n;
    a.stride = stride;
    a.img = static_cast<const uint4*>(t.img);
    a.img_words = t.img_bytes / 16;
    a.start = t.start + kAbsBase;
    a.acc_col = t.ncols * 2u;
    a.count = count;
    a.results = results;
    if (ls) ls->kernels = 1;
    return results ? run_fixed_abs<2, true>(a, t.img_bytes, st) : run_fixed_abs<2, false>(a, t.img_bytes, st);
}

}  // namespace rxg
