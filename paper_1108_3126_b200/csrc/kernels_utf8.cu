// UTF-8 validation of input buffers on the device, reproducing where
// rx::decode_utf8 (utf8.cpp:16-46) throws "invalid UTF-8 at byte N".
//
// decode_utf8 is sequential, but its first error position is a minimum of
// per-byte candidates that each thread can compute from a 7-byte window:
// before the first error every decoded sequence is lead + continuations and
// continuation bytes (10xxxxxx) are never leads, so
//   - a non-continuation byte i starts a sequence: it errs at i (bad lead
//     0x80-0xBF is impossible here; 0xF8-0xFF), at i (string ends inside the
//     sequence), at i+k (byte i+k is not a continuation), at i (overlong,
//     surrogate, > 0x10FFFF) or not at all;
//   - a continuation byte j errs at j iff no lead of the same string within
//     j-3..j-1 covers it (the nearest non-continuation byte L before j, if in
//     the string, covers j iff its sequence length exceeds j-L).
// No candidate lies before the true first error and the true one is a
// candidate, so the minimum is exact. Strings are decoded separately (the
// `rxvm match` getline loop, rxvm.cpp:100-112): the delimiter ends a string
// and a sequence running into it is truncated (error at its lead).
//
// Roofline: HBM read of the buffer once (16 B per thread per load, four
// loads in flight); all-ASCII 16-byte groups exit after one OR/AND test.
#include "launch.hpp"
#include "utf8.hpp"

namespace rxg {

namespace {

struct U8Args {
    const uint8_t* text;
    uint64_t len;
    int32_t delim;
    uint32_t stride;
    uint64_t base;
    unsigned long long* first_bad;
};

__device__ __forceinline__ bool is_cont(uint32_t b) { return (b & 0xC0u) == 0x80u; }

__device__ __forceinline__ uint32_t seq_len(uint32_t b) {
    if (b < 0x80u) return 1;
    if ((b & 0xE0u) == 0xC0u) return 2;
    if ((b & 0xF0u) == 0xE0u) return 3;
    if ((b & 0xF8u) == 0xF0u) return 4;
    return 0;   // 0x80-0xBF (continuation) or 0xF8-0xFF: not a lead
}

// First index >= i where the string containing i ends (exclusive end).
__device__ __forceinline__ uint64_t string_end(const U8Args& a, uint64_t i, uint32_t span) {
    uint64_t e = a.len;
    if (a.stride) e = min(e, (i / a.stride + 1) * a.stride);
    if (a.delim >= 0)
        for (uint32_t k = 1; k < span && i + k < e; ++k)
            if (a.text[i + k] == static_cast<uint8_t>(a.delim)) {
                e = i + k;
                break;
            }
    return e;
}

// Error position decode_utf8 would report for byte i (~0 = none), see above.
__device__ __noinline__ uint64_t candidate(const U8Args& a, uint64_t i) {
    const uint32_t b0 = a.text[i];
    if (b0 < 0x80u) return ~0ull;
    if (is_cont(b0)) {
        const uint64_t s0 = a.stride ? i - i % a.stride : 0;   // first byte of i's string (stride layout)
        for (uint32_t d = 1; d <= 3 && i >= d && i - d >= s0; ++d) {
            const uint32_t b = a.text[i - d];
            if (is_cont(b)) continue;
            if (a.delim >= 0 && b == static_cast<uint32_t>(a.delim)) return i;   // string starts after b
            return seq_len(b) > d ? ~0ull : i;
        }
        return i;   // no lead within reach
    }
    const uint32_t n = seq_len(b0);
    if (n == 0) return i;
    if (i + n > string_end(a, i, n)) return i;   // truncated
    uint32_t cp = b0 & (n == 2 ? 0x1Fu : (n == 3 ? 0x0Fu : 0x07u));
    for (uint32_t k = 1; k < n; ++k) {
        const uint32_t b = a.text[i + k];
        if (!is_cont(b)) return i + k;
        cp = (cp << 6) | (b & 0x3Fu);
    }
    const uint32_t lo = n == 2 ? 0x80u : (n == 3 ? 0x800u : 0x10000u);
    if (cp < lo || cp > 0x10FFFFu || (cp >= 0xD800u && cp <= 0xDFFFu)) return i;
    return ~0ull;
}

constexpr int kUnroll = 4;

// Top bit of each byte of x -> 4-bit mask (byte k -> bit k).
__device__ __forceinline__ uint32_t m4(uint32_t x) { return ((x & 0x80808080u) * 0x00204081u) >> 28; }

// Sufficient test that no byte of the 16-byte group at p is a candidate
// (exact on the cases it accepts; anything else goes to the per-byte rules).
// Window w = bytes [p-4, p+20), bit k of a mask = window byte k, the group
// is bits 4..19. Valid sequences <=> continuation bytes are exactly where a
// lead expects them (E), no F8-FF, no overlong / surrogate / > U+10FFFF lead
// pair, and (fixed stride) no expected continuation on a string start.
// A continuation in bits 20..22 that no group lead expects only forces the
// exact path; a lead in bits 1..3 is the previous group's: its errors are
// found there, and any miss it causes here lies after that error.
__device__ __forceinline__ bool group_ok(const U8Args& a, const uint32_t (&w)[6], uint64_t p) {
    uint32_t cont = 0, l2 = 0, l3 = 0, l4 = 0, bad = 0;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        const uint32_t x = w[j], s1 = x << 1, s2 = x << 2, s3 = x << 3, s4 = x << 4;
        const uint32_t c0 = x & s1, e0 = c0 & s2, f0 = e0 & s3, f8 = f0 & s4;
        cont |= m4(x & ~s1) << (4 * j);
        l2 |= m4(c0 & ~e0) << (4 * j);
        l3 |= m4(e0 & ~f0) << (4 * j);
        l4 |= m4(f0 & ~f8) << (4 * j);
        bad |= m4(f8) << (4 * j);
    }
    const uint32_t e = ((l2 | l3 | l4) << 1) | ((l3 | l4) << 2) | (l4 << 3);
    if (((cont ^ e) & 0x7FFFF0u) || (bad & 0xFFFF0u)) return false;
    uint32_t special = 0;
#pragma unroll
    for (int j = 1; j < 5; ++j) {
        const uint32_t x = w[j], y = __funnelshift_r(w[j], w[j + 1], 8);   // y byte k = byte after x byte k
        special |= __vcmpeq4(x & 0xFEFEFEFEu, 0xC0C0C0C0u);                               // C0 C1: overlong
        special |= __vcmpeq4(x, 0xE0E0E0E0u) & __vcmpltu4(y, 0xA0A0A0A0u);              // E0 80-9F: overlong
        special |= __vcmpeq4(x, 0xEDEDEDEDu) & __vcmpgeu4(y, 0xA0A0A0A0u);              // ED A0-BF: surrogate
        special |= __vcmpeq4(x, 0xF0F0F0F0u) & __vcmpltu4(y, 0x90909090u);              // F0 80-8F: overlong
        special |= (__vcmpeq4(x, 0xF4F4F4F4u) & __vcmpgeu4(y, 0x90909090u)) | __vcmpgtu4(x, 0xF4F4F4F4u);   // > U+10FFFF
    }
    if (special) return false;
    if (a.stride) {   // string starts in the window must not be expected continuations
        const uint64_t w0 = p - 4;
        uint32_t k = static_cast<uint32_t>((a.stride - w0 % a.stride) % a.stride), starts = 0;
        for (; k < 24; k += a.stride) starts |= 1u << k;
        if (e & starts & 0x7FFFF0u) return false;
    }
    return true;
}

__global__ void __launch_bounds__(256) k_utf8_check(const __grid_constant__ U8Args a) {
    // 16-byte groups from the first aligned address; head and tail bytes in thread 0
    const uint64_t head = min(a.len, static_cast<uint64_t>((16 - (reinterpret_cast<uintptr_t>(a.text) & 15)) & 15));
    const uint64_t groups = (a.len - head) / 16;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long best = ~0ull;
    const uint4* v16 = reinterpret_cast<const uint4*>(a.text + head);
    for (uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g0 < groups;
         g0 += nthreads * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t g = g0 + u * nthreads;
            v[u] = g < groups ? __ldcs(v16 + g) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (((v[u].x | v[u].y | v[u].z | v[u].w) & 0x80808080u) == 0) continue;
            const uint64_t p = head + (g0 + u * nthreads) * 16;
            if (p >= 4 && p + 20 <= a.len) {   // register window [p-4, p+20)
                const uint32_t w[6] = {*reinterpret_cast<const uint32_t*>(a.text + p - 4), v[u].x, v[u].y, v[u].z, v[u].w,
                                       *reinterpret_cast<const uint32_t*>(a.text + p + 16)};
                if (!group_ok(a, w, p))
                    for (uint64_t i = p; i < p + 16 && i < best; ++i)
                        best = min(best, static_cast<unsigned long long>(candidate(a, i)));
            } else {
                for (uint64_t i = p; i < p + 16 && i < best; ++i)
                    best = min(best, static_cast<unsigned long long>(candidate(a, i)));
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (uint64_t i = 0; i < head; ++i) best = min(best, static_cast<unsigned long long>(candidate(a, i)));
        for (uint64_t i = head + groups * 16; i < a.len; ++i) best = min(best, static_cast<unsigned long long>(candidate(a, i)));
    }
    if (best != ~0ull) atomicMin(a.first_bad, a.base + best);   // errors are rare: no warp reduction
}

}  // namespace

cudaError_t launch_utf8_check(const uint8_t* text, uint64_t len, int32_t delim, uint32_t stride, uint64_t base,
                              unsigned long long* first_bad, int device, cudaStream_t st) {
    if (len == 0) return cudaSuccess;
    U8Args a{text, len, delim, stride, base, first_bad};
    const uint64_t groups = len / 16 + 1;
    const uint64_t want = (groups + 256ull * kUnroll - 1) / (256ull * kUnroll);
    const uint64_t cap = static_cast<uint64_t>(device_sm_count(device)) * 8;
    const int grid = static_cast<int>(want < cap ? want : cap);
    k_utf8_check<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rxg
