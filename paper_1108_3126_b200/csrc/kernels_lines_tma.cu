// K2 (lines), TMA-staged: the memoized lockstep step over lines of one
// buffer, count of accepted lines and (RES) one result byte per line.
//
// Data path per warp: the warp owns 32 * K consecutive equal byte ranges
// ("rows" of a 2-D view [rows][chunk] of the input), K per lane. A TMA
// tensor map streams 32-byte column slices of those rows into a shared-memory
// ring (SWIZZLE_32B, so the per-lane 16-byte reads of 8 consecutive rows hit
// 8 distinct bank groups). One elected lane arms the stage mbarrier and
// issues the copy; all lanes wait on its phase. Shapes (warps x K x stages)
// per table layout are listed above launch_any; one CTA per SM.
//
// Step per input byte, direct layout (the memoized lockstep macro step, see
// tables.hpp and lines_tma_table.cpp):
//     a = IDP.4A(word, c<<8k, s)   extract byte k, scale by the column stride c, add the row
//     s = LDS.U16 [a]              s and the entries are absolute shared addresses
//     n += s >> 15 (LEA.HI)        START_A (the accepted-line-end row) is the only
//                                  row at >= 0x8000 the main loop can enter
// Class layouts (larger DFAs) index rows by state and columns by byte class
// (a class map) or by min(b ^ x, k) (range-clamped columns).
//
// Line ownership (every line matched exactly once): a range owns the lines
// starting in it after its first byte, plus the line starting right after
// it when its last byte is the delimiter; it enters in SKIP (range 0 in the
// start state) and finishes its last line through the tail copy of the
// table with direct global loads (finish_lines, range_direct).
//
// Per-line results (RES) in one pass: the byte loop is the count walk; each
// 4-byte word adds a has-zero delimiter mask, and per 32-byte stage column a
// chain with one line end records that line's result as the column's count
// difference (several: the column is walked again from its entry row). A
// range's owned results go out as range-local bits and a count, each warp
// tile's total as well; k_lt_scatter places them (one tile per warp, its
// base summed from the totals before it).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "options.hpp"
#include "launch.hpp"
#include "lines_tma.hpp"
#include "tma_common.cuh"

namespace rxg {

namespace {

constexpr int kMaxSlots = 128;

struct Args {
    const uint8_t* text;
    uint64_t len;
    uint64_t rows;         // full ranges covered by the tensor map
    uint64_t tiles;        // ceil(rows / rows per warp)
    uint32_t chunk;        // range width (multiple of the slice)
    uint32_t rem_piece;    // remainder [rows*chunk, len) split in pieces (direct loads)
    uint32_t rem_pieces;
    const uint4* img_lo;
    uint32_t lo_addr, lo_words;
    const uint4* img_hi;
    uint32_t hi_addr, hi_words;
    uint32_t bar_addr;
    uint32_t stage_addr[kMaxSlots];
    uint32_t start, skip, void_row, tail_delta, term_acc;
    uint32_t delim;
    uint32_t delim4, delim_hi4;                 // RES: the delimiter in every byte; its bit 7 in every byte
    uint32_t row_bytes, cmap_addr, acc_shift;   // class layouts
    uint32_t rows_addr, range_x, range_k;       // range-clamped columns
    uint32_t range_x4;                          // range_x in every byte (XOR a whole word)
    uint32_t acc_mul;                           // class layouts: 2^(32 - acc_shift) (count = hi32(s * acc_mul))
    uint32_t col_bytes;                         // direct layout: column stride
    unsigned long long* count;
    unsigned long long* slot;                   // CountSlot (launch.hpp)
    int accumulate;
    // per-line results (RES), in one pass: every range records the results of
    // the lines it owns as range-local bits plus its line count; a scan of
    // the counts and a scatter kernel place them (no delimiter pre-pass)
    uint32_t* rbits;                            // rwords words per range, transposed: word k of range r at k * nranges + r
    uint32_t rwords;
    uint64_t nranges;
    unsigned long long* rcount;                 // owned lines per range
    uint32_t* tsum;                             // owned lines per warp tile (+ one for the remainder pieces)
};

// Per-line results bookkeeping of one range (RES): the results of the lines
// it owns, in order, packed 32 to a word; own = whether the line the walk is
// in belongs to this range (it started inside it).
struct LineCursor {
    uint32_t lj;     // owned lines recorded so far
    uint32_t bits;   // the current word of results
    uint32_t* out;   // the range's next result word
    uint64_t stride; // words between a range's consecutive result words (the range count)
    bool own;
    bool live;       // false for lanes past the last range (they read zero fill)

    __device__ __forceinline__ void push(uint32_t v) {
        bits |= v << (lj & 31);
        if ((++lj & 31) == 0) {
            *out = bits;
            out += stride;
            bits = 0;
        }
    }
    __device__ __forceinline__ void close(unsigned long long* count) {
        if (lj & 31) *out = bits;
        *count = lj;
    }
};

__device__ __forceinline__ LineCursor cursor_of(const Args& a, uint64_t range, bool own, bool live) {
    return LineCursor{0u, 0u, a.rbits ? a.rbits + range : nullptr, a.nranges, own, live};
}

// Kernel shape: warps per CTA, ranges per lane, bytes per range per stage, ring depth.
template <int W, int K, int SL, int ST>
struct Shape {
    static constexpr int warps = W, chains = K, slice = SL, stages = ST, rows = 32 * K;
    static constexpr uint32_t stage_bytes = static_cast<uint32_t>(rows * SL);
    static_assert(W * ST <= kMaxSlots, "stage table too small");
};

__device__ __forceinline__ uint32_t tab(uint32_t addr) {
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// One memoized step on byte b. Direct layout: s is an absolute row address.
// Class layout: s is a row index, the class map gives the column address.
// Table layouts (template parameter L): 0 direct, 1 class (class-map LDS),
// 2 class rows with range-clamped columns (column = min(b ^ x, k), no LDS).
template <int L>
__device__ __forceinline__ uint32_t step_b(const Args& a, uint32_t s, uint32_t b) {
    if constexpr (L == 2) return tab(s * a.row_bytes + a.rows_addr + 2u * min(b ^ a.range_x, a.range_k));
    else if constexpr (L == 1) return tab(s * a.row_bytes + lds32(a.cmap_addr + b * 4u));
    else return tab(s + b * a.col_bytes);
}

template <int L, bool IDP = false>
__device__ __forceinline__ uint32_t step(const Args& a, uint32_t s, uint32_t word, int k) {
    if constexpr (IDP && L != 2) {
        // one IDP.4A.U8 extracts byte k, scales it by the column stride and adds the row
        // (replaces PRMT + IMAD; measured neutral on (c)/(d): the loop is shared-memory bound)
        if constexpr (L == 1) return tab(s * a.row_bytes + lds32(__dp4a(word, 4u << (8 * k), a.cmap_addr)));
        else return tab(__dp4a(word, a.col_bytes << (8 * k), s));
    }
    return step_b<L>(a, s, __byte_perm(word, 0, 0x4440 + k));
}

// Range layout step on byte k of a word already XORed with range_x in every
// byte: PRMT, IMNMX, IMAD, LDS.
__device__ __forceinline__ uint32_t step_rx(const Args& a, uint32_t s, uint32_t wx, int k) {
    return tab(s * a.row_bytes + a.rows_addr + 2u * min(__byte_perm(wx, 0, 0x4440 + k), a.range_k));
}

// 1 iff s is START_A (the accepted-line-end row).
template <int L>
__device__ __forceinline__ uint32_t counted(const Args& a, uint32_t s) {
    if constexpr (L != 0) return s >> a.acc_shift;   // (a shift: IMAD.HI by acc_mul measured slower on the FMA pipe)
    else return __umulhi(s, 1u << 17);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LTMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LTMA_WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

template <uint32_t BYTES>
__device__ __forceinline__ void tma_issue(const CUtensorMap* map, uint32_t dst, uint32_t bar, int32_t x, int32_t y) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "n"(BYTES) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// Physical 16-byte granule of logical granule g in row r of a stage: the
// TMA swizzle (none / 32B / 64B / 128B by slice width) XORs the granule
// index with row bits so 8 consecutive rows hit 8 distinct bank groups.
template <int SL>
__device__ __forceinline__ uint32_t granule(uint32_t r, uint32_t g) {
    if constexpr (SL == 16) return 0;
    else if constexpr (SL == 32) return g ^ ((r >> 2) & 1u);
    else if constexpr (SL == 64) return g ^ ((r >> 1) & 3u);
    else return g ^ (r & 7u);
}

// Finish the line straddling a range end with direct loads (tail copy rows).
template <int L>
__device__ uint32_t finish_line(const Args& a, uint32_t s, uint64_t pos) {
    while (pos < a.len) {
        if (pos + 16 <= a.len) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k) s = step<L>(a, s, word_of(v, w), k);
            pos += 16;
        } else {
            for (; pos < a.len; ++pos) s = step_b<L>(a, s, a.text[pos]);
        }
        if (s >= a.term_acc) return s;
    }
    return step_b<L>(a, s, a.delim);
}

// One byte of a RES walk: step, count, and at a delimiter record the line
// that just ended (if owned) and move to the next one.
template <int L>
__device__ __forceinline__ uint32_t step_res(const Args& a, uint32_t s, uint32_t b, uint32_t& cnt, LineCursor& lc) {
    s = step_b<L>(a, s, b);
    const uint32_t c = counted<L>(a, s);
    cnt += c;
    if (b == a.delim) {
        if (lc.own) lc.push(c);
        lc.own = lc.live;
    }
    return s;
}

// Walk [b0, b1) from s through the tail rows, stopping once a TERM row is
// reached; at the end of the buffer the virtual final delimiter is applied.
template <int L>
__device__ uint32_t walk_block(const Args& a, uint32_t s, uint64_t b0, uint64_t b1) {
    uint64_t p = b0;
    for (; p < b1 && s < a.term_acc; p += 16) {
        if (p + 16 <= b1 && !(p & 15)) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + p));
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k) s = step<L>(a, s, word_of(v, w), k);
        } else {
            for (uint64_t q = p; q < min(p + 16, b1); ++q) s = step_b<L>(a, s, a.text[q]);
        }
    }
    if (b1 == a.len && s < a.term_acc) s = step_b<L>(a, s, a.delim);
    return s;
}

// A long straddling line (one chain, warp-uniform s0 / p0), walked by the
// whole warp: each lane takes the next kCoopBlock bytes, guesses its entry state by
// walking the 64 bytes before its block from the start row, walks the block,
// and the guesses are checked in lane order against the exact exit of the
// lane before (a wrong one is re-walked from it). A delimiter inside a lookback
// means the line ended there, so the TERM row the guess reaches is then right.
constexpr uint32_t kCoopBlock = 1024;
constexpr uint64_t kCoopTail = 16384;   // bytes a chain walks alone before the warp takes over

template <int L>
__device__ uint32_t coop_walk(const Args& a, uint32_t s_true, uint64_t p0) {
    const uint32_t lane = threadIdx.x & 31;
    while (s_true < a.term_acc && p0 < a.len) {
        const uint64_t b0 = p0 + static_cast<uint64_t>(lane) * kCoopBlock;
        const uint64_t b1 = min(b0 + kCoopBlock, a.len);
        uint32_t g, e;
        if (b0 >= a.len) {
            g = e = a.term_acc;   // past the buffer: passes its entry through (fixed below)
        } else {
            g = lane == 0 ? s_true : walk_block<L>(a, a.start + a.tail_delta, b0 - 64, b0);
            e = walk_block<L>(a, g, b0, b1);
        }
        for (;;) {
            const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, e, 1);
            const bool ok = lane == 0 || g == up;
            const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok);
            if (!bad) break;
            const int m = __ffs(bad) - 1;
            const uint32_t ent = __shfl_sync(0xFFFFFFFFu, e, m - 1);   // exact: lanes < m agree
            if (ent >= a.term_acc) {   // the line ended before block m
                if (lane >= static_cast<uint32_t>(m)) g = e = ent;
                break;
            }
            if (lane == static_cast<uint32_t>(m)) {
                g = ent;
                e = b0 >= a.len ? ent : walk_block<L>(a, ent, b0, b1);
            }
        }
        s_true = __shfl_sync(0xFFFFFFFFu, e, 31);
        p0 += 32ull * kCoopBlock;
    }
    return s_true;
}

// The straddling lines of all of a lane's ranges, walked interleaved (their
// loads in flight together) instead of one after the other. s[j] enters as
// the tail-copy row; TERM rows absorb, so a finished chain keeps stepping
// harmlessly until the others are done. Returns per chain whether its line
// was accepted (live[j] false: no straddling line).
template <int L, int K>
__device__ void finish_lines(const Args& a, uint32_t (&s)[K], uint64_t (&pos)[K], const bool (&live)[K],
                             uint32_t (&ok)[K]) {
    bool more = false;
    uint64_t begin[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        more |= live[j];
        begin[j] = pos[j];
    }
    while (__any_sync(0xFFFFFFFFu, more)) {
        // 16 * U bytes per chain per round trip (lines end within a few dozen
        // bytes; measured better than 32 bytes on (c) despite a 16-byte spill)
        constexpr int U = 4;
        uint4 v[K][U];
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[j][u] = live[j] && s[j] < a.term_acc && pos[j] + 16 * (u + 1) <= a.len
                              ? __ldg(reinterpret_cast<const uint4*>(a.text + pos[j]) + u)
                              : make_uint4(0, 0, 0, 0);
        more = false;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (!live[j] || s[j] >= a.term_acc) continue;
            if (pos[j] + 16 * U <= a.len) {
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int w = 0; w < 4; ++w)
#pragma unroll
                        for (int k = 0; k < 4; ++k) s[j] = step<L>(a, s[j], word_of(v[j][u], w), k);
                pos[j] += 16 * U;
            } else if (pos[j] + 16 <= a.len) {
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k) s[j] = step<L>(a, s[j], word_of(v[j][0], w), k);
                pos[j] += 16;
            } else {   // the last bytes of the buffer, then the virtual delimiter
                for (; pos[j] < a.len; ++pos[j]) s[j] = step_b<L>(a, s[j], a.text[pos[j]]);
                if (s[j] < a.term_acc) s[j] = step_b<L>(a, s[j], a.delim);
            }
            more |= s[j] < a.term_acc;
        }
        bool long_tail = false;
#pragma unroll
        for (int j = 0; j < K; ++j) long_tail |= live[j] && s[j] < a.term_acc && pos[j] - begin[j] >= kCoopTail;
        if (__any_sync(0xFFFFFFFFu, long_tail)) break;
    }
    // lines still open after kCoopTail bytes: the whole warp walks them, one at a time
#pragma unroll
    for (int j = 0; j < K; ++j) {
        uint32_t need = __ballot_sync(0xFFFFFFFFu, live[j] && s[j] < a.term_acc);
        while (need) {
            const int src = __ffs(need) - 1;
            need &= need - 1;
            const uint32_t st = coop_walk<L>(a, __shfl_sync(0xFFFFFFFFu, s[j], src), __shfl_sync(0xFFFFFFFFu, pos[j], src));
            if (lane_id() == static_cast<uint32_t>(src)) s[j] = st;
        }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) ok[j] = live[j] && s[j] == a.term_acc;
}

// Line ownership. Every range but the first starts in SKIP (no read of the
// byte before it), so the line starting exactly at a range's first byte is
// skipped there; the previous range takes it instead: a range whose last
// byte is the delimiter walks the next line from the start state, exactly
// like a line straddling its end. Each line is matched by one range.
//
// A range processed entirely with direct loads (the remainder pieces).
template <int L, bool RES>
__device__ uint32_t range_direct(const Args& a, uint64_t c0, uint64_t c1, uint64_t range, uint32_t& cnt) {
    uint32_t s = c0 == 0 ? a.start : a.skip;
    LineCursor lc = cursor_of(a, range, s == a.start, true);
    uint32_t last = 0;
    uint64_t pos = c0;
    for (; pos + 16 <= c1; pos += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if constexpr (RES) {
                    s = step_res<L>(a, s, __byte_perm(word_of(v, w), 0, 0x4440 + k), cnt, lc);
                } else {
                    s = step<L>(a, s, word_of(v, w), k);
                    cnt += counted<L>(a, s);
                }
            }
        last = v.w >> 24;
    }
    for (; pos < c1; ++pos) {
        last = a.text[pos];
        if constexpr (RES) {
            s = step_res<L>(a, s, last, cnt, lc);
        } else {
            s = step_b<L>(a, s, last);
            cnt += counted<L>(a, s);
        }
    }
    const bool next_line = last == a.delim && c1 < a.len;
    if (next_line || (s != a.skip && last != a.delim)) {
        const uint32_t ok = finish_line<L>(a, (next_line ? a.start : s) + a.tail_delta, c1) == a.term_acc;
        cnt += ok;
        if constexpr (RES) lc.push(ok);
    }
    if constexpr (RES) lc.close(a.rcount + range);
    return RES ? lc.lj : 0u;   // owned lines (RES)
}

// RES: a stage column that holds several line ends, walked again from its
// entry row in byte order. Returns the owned lines' results (x, in order from
// bit 0), their number (y bits 0-7) and the ownership after the column (y bit
// 8); in registers, so the caller's LineCursor stays out of local memory.
template <class C, int L>
__device__ __noinline__ uint2 res_rewalk(const Args& a, uint32_t s, uint32_t stage, uint32_t r, bool own, bool live) {
    uint32_t bits = 0, n = 0;
    for (int g = 0; g < C::slice / 16; ++g) {
        const uint4 v = lds128(stage + r * C::slice + (granule<C::slice>(r, g) << 4));
        for (int w = 0; w < 4; ++w) {
            const uint32_t x = word_of(v, w);
            for (int k = 0; k < 4; ++k) {
                const uint32_t b = (x >> (8 * k)) & 0xFFu;
                s = step_b<L>(a, s, b);
                if (b == a.delim) {
                    if (own) bits |= counted<L>(a, s) << n++;
                    own = live;
                }
            }
        }
    }
    return make_uint2(bits, n | (own ? 256u : 0u));
}

template <class C, int L, bool RES>
__global__ void __launch_bounds__(C::warps * 32, 1) k_lines_tma(const __grid_constant__ Args a,
                                                             const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    if (base != kLtSmemBase) __trap();   // the table's absolute addresses assume this window
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * C::stages * 8;
    // the table images arrive by bulk copy (one request each, not a per-thread
    // load/store loop); the stage ring may live in the image's unused rows, so
    // no stage is filled before the images have landed
    const uint32_t tbar = a.bar_addr + C::warps * C::stages * 8;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
        mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tbar),
                     "r"((a.lo_words + a.hi_words) * 16u)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         a.lo_addr),
                     "l"(reinterpret_cast<uint64_t>(a.img_lo)), "r"(a.lo_words * 16u), "r"(tbar)
                     : "memory");
        if (a.hi_words)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             a.hi_addr),
                         "l"(reinterpret_cast<uint64_t>(a.img_hi)), "r"(a.hi_words * 16u), "r"(tbar)
                         : "memory");
    }
    if (lane == 0) {
        for (int st = 0; st < C::stages; ++st) mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();   // barrier initialisation visible to every thread
    // class layouts may put ring stages in the image's unused rows: no stage
    // is filled before the image has landed. The direct layout's ring lies
    // outside the image, so its first stages are requested before the wait
    // (the table copy and the first data round trip overlap).
    if constexpr (L != 0) mbar_wait(tbar, 0);

    uint32_t cnt = 0;
    if (blockIdx.x == 0 && warp == 0 && a.rem_pieces) {
        mbar_wait(tbar, 0);
        const uint64_t r0 = a.rows * a.chunk;
        uint32_t own = 0;
        for (uint32_t p = lane; p < a.rem_pieces; p += 32) {
            const uint64_t c0 = r0 + static_cast<uint64_t>(p) * a.rem_piece;
            own += range_direct<L, RES>(a, c0, min(c0 + a.rem_piece, a.len), a.rows + p, cnt);
        }
        if constexpr (RES) {   // the remainder pieces are the scatter's last unit
            own = __reduce_add_sync(0xFFFFFFFFu, own);
            if (lane == 0) a.tsum[a.tiles] = own;
        }
    }
    if constexpr (RES) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && !a.rem_pieces) a.tsum[a.tiles] = 0;
    }

    uint32_t phase = 0;   // bit st = parity of stage st's next completion
    const uint32_t ncol = a.chunk / C::slice;
    const uint32_t* stage = a.stage_addr + warp * C::stages;
    // tiles interleave the CTAs (tile = warp * grid + cta): small inputs spread over every SM
    for (uint64_t tile = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x; tile < a.tiles;
         tile += static_cast<uint64_t>(gridDim.x) * C::warps) {
        const uint64_t row0 = tile * C::rows;
        if (lane == 0) {
            const uint32_t pro = ncol < C::stages ? ncol : C::stages;
            for (uint32_t st = 0; st < pro; ++st)
                tma_issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>(st * C::slice),
                                          static_cast<int32_t>(row0));
        }
        if constexpr (L == 0) mbar_wait(tbar, 0);
        uint32_t s[C::chains];
        bool valid[C::chains];
        LineCursor lc[C::chains];
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            const uint64_t row = row0 + j * 32 + lane;
            valid[j] = row < a.rows;
            s[j] = a.void_row;
            if (valid[j]) s[j] = row == 0 ? a.start : a.skip;   // see the ownership note above range_direct
            lc[j] = cursor_of(a, RES && valid[j] ? row : 0, valid[j] && s[j] == a.start, valid[j]);
        }
        uint32_t last[C::chains] = {};
        // RES: accepted line ends per chain; a 32-byte column holding one line
        // end gives that line's result as the difference across the column
        uint32_t cj[C::chains];
#pragma unroll
        for (int j = 0; j < C::chains; ++j) cj[j] = 0;
        for (uint32_t col = 0; col < ncol; ++col) {
            const uint32_t st = col % C::stages;
            mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
            phase ^= 1u << st;
            // RES: per chain, the column's delimiters as one bit each (byte 4w+k of
            // the column at bit 8k+w: the order does not matter, only the count)
            uint32_t dl[C::chains], s_in[C::chains], c_in[C::chains];
#pragma unroll
            for (int j = 0; j < C::chains; ++j) {
                dl[j] = 0;
                s_in[j] = s[j];
                c_in[j] = cj[j];
            }
#pragma unroll
            for (int g = 0; g < C::slice / 16; ++g) {
                uint4 v[C::chains];
#pragma unroll
                for (int j = 0; j < C::chains; ++j) {
                    const uint32_t r = j * 32 + lane;
                    v[j] = lds128(stage[st] + r * C::slice + (granule<C::slice>(r, g) << 4));
                }
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    uint32_t wx[C::chains];   // range layout: the word XORed once, not each byte
#pragma unroll
                    for (int j = 0; j < C::chains; ++j) wx[j] = L == 2 ? word_of(v[j], w) ^ a.range_x4 : 0u;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < C::chains; ++j) {
                            s[j] = L == 2 ? step_rx(a, s[j], wx[j], k) : step<L, true>(a, s[j], word_of(v[j], w), k);
                            if constexpr (RES) cj[j] += counted<L>(a, s[j]);
                            else cnt += counted<L>(a, s[j]);
                        }
                    if constexpr (RES) {
#pragma unroll
                        for (int j = 0; j < C::chains; ++j) {
                            // bit 7 of each byte: byte == delimiter, by the has-zero test on
                            // x ^ delim (3 ops). A borrow can flag extra bytes, but only in a word
                            // that holds a delimiter: a column with one line end never reads as
                            // none or as one, only as several (the exact re-walk below)
                            const uint32_t u = word_of(v[j], w) ^ a.delim4;
                            const uint32_t z = (u - 0x01010101u) & ~u & 0x80808080u;
                            dl[j] |= z >> (7 - (4 * (g & 1) + w));
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < C::chains; ++j) last[j] = v[j].w >> 24;
            }
            if constexpr (RES) {
                static_assert(C::slice == 32, "RES records one 32-byte column at a time");
#pragma unroll
                for (int j = 0; j < C::chains; ++j) {
                    const uint32_t nd = __popc(dl[j]);
                    if (nd == 1) {
                        if (lc[j].own) lc[j].push(cj[j] - c_in[j]);
                        lc[j].own = lc[j].live;
                    } else if (nd > 1) {   // several line ends: walk the column again, in byte order
                        const uint2 rw = res_rewalk<C, L>(a, s_in[j], stage[st], j * 32 + lane, lc[j].own, lc[j].live);
                        for (uint32_t i = 0; i < (rw.y & 0xFFu); ++i) lc[j].push((rw.x >> i) & 1u);
                        lc[j].own = (rw.y >> 8) & 1u;
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && col + C::stages < ncol) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>((col + C::stages) * C::slice),
                                          static_cast<int32_t>(row0));
            }
        }
        if constexpr (RES) {
#pragma unroll
            for (int j = 0; j < C::chains; ++j) cnt += cj[j];
        }
        {
            bool live[C::chains];
            uint64_t pos[C::chains];
            uint32_t ok[C::chains];
#pragma unroll
            for (int j = 0; j < C::chains; ++j) {
                pos[j] = (row0 + j * 32 + lane + 1) * a.chunk;
                const bool next_line = last[j] == a.delim && pos[j] < a.len;   // the line starting right after
                live[j] = valid[j] && (next_line || (s[j] != a.skip && last[j] != a.delim));
                s[j] = (next_line ? a.start : s[j]) + a.tail_delta;
            }
            finish_lines<L, C::chains>(a, s, pos, live, ok);
#pragma unroll
            for (int j = 0; j < C::chains; ++j) {
                cnt += ok[j];
                if constexpr (RES) {
                    if (live[j]) lc[j].push(ok[j]);
                    if (valid[j]) lc[j].close(a.rcount + row0 + j * 32 + lane);
                }
            }
            if constexpr (RES) {   // the tile's owned lines: the scatter places tiles from these
                uint32_t own = 0;
#pragma unroll
                for (int j = 0; j < C::chains; ++j) own += valid[j] ? lc[j].lj : 0u;
                own = __reduce_add_sync(0xFFFFFFFFu, own);
                if (lane == 0) a.tsum[tile] = own;
            }
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    tma::publish_count(a.slot, a.count, a.accumulate != 0, cnt, a.bar_addr + C::warps * C::stages * 8 + 8);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Stage slots: first the gap below the main rows, then after the upper rows.
template <class C>
uint32_t place_stages(const LtTable& t, Args& a) {
    int k = 0;
    // free space inside the table image: below the main rows (direct layout)
    // or the unused rows below START_A (class layout)
    const uint32_t lo = t.cls ? align_up(t.hole_lo, 1024) : kLtSmemBase;
    const uint32_t hi = t.cls ? t.hole_hi : t.lo_addr;
    for (uint32_t p = lo; p + C::stage_bytes <= hi && k < C::warps * C::stages; p += C::stage_bytes)
        a.stage_addr[k++] = p;
    uint32_t p = align_up(t.cls ? t.smem_table_end : kLtAccAddr + t.hi_bytes, 1024);
    for (; k < C::warps * C::stages; ++k, p += C::stage_bytes) a.stage_addr[k] = p;
    a.bar_addr = align_up(p, 8);
    return a.bar_addr + C::warps * C::stages * 8 + 8 + 4 * C::warps - kLtSmemBase;   // ring barriers, table barrier, warp sums
}

CUtensorMapSwizzle swizzle_of(int slice) {
    switch (slice) {
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
    }
}

// Per-line results (RES), second pass, one launch: a warp takes one walk
// tile (its R consecutive ranges; the last unit is the remainder pieces).
// The tile's first line is the sum of the owned-line totals of the tiles
// before it: each block sums the totals before its first tile (a few
// thousand u32 values, cached), each warp adds those of the block's earlier
// tiles. Within the tile, 32 ranges at a time: lane j holds range j's count
// and first two result words (coalesced: the words are transposed), a warp
// scan gives the ranges' offsets, and the warp writes each range's bytes,
// up to 32 consecutive bytes per store. (A decoupled look-back over all
// ranges measured slower: ~9.5k warps start together and look back far.)
__global__ void __launch_bounds__(256) k_lt_scatter(const uint32_t* __restrict__ rbits,
                                                    const unsigned long long* __restrict__ count,
                                                    const uint32_t* __restrict__ tsum, uint64_t nunits, uint32_t R,
                                                    uint64_t rows, uint64_t nranges, uint8_t* __restrict__ results) {
    __shared__ unsigned long long part[8];
    __shared__ uint32_t wbits[8][66];   // per warp: a group's results as bits (32 ranges x <= 64 lines, + slack)
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t u0 = static_cast<uint64_t>(blockIdx.x) * 8;
    unsigned long long acc = 0;
    for (uint64_t i = threadIdx.x; i < u0; i += blockDim.x) acc += tsum[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    const uint64_t u = u0 + warp;
    if (u >= nunits) return;
    unsigned long long prefix = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) prefix += part[w];
    prefix += __reduce_add_sync(0xFFFFFFFFu, lane < warp ? tsum[u0 + lane] : 0u);
    const bool pieces = u + 1 == nunits;
    const uint64_t rb = pieces ? rows : u * R;
    const uint64_t re = pieces ? nranges : min(rb + R, rows);
    uint8_t* out = results + prefix;
    uint32_t run = 0;   // lines of this tile placed so far
    uint32_t* bitbuf = wbits[warp];
    for (uint64_t r0 = rb; r0 < re; r0 += 32) {
        const uint64_t r = r0 + lane;
        const bool in = r < re;
        const uint32_t n = in ? static_cast<uint32_t>(count[r]) : 0u;
        const uint32_t w0 = n ? __ldg(rbits + r) : 0u, w1 = n > 32 ? __ldg(rbits + nranges + r) : 0u;
        uint32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t rel = incl - n;   // within this group of 32 ranges
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        uint8_t* gout = out + run;
        run += total;
        if (total == 0) continue;
        if (!__any_sync(0xFFFFFFFFu, n > 64)) {
            // the group's results as one bit array (at most 32 * 64 bits), then
            // 16 bytes per lane store: 16 bits spread to bytes, aligned 16-byte
            // stores inside, byte stores in the partial chunks at the edges
            bitbuf[lane] = 0u;
            bitbuf[lane + 32] = 0u;
            if (lane < 2) bitbuf[lane + 64] = 0u;
            __syncwarp();
            if (n) {
                const uint32_t k = rel >> 5, sh = rel & 31u;
                atomicOr(bitbuf + k, w0 << sh);
                if (sh) atomicOr(bitbuf + k + 1, w0 >> (32 - sh));
                if (n > 32) {
                    atomicOr(bitbuf + k + 1, w1 << sh);
                    if (sh) atomicOr(bitbuf + k + 2, w1 >> (32 - sh));
                }
            }
            __syncwarp();
            const uintptr_t g0 = reinterpret_cast<uintptr_t>(gout), ga = g0 & ~uintptr_t(15);
            const uint32_t nchunks = static_cast<uint32_t>((g0 + total - ga + 15) >> 4);
            for (uint32_t c = lane; c < nchunks; c += 32) {
                const uintptr_t cb = ga + 16u * c;   // chunk start (global address)
                const int32_t b0 = static_cast<int32_t>(static_cast<intptr_t>(cb) - static_cast<intptr_t>(g0));   // bit of its first byte
                if (b0 >= 0 && b0 + 16 <= static_cast<int32_t>(total)) {
                    const uint32_t bw = static_cast<uint32_t>(b0) >> 5, bs = static_cast<uint32_t>(b0) & 31u;
                    const uint32_t lo = bitbuf[bw], hi = bs + 16 > 32 ? bitbuf[bw + 1] : 0u;
                    const uint32_t bits16 = __funnelshift_r(lo, hi, bs) & 0xFFFFu;
                    uint4 v;
                    v.x = ((bits16 & 0xFu) * 0x00204081u) & 0x01010101u;
                    v.y = (((bits16 >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
                    v.z = (((bits16 >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
                    v.w = (((bits16 >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
                    *reinterpret_cast<uint4*>(cb) = v;
                } else {   // a partial chunk: only this group's bytes
                    for (int32_t i = 0; i < 16; ++i) {
                        const int32_t bi = b0 + i;
                        if (bi < 0 || bi >= static_cast<int32_t>(total)) continue;
                        reinterpret_cast<uint8_t*>(cb)[i] = static_cast<uint8_t>((bitbuf[bi >> 5] >> (bi & 31)) & 1u);
                    }
                }
            }
            __syncwarp();
            continue;
        }
        // ranges with more than 64 lines (short lines): each range's bytes in turn
#pragma unroll 4
        for (uint32_t j = 0; j < 32; ++j) {
            const uint32_t nj = __shfl_sync(0xFFFFFFFFu, n, j);
            if (nj == 0) continue;
            const uint32_t bj = __shfl_sync(0xFFFFFFFFu, rel, j);
            const uint32_t x0 = __shfl_sync(0xFFFFFFFFu, w0, j);
            if (lane < nj) gout[bj + lane] = static_cast<uint8_t>((x0 >> lane) & 1u);
            if (nj > 32) {
                const uint32_t x1 = __shfl_sync(0xFFFFFFFFu, w1, j);
                for (uint32_t i = 32 + lane; i < nj; i += 32) {
                    const uint32_t w = i < 64 ? x1 : __ldg(rbits + (i >> 5) * nranges + r0 + j);
                    gout[bj + i] = static_cast<uint8_t>((w >> (i & 31)) & 1u);
                }
            }
        }
    }
}

template <class C, int L, bool RES>
int per_sm_of(uint32_t smem) {
    int per_sm = 0;
    auto* k = k_lines_tma<C, L, RES>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::warps * 32, smem);
    return per_sm < 1 ? 1 : per_sm;
}

template <class C, int L>
uint32_t auto_chunk(const LtTable& t, uint64_t len) {
    Args a{};
    const uint32_t smem = place_stages<C>(t, a);
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t rows = static_cast<uint64_t>(per_sm_of<C, L, false>(smem)) * device_sm_count(dev) * C::warps * C::rows;
    uint64_t c = (len + rows - 1) / rows;
    c = (c + C::slice - 1) / C::slice * C::slice;
    // Small inputs (a strong-scaled shard): one wave of ranges makes them so
    // short that each range's fixed costs (entry, straddling-line tail) rule;
    // up to 2 KB, half a wave of twice-as-long ranges is faster. Measured on
    // config (c) shards, direct layout (tools/chunk_sweep.py): 1/8 of the job
    // 384 -> 768 B per range 54.3 -> 48.1 us, 1/4 768 -> 1536 B 76.8 -> 70.7
    // us, 1/2 and the whole job unchanged.
    if (L == 0) c = std::max<uint64_t>(c, std::min<uint64_t>(2048, 2 * c));
    if (c < 4u * C::slice) c = 4u * C::slice;
    if (c > (1u << 20)) c = 1u << 20;
    return static_cast<uint32_t>(c);
}

// Ranges of a launch: full TMA rows plus the remainder pieces.
struct RangeSplit {
    uint64_t rows;
    uint32_t rem_piece, rem_pieces;
};

RangeSplit split_ranges(uint64_t len, uint32_t chunk) {
    RangeSplit r{};
    r.rows = len / chunk;
    const uint64_t rem = len - r.rows * chunk;
    r.rem_piece = static_cast<uint32_t>(((rem + 31) / 32 + 15) & ~uint64_t(15));
    if (r.rem_piece < 16) r.rem_piece = 16;
    r.rem_pieces = rem ? static_cast<uint32_t>((rem + r.rem_piece - 1) / r.rem_piece) : 0;
    return r;
}

// RES scratch: [counts | bases | scan temp | result bits (rwords per range, transposed)].
uint32_t res_words(uint32_t chunk, uint32_t rem_piece) {
    return ((chunk > rem_piece ? chunk : rem_piece) + 1 + 31) / 32;
}

// RES scratch: [owned lines per range (u64) | per-tile totals (u32; tiles <= ranges / 32,
// + the remainder unit) | result bits (rwords per range, transposed)].
size_t res_tsum_bytes(uint64_t nranges) { return ((nranges / 32 + 2) * sizeof(uint32_t) + 255) & ~size_t(255); }

size_t res_scratch_bytes(uint64_t nranges, uint32_t rwords) {
    return nranges * sizeof(unsigned long long) + res_tsum_bytes(nranges) + nranges * rwords * 4ull + 256;
}

template <class C, int L, bool RES>
cudaError_t launch(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                   unsigned long long* count, uint8_t* results, void* scratch, size_t scratch_bytes,
                   CountSlot cs, cudaStream_t st) {
    if (len == 0) {   // nothing to launch: the count is 0 (or unchanged when accumulating)
        return cs.accumulate ? cudaSuccess : cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    }
    if (chunk == 0) chunk = auto_chunk<C, L>(t, len);
    if (chunk % C::slice) return cudaErrorInvalidValue;
    Args a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    const RangeSplit rs = split_ranges(len, chunk);
    a.rows = rs.rows;
    a.tiles = (a.rows + C::rows - 1) / C::rows;
    a.rem_piece = rs.rem_piece;
    a.rem_pieces = rs.rem_pieces;
    const uint64_t nr = rs.rows + rs.rem_pieces;
    if constexpr (RES) {
        a.rwords = res_words(chunk, rs.rem_piece);
        a.nranges = nr;
        if (!scratch || scratch_bytes < res_scratch_bytes(nr, a.rwords)) return cudaErrorInvalidValue;
        a.rcount = static_cast<unsigned long long*>(scratch);
        a.tsum = reinterpret_cast<uint32_t*>(a.rcount + nr);
        a.rbits = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(a.tsum) + res_tsum_bytes(nr));
    }
    a.img_lo = static_cast<const uint4*>(t.d_lo);
    a.lo_addr = t.lo_addr;
    a.lo_words = t.lo_bytes / 16;
    a.img_hi = static_cast<const uint4*>(t.d_hi);
    a.hi_addr = t.hi_addr;
    a.hi_words = t.hi_bytes / 16;
    const uint32_t smem = place_stages<C>(t, a);
    a.start = t.start;
    a.skip = t.skip;
    a.void_row = t.void_row;
    a.tail_delta = t.tail_delta;
    a.term_acc = t.term_acc;
    a.delim = delim;
    a.delim4 = delim * 0x01010101u;
    a.delim_hi4 = a.delim4 & 0x80808080u;
    a.row_bytes = t.row_bytes;
    a.cmap_addr = t.cmap_addr;
    a.acc_shift = t.acc_shift;
    a.col_bytes = t.col_bytes;
    a.rows_addr = kLtSmemBase + 1024;
    a.range_x = t.range_x;
    a.range_k = t.range_k;
    a.range_x4 = t.range_x * 0x01010101u;
    a.acc_mul = t.cls ? 1u << (32 - t.acc_shift) : 0u;
    a.count = count;
    a.slot = cs.p;
    a.accumulate = cs.accumulate ? 1 : 0;

    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (a.rows > 0) {
        auto enc = encode_fn();
        if (!enc) return cudaErrorNotSupported;
        const cuuint64_t dims[2] = {chunk, a.rows};
        const cuuint64_t strides[1] = {chunk};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(C::slice), static_cast<cuuint32_t>(C::rows)};
        const cuuint32_t estr[2] = {1, 1};
        CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        if (const char* e = rxg::option("RXG_TMA_PROMO")) {   // tuning override
            const int v = std::atoi(e);
            promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                    : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                    : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        }
        const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(text), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(C::slice), promo,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    const int per_sm = per_sm_of<C, L, RES>(smem);
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = static_cast<uint64_t>(per_sm) * device_sm_count(dev);
    const uint64_t want = a.tiles;   // at most one tile per CTA needed to reach every SM
    const int grid = static_cast<int>(want == 0 ? 1 : (want < cap ? want : cap));
    k_lines_tma<C, L, RES><<<grid, C::warps * 32, smem, st>>>(a, map);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !RES) return e;
    // per-line results: place each tile's owned lines (tile totals summed in the scatter)
    const uint64_t nunits = a.tiles + 1;
    k_lt_scatter<<<static_cast<unsigned>((nunits + 7) / 8), 256, 0, st>>>(a.rbits, a.rcount, a.tsum, nunits,
                                                                          static_cast<uint32_t>(C::rows), a.rows, nr,
                                                                          results);
    return cudaGetLastError();
}

// Kernel shapes (RXG_LT_SHAPE=0 forces S0 for tuning runs; unset = per-layout default).
// Measured on config (c), 1 GB, B200 (tools/ab_lines.py): 16-byte slices are
// TMA-request bound (~3.3 TB/s); 32-byte slices with 24 warps x 2 ranges x 3
// stages reach ~5.05 TB/s, x 3 ranges x 2 stages ~5.1-5.25 TB/s (direct layout);
// 24x4x2, 32x3x2 and 16x4x3 measured 4.77-5.0 TB/s with the paired rows;
// the class layout uses SC (below).
using S0 = Shape<24, 2, 32, 3>;
using S6 = Shape<24, 3, 32, 2>;
// class layout (two LDS per byte, random rows): fewer warps and a deeper ring,
// (d) 1,761 GB/s vs 1,681 for S0 (16x2x5 1,737, 12x2x6 1,724, 20x2x4 1,697,
// 16x3x2 1,676, 24x2x2 1,683, 32x2x2 1,603)
using SC = Shape<16, 2, 32, 4>;
// range-clamped class rows: larger rows, a shallower ring so table + ring fit
// ((d) 2,130 GB/s; 12x2x4 2,066, 16x3x2 2,026, 24x2x2 2,059)
using SR = Shape<16, 2, 32, 3>;

int shape_id() {
    const char* e = rxg::option("RXG_LT_SHAPE");
    return e ? std::atoi(e) : -1;
}

template <bool RES>
cudaError_t launch_any(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                       unsigned long long* count, uint8_t* results, void* scratch, size_t scratch_bytes,
                       CountSlot cs, cudaStream_t st) {
    if (t.cls && t.range_k)
        return launch<SR, 2, RES>(t, text, len, delim, chunk, count, results, scratch, scratch_bytes, cs, st);
    if (t.cls) return launch<SC, 1, RES>(t, text, len, delim, chunk, count, results, scratch, scratch_bytes, cs, st);
    if (shape_id() == 0)
        return launch<S0, 0, RES>(t, text, len, delim, chunk, count, results, scratch, scratch_bytes, cs, st);
    return launch<S6, 0, RES>(t, text, len, delim, chunk, count, results, scratch, scratch_bytes, cs, st);
}

}  // namespace

cudaError_t launch_lines_tma(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                             unsigned long long* count, CountSlot cs, cudaStream_t st) {
    return launch_any<false>(t, text, len, delim, chunk, count, nullptr, nullptr, 0, cs, st);
}

uint32_t lines_tma_chunk(const LtTable& t, uint64_t len, uint32_t chunk) {
    if (chunk) return chunk;
    if (t.cls && t.range_k) return auto_chunk<SR, 2>(t, len);
    if (t.cls) return auto_chunk<SC, 1>(t, len);
    if (shape_id() == 0) return auto_chunk<S0, 0>(t, len);
    return auto_chunk<S6, 0>(t, len);
}

size_t lines_tma_results_scratch(uint64_t len, uint32_t chunk) {
    const RangeSplit rs = split_ranges(len, chunk);
    return res_scratch_bytes(rs.rows + rs.rem_pieces, res_words(chunk, rs.rem_piece));
}

cudaError_t launch_lines_tma_results(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim,
                                     uint32_t chunk, unsigned long long* count, uint8_t* results, void* scratch,
                                     size_t scratch_bytes, CountSlot cs, cudaStream_t st) {
    return launch_any<true>(t, text, len, delim, chunk, count, results, scratch, scratch_bytes, cs, st);
}

uint32_t lines_tma_slice() { return 32; }

}  // namespace rxg
