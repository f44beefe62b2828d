// K2b: the bitset lockstep step (SURVEY.md §8(a) "verified restatement",
// north_star (2) second bullet) over batches of strings, on K2's TMA data
// path (kernels_lines_tma.cu): every lane owns byte ranges ("rows" of a 2-D
// [rows][chunk] view of the input), a TMA tensor map streams 32-byte column
// slices of a warp's rows through a 3-stage shared-memory ring, and the
// line-ownership rules are K2's: a range enters its first (partial) line in
// SKIP — here the empty set, which never accepts — and finishes the line
// straddling its end with direct loads.
//
// State: the position set E, WT 32-bit words in the lane's registers
// (positions in the heap's left-to-right order; the accept bit A moved to bit
// 31 of the last word). Per input byte b:
//     f      = E & M[b]                                   (positions that match b)
//     E'     = shift1(f & SH) | OR{ R[g] : f & T[g] != 0 }  (one-bit successors of
//              consecutive literals, then the deduplicated residual follow rows)
//     line end (b == delimiter, or the last byte of a fixed-stride string):
//              count += A in E;  E = E0
// M is a 256-row table in shared memory (random rows across lanes); SH, E0,
// the first 4 trigger / residual rows live in registers for WT <= 4 and are
// read as shared-memory broadcasts otherwise; further groups loop over
// shared memory. This is the engine for patterns whose memoized step (DFA)
// exceeds its cap; it is exact for every pattern whose position set fits
// 16 words (511 positions).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>

#include "bits.hpp"
#include "tma_common.cuh"

namespace rxg {

// ── host tables ───────────────────────────────────────────────────────────

BitsTables make_bits_tables(const Program& p, int32_t delim) {
    BitsTables t;
    const int32_t Wsrc = p.W;
    int32_t wt = (p.n_pos + 1 + 31) / 32;   // A gets bit 32*wt - 1 (>= n_pos)
    int32_t WT = 1;
    while (WT < wt) WT *= 2;
    if (WT > kBitsMaxWords) return t;   // too many positions for a lane's registers
    t.WT = WT;
    const int32_t A = WT * 32 - 1;
    auto remap = [&](const uint32_t* src, uint32_t* dst) {   // source bitset (A = n_pos) -> kernel bitset
        for (int32_t q = 0; q < p.n_pos; ++q)
            if ((src[q >> 5] >> (q & 31)) & 1u) dst[q >> 5] |= 1u << (q & 31);
        if ((src[p.n_pos >> 5] >> (p.n_pos & 31)) & 1u) dst[A >> 5] |= 1u << (A & 31);
    };
    // follow rows F'(q) in the kernel bit order
    std::vector<uint32_t> fol(static_cast<size_t>(p.n_pos) * WT, 0u);
    for (int32_t q = 0; q < p.n_pos; ++q) remap(&p.follow[static_cast<size_t>(q) * Wsrc], &fol[static_cast<size_t>(q) * WT]);
    // shift + deduplicated residual rows (as build_bitset_plan): a row owned by
    // one position that holds q+1 (a real position, never A) is split
    std::unordered_map<std::string, int32_t> users, ids;
    auto key = [&](const uint32_t* r) { return std::string(reinterpret_cast<const char*>(r), WT * 4); };
    for (int32_t q = 0; q < p.n_pos; ++q) ++users[key(&fol[static_cast<size_t>(q) * WT])];
    std::vector<uint32_t> SH(WT, 0u), rows, trig;
    std::vector<uint32_t> resid(WT);
    for (int32_t q = 0; q < p.n_pos; ++q) {
        const uint32_t* row = &fol[static_cast<size_t>(q) * WT];
        std::copy(row, row + WT, resid.begin());
        const int32_t nb = q + 1;
        if (nb < p.n_pos && users[key(row)] == 1 && ((row[nb >> 5] >> (nb & 31)) & 1u)) {
            SH[q >> 5] |= 1u << (q & 31);
            resid[nb >> 5] &= ~(1u << (nb & 31));
        }
        bool any = false;
        for (uint32_t x : resid) any |= x != 0;
        if (!any) continue;
        auto it = ids.find(key(resid.data()));
        if (it == ids.end()) {
            it = ids.emplace(key(resid.data()), t.G++).first;
            rows.insert(rows.end(), resid.begin(), resid.end());
            trig.insert(trig.end(), WT, 0u);
        }
        trig[static_cast<size_t>(it->second) * WT + (q >> 5)] |= 1u << (q & 31);
    }
    t.GR = 2;
    std::vector<uint32_t> E0(WT, 0u);
    remap(p.init.data(), E0.data());
    std::vector<uint32_t> M(static_cast<size_t>(256) * WT, 0u);
    for (int b = 0; b < 256; ++b) {
        const int32_t c = p.byte_class[b];
        if (c && b != delim) remap(&p.class_mask[static_cast<size_t>(c) * Wsrc], &M[static_cast<size_t>(b) * WT]);
        M[static_cast<size_t>(b) * WT + (A >> 5)] &= ~(1u << (A & 31));   // A matches no byte
    }
    auto tg = [&](int32_t g, int32_t w) { return g < t.G ? trig[static_cast<size_t>(g) * WT + w] : 0u; };
    auto rg = [&](int32_t g, int32_t w) { return g < t.G ? rows[static_cast<size_t>(g) * WT + w] : 0u; };
    std::vector<uint32_t>& img = t.img;
    if (WT <= 4) {
        // per byte: [M, D (1 on the delimiter, else 0), pad]; then T_g, R_g of the
        // groups >= 2 (broadcast rows); registers: SH, E0, T_0, R_0, T_1, R_1
        t.row_words = WT == 1 ? 2 : (WT + 1 + 3) / 4 * 4;
        img.assign(static_cast<size_t>(256) * t.row_words, 0u);
        for (int b = 0; b < 256; ++b) {
            uint32_t* r = &img[static_cast<size_t>(b) * t.row_words];
            for (int32_t w = 0; w < WT; ++w) r[w] = M[static_cast<size_t>(b) * WT + w];
            r[WT] = b == delim ? 1u : 0u;
        }
        t.xg_off = static_cast<uint32_t>(img.size()) * 4;
        for (int32_t g = 2; g < t.G; ++g) {
            for (int32_t w = 0; w < WT; ++w) img.push_back(tg(g, w));
            for (int32_t w = 0; w < WT; ++w) img.push_back(rg(g, w));
        }
        t.regs.insert(t.regs.end(), SH.begin(), SH.end());
        t.regs.insert(t.regs.end(), E0.begin(), E0.end());
        for (int32_t g = 0; g < 2; ++g) {
            for (int32_t w = 0; w < WT; ++w) t.regs.push_back(tg(g, w));
            for (int32_t w = 0; w < WT; ++w) t.regs.push_back(rg(g, w));
        }
    } else {
        // per byte: [M, D, pad 3] (the 4-word pad skews rows across banks);
        // broadcast rows SH, E0, then (T_g, R_g) for every group
        t.row_words = WT + 4;
        img.assign(static_cast<size_t>(256) * t.row_words, 0u);
        for (int b = 0; b < 256; ++b) {
            uint32_t* r = &img[static_cast<size_t>(b) * t.row_words];
            for (int32_t w = 0; w < WT; ++w) r[w] = M[static_cast<size_t>(b) * WT + w];
            r[WT] = b == delim ? 1u : 0u;
        }
        t.xg_off = static_cast<uint32_t>(img.size()) * 4;
        img.insert(img.end(), SH.begin(), SH.end());
        img.insert(img.end(), E0.begin(), E0.end());
        for (int32_t g = 0; g < std::max(t.G, 2); ++g) {
            for (int32_t w = 0; w < WT; ++w) img.push_back(tg(g, w));
            for (int32_t w = 0; w < WT; ++w) img.push_back(rg(g, w));
        }
    }
    if (t.regs.empty()) t.regs.push_back(0u);
    while (img.size() % 4) img.push_back(0u);
    t.ok = img.size() * 4 <= kBitsMaxTableBytes;
    return t;
}

namespace {

constexpr int kMaxSlots = 128;

struct BArgs {
    const uint8_t* text;
    uint64_t len;
    uint64_t rows;         // full ranges covered by the tensor map
    uint64_t tiles;
    uint32_t chunk;
    uint32_t rem_piece, rem_pieces;   // lines: remainder [rows*chunk, len) in pieces (direct loads)
    uint32_t stride;                  // fixed-stride strings (0: lines)
    uint32_t delim4;                  // delimiter in every byte
    int32_t n_groups;
    uint32_t two;         // the constant 2 (a register operand keeps IMAD on the FMA pipe)
    const uint4* img;
    uint32_t img_words;   // 16-byte units
    uint32_t tab;         // shared address of M
    uint32_t cmap;        // shared address of the byte -> class map (extra groups, WT <= 4)
    uint32_t xt;          // shared address of the extra groups' per-class M & T_g rows (WT <= 4)
    uint32_t xt_row_bytes;
    uint32_t xg;          // shared address of the extra R_g rows (WT <= 4) / the broadcast rows (WT > 4)
    const uint32_t* regs_g;   // the same rows in global memory (WT <= 4: loaded into registers)
    uint32_t bar_addr;
    uint32_t stage_addr[kMaxSlots];
    unsigned long long* count;
    unsigned long long* slot;
    int accumulate;
    uint8_t* results;                        // per string 0/1, or null
    const unsigned long long* line_base;     // lines + results: delimiters before each range
};

template <int W, int K, int SL, int ST>
struct Shape {
    static constexpr int warps = W, chains = K, slice = SL, stages = ST, rows = 32 * K;
    static constexpr uint32_t stage_bytes = static_cast<uint32_t>(rows * SL);
};

// Loop-invariant rows: E0 and R_0, R_1 in registers (REG, WT <= 4), or the
// broadcast area of shared memory (SH, E0, then T_g, R_g per group).
template <int WT, int GR, bool REG>
struct Rows {
    uint32_t sh[REG ? WT : 1], e0[REG ? WT : 1], tr[REG ? 2 : 1][REG ? WT : 1], rr[REG ? 2 : 1][REG ? WT : 1];
    uint32_t base;   // !REG: shared address of the broadcast rows

    __device__ void load(const BArgs& a) {
        if constexpr (REG) {
            const uint32_t* g = a.regs_g;
#pragma unroll
            for (int w = 0; w < WT; ++w) {
                sh[w] = __ldg(g + w);
                e0[w] = __ldg(g + WT + w);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    tr[k][w] = __ldg(g + 2 * WT + 2 * k * WT + w);
                    rr[k][w] = __ldg(g + 3 * WT + 2 * k * WT + w);
                }
            }
        } else {
            base = a.xg;
        }
    }
    // words 4*w4 .. 4*w4+3 of broadcast row r (0 SH, 1 E0, 2+2g T_g, 3+2g R_g)
    __device__ __forceinline__ void get4(int r, int w4, uint32_t (&out)[4]) const {
        const uint4 v = tma::lds128(base + (r * WT + w4 * 4) * 4);
        out[0] = v.x;
        out[1] = v.y;
        out[2] = v.z;
        out[3] = v.w;
    }
};

template <int N>
__device__ __forceinline__ void load_words(uint32_t addr, uint32_t (&m)[N]) {
    if constexpr (N == 1) {
        m[0] = tma::lds32(addr);
    } else if constexpr (N == 2) {
        uint32_t x, y;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
        m[0] = x;
        m[1] = y;
    } else {
        static_assert(N % 4 == 0, "rows are loaded 16 bytes at a time");
#pragma unroll
        for (int w = 0; w < N; w += 4) {
            const uint4 v = tma::lds128(addr + 4 * w);
            m[w] = v.x;
            m[w + 1] = v.y;
            m[w + 2] = v.z;
            m[w + 3] = v.w;
        }
    }
}

// Row width in words (BitsTables::row_words).
template <int WT>
__host__ __device__ constexpr int row_words() {
    return WT == 1 ? 2 : WT <= 4 ? (WT + 1 + 3) / 4 * 4 : WT + 4;
}

// The REG step on a row already loaded (rows of several bytes are loaded
// ahead: they depend on the input only, not on E).
template <int WT, int GR, bool REG, bool XG>
__device__ __forceinline__ void bstep_row(const BArgs& a, const Rows<WT, GR, REG>& R, uint32_t (&E)[WT],
                                          const uint32_t (&row)[row_words<WT>()], uint32_t row_addr, uint32_t cm,
                                          uint32_t& m, uint32_t& cnt) {

    uint32_t nx[WT];
    {
        // shift part: E & M & SH moved up one position (one 3-input LOP3 per word)
        uint32_t prev = 0;
#pragma unroll
        for (int w = 0; w < WT; ++w) {
            const uint32_t sh = E[w] & row[w] & R.sh[w];
            // (a register 2, not a literal: keeps the shift an IMAD on the FMA pipe)
            nx[w] = WT == 1 ? sh * a.two : __funnelshift_l(prev, sh, 1);
            prev = sh;
        }
        // the two register groups: any E & M & T_g fires R_g
        uint32_t acc0 = 0, acc1 = 0;
#pragma unroll
        for (int w = 0; w < WT; ++w) {
            acc0 |= E[w] & row[w] & R.tr[0][w];
            acc1 |= E[w] & row[w] & R.tr[1][w];
        }
        if constexpr (WT == 1) {
            // predicated ORs (2 ALU ops) instead of SEL, SEL, OR3 (3)
            asm("{\n\t.reg .pred p0, p1;\n\t"
                "setp.ne.u32 p0, %1, 0;\n\t"
                "setp.ne.u32 p1, %2, 0;\n\t"
                "@p0 or.b32 %0, %0, %3;\n\t"
                "@p1 or.b32 %0, %0, %4;\n\t}"
                : "+r"(nx[0])
                : "r"(acc0), "r"(acc1), "r"(R.rr[0][0]), "r"(R.rr[1][0]));
        } else {
#pragma unroll
            for (int w = 0; w < WT; ++w) {
                if (acc0) nx[w] |= R.rr[0][w];
                if (acc1) nx[w] |= R.rr[1][w];
            }
        }
        if constexpr (XG) {   // groups >= 2: T_g, R_g broadcast rows
            (void)row_addr;
            for (int g = 2; g < a.n_groups; ++g) {
                const uint32_t tb = a.xg + static_cast<uint32_t>(g - 2) * 2u * WT * 4u;
                uint32_t acc = 0;
#pragma unroll
                for (int w = 0; w < WT; ++w) acc |= E[w] & row[w] & tma::lds32(tb + w * 4u);
                if (acc) {
#pragma unroll
                    for (int w = 0; w < WT; ++w) nx[w] |= tma::lds32(tb + (WT + w) * 4u);
                }
            }
        }
    }
    // String end without a select: D is 1 on the delimiter (else 0) and the
    // delimiter's M row is empty, so nx is empty there. Count A (bit 31 of the
    // last word) as (E * D) >> 31 (IMAD, LEA.HI), restart as E0 * D + nx
    // (IMAD). Lanes past the last range hold E0 = 0 in R (they never count).
    (void)cm;
    const uint32_t D = row[WT];
    cnt += (E[WT - 1] * D) >> 31;
#pragma unroll
    for (int w = 0; w < WT; ++w) E[w] = R.e0[w] * D + nx[w];
    m = D;
}

// One bitset step on the byte whose table row is at row_addr. On the
// delimiter (the row's D word, returned in m) the accept bit of E is counted
// (masked by cm) and E restarts from E0.
template <int WT, int GR, bool REG, bool XG>
__device__ __forceinline__ void bstep(const BArgs& a, const Rows<WT, GR, REG>& R, uint32_t (&E)[WT], uint32_t row_addr,
                                      uint32_t cm, uint32_t& m, uint32_t& cnt) {
    if constexpr (REG) {
        uint32_t row[row_words<WT>()];
        load_words<row_words<WT>()>(row_addr, row);
        bstep_row<WT, GR, REG, XG>(a, R, E, row, row_addr, cm, m, cnt);
    } else {
        uint32_t nx[WT];
        uint32_t D;
        uint32_t M[WT], f[WT];
        load_words<WT>(row_addr, M);
        D = tma::lds32(row_addr + WT * 4u);
#pragma unroll
        for (int w = 0; w < WT; ++w) f[w] = E[w] & M[w];
        uint32_t prev = 0;
#pragma unroll
        for (int w4 = 0; w4 < WT / 4; ++w4) {
            uint32_t sh[4];
            R.get4(0, w4, sh);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t x = f[w4 * 4 + j] & sh[j];
                nx[w4 * 4 + j] = __funnelshift_l(prev, x, 1);
                prev = x;
            }
        }
        const int ng = a.n_groups;
        for (int g = 0; g < ng; ++g) {
            uint32_t acc = 0;
#pragma unroll
            for (int w4 = 0; w4 < WT / 4; ++w4) {
                uint32_t tr[4];
                R.get4(2 + 2 * g, w4, tr);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc |= f[w4 * 4 + j] & tr[j];
            }
            if (acc) {
#pragma unroll
                for (int w4 = 0; w4 < WT / 4; ++w4) {
                    uint32_t rr[4];
                    R.get4(3 + 2 * g, w4, rr);
#pragma unroll
                    for (int j = 0; j < 4; ++j) nx[w4 * 4 + j] |= rr[j];
                }
            }
        }
        // D: 1 on the delimiter, else 0. E0 is read only at a line end (rare):
        // E0 at a delimiter (nx is empty there), nx otherwise
        if (D) {
            cnt += (E[WT - 1] & cm) >> 31;
#pragma unroll
            for (int w4 = 0; w4 < WT / 4; ++w4) {
                uint32_t e0[4];
                R.get4(1, w4, e0);
#pragma unroll
                for (int j = 0; j < 4; ++j) E[w4 * 4 + j] = e0[j];
            }
        } else {
#pragma unroll
            for (int w = 0; w < WT; ++w) E[w] = nx[w];
        }
        m = D;
    }
}

template <int WT>
__device__ __forceinline__ bool any_bit(const uint32_t (&E)[WT]) {
    uint32_t x = 0;
#pragma unroll
    for (int w = 0; w < WT; ++w) x |= E[w];
    return x != 0;
}

template <int WT>
__device__ __forceinline__ void set_empty(uint32_t (&E)[WT]) {
#pragma unroll
    for (int w = 0; w < WT; ++w) E[w] = 0u;
}

// Byte k of a 32-bit word as the shared-memory address of its table row.
template <int WT>
__device__ __forceinline__ uint32_t row_of(const BArgs& a, uint32_t word, int k) {
    constexpr uint32_t rb = row_words<WT>() * 4u;
    static_assert(rb <= 255, "IDP.4A scales bytes by an 8-bit factor");
    return __dp4a(word, rb << (8 * k), a.tab);
}
template <int WT>
__device__ __forceinline__ uint32_t row_b(const BArgs& a, uint32_t b) {
    return a.tab + b * (row_words<WT>() * 4u);
}

// The line the walk is in from `pos` on, with direct loads, until its
// delimiter (or the end of the buffer, a virtual delimiter): its result.
// E entered holds the state before pos; an empty set ends the walk early.
template <int WT, int GR, bool REG, bool XG>
__device__ __forceinline__ void set_e0(const Rows<WT, GR, REG>& R, uint32_t (&E)[WT]) {
    if constexpr (REG) {
#pragma unroll
        for (int w = 0; w < WT; ++w) E[w] = R.e0[w];
    } else {
#pragma unroll
        for (int w4 = 0; w4 < WT / 4; ++w4) {
            uint32_t e0[4];
            R.get4(1, w4, e0);
#pragma unroll
            for (int j = 0; j < 4; ++j) E[w4 * 4 + j] = e0[j];
        }
    }
}

// The line the walk is in from `pos` on, with direct loads, until its
// delimiter (or the end of the buffer, a virtual delimiter): its result.
// E holds the state before pos; an empty set ends the walk early.
template <int WT, int GR, bool REG, bool XG>
__device__ __noinline__ uint32_t finish_line(const BArgs& a, const Rows<WT, GR, REG>& R, uint32_t (&E)[WT], uint64_t pos) {
    const uint32_t d = a.delim4 & 0xFFu;
    uint32_t c = 0;
    while (pos < a.len && any_bit(E)) {
        if (!(pos & 15) && pos + 16 <= a.len) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t x = tma::word_of(v, w);
                const uint32_t dm = __vcmpeq4(x, a.delim4);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if ((dm >> (8 * k)) & 1u) return E[WT - 1] >> 31;
                    uint32_t mm;
                    bstep<WT, GR, REG, XG>(a, R, E, row_of<WT>(a, x, k), ~0u, mm, c);
                }
            }
            pos += 16;
        } else {
            const uint32_t b = a.text[pos];
            if (b == d) return E[WT - 1] >> 31;
            uint32_t mm;
            bstep<WT, GR, REG, XG>(a, R, E, row_b<WT>(a, b), ~0u, mm, c);
            ++pos;
        }
    }
    return pos >= a.len ? E[WT - 1] >> 31 : 0u;
}

// A remainder piece [c0, c1) of a line batch with direct loads, under K2's
// ownership rules (range_direct in kernels_lines_tma.cu).
template <int WT, int GR, bool REG, bool XG>
__device__ __noinline__ void piece_direct(const BArgs& a, const Rows<WT, GR, REG>& R, uint64_t c0, uint64_t c1, uint64_t range,
                             uint32_t& cnt) {
    uint32_t E[WT];
    const uint32_t d = a.delim4 & 0xFFu;
    bool own = c0 == 0;
    if (own) set_e0<WT, GR, REG, XG>(R, E);
    else set_empty(E);
    uint64_t li = a.results ? a.line_base[range] : 0;
    uint32_t last = 0;
    for (uint64_t pos = c0; pos < c1; ++pos) {
        const uint32_t b = a.text[pos];
        if (b == d) {
            if (own && a.results) a.results[li] = static_cast<uint8_t>(E[WT - 1] >> 31);
            ++li;
            own = true;
        }
        uint32_t mm;   // the delimiter row counts A and restarts from E0
        bstep<WT, GR, REG, XG>(a, R, E, row_b<WT>(a, b), ~0u, mm, cnt);
        last = b;
    }
    const bool next_line = last == d && c1 < a.len;
    if (next_line || (own && last != d && c1 > c0)) {
        if (next_line) set_e0<WT, GR, REG, XG>(R, E);
        const uint32_t ok = finish_line<WT, GR, REG, XG>(a, R, E, c1);
        cnt += ok;
        if (a.results) a.results[li] = static_cast<uint8_t>(ok);
    }
}

// Fixed-stride strings [s0, s1) with direct loads (the strings past the last full TMA row).
template <int WT, int GR, bool REG, bool XG>
__device__ __noinline__ void strings_direct(const BArgs& a, const Rows<WT, GR, REG>& R, uint64_t s0, uint64_t s1, uint32_t& cnt) {
    for (uint64_t i = s0; i < s1; ++i) {
        uint32_t E[WT];
        set_e0<WT, GR, REG, XG>(R, E);
        uint32_t c = 0;
        for (uint32_t k = 0; k < a.stride; ++k) {
            const uint32_t b = a.text[i * a.stride + k];
            uint32_t mm;
            bstep<WT, GR, REG, XG>(a, R, E, row_b<WT>(a, b), ~0u, mm, c);
        }
        const uint32_t ok = E[WT - 1] >> 31;
        cnt += ok;
        if (a.results) a.results[i] = static_cast<uint8_t>(ok);
    }
}

template <class C, int WT, int GR, bool REG, bool XG, bool FIXED, bool RES>
__global__ void __launch_bounds__(C::warps * 32, 1) k_bits_tma(const __grid_constant__ BArgs a,
                                                             const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * C::stages * 8;
    const uint32_t tbar = a.bar_addr + C::warps * C::stages * 8;
    // the table and ring addresses are absolute: the dynamic window must start at
    // 0x400 (the host checks cudaDevAttrReservedSharedMemoryPerBlock before choosing this kernel)
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kLtSmemBase) __trap();
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
        tma::mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma::bulk_load(a.tab, a.img, a.img_words * 16u, tbar);
    }
    if (lane == 0) {
        for (int st = 0; st < C::stages; ++st) tma::mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    Rows<WT, GR, REG> R;
    R.load(a);
    constexpr int GR_ = GR;
    (void)GR_;
    __syncthreads();
    tma::mbar_wait(tbar, 0);

    uint32_t cnt = 0;
    if (blockIdx.x == 0 && warp == 0) {   // the input past the last full TMA row, with direct loads
        const uint64_t r0 = a.rows * a.chunk;
        if constexpr (FIXED) {
            const uint64_t n0 = r0 / a.stride, n1 = a.len / a.stride;
            for (uint64_t i = n0 + lane; i < n1; i += 32) strings_direct<WT, GR, REG, XG>(a, R, i, i + 1, cnt);
        } else {
            for (uint32_t p = lane; p < a.rem_pieces; p += 32) {
                const uint64_t c0 = r0 + static_cast<uint64_t>(p) * a.rem_piece;
                piece_direct<WT, GR, REG, XG>(a, R, c0, min(c0 + a.rem_piece, a.len), a.rows + p, cnt);
            }
        }
    }

    uint32_t phase = 0;
    const uint32_t ncol = a.chunk / C::slice;
    const uint32_t* stage = a.stage_addr + warp * C::stages;
    for (uint64_t tile = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x; tile < a.tiles;
         tile += static_cast<uint64_t>(gridDim.x) * C::warps) {
        const uint64_t row0 = tile * C::rows;
        if (lane == 0) {
            const uint32_t pro = ncol < C::stages ? ncol : C::stages;
            for (uint32_t st = 0; st < pro; ++st)
                tma::issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>(st * C::slice),
                                           static_cast<int32_t>(row0));
        }
        uint32_t E[C::chains][WT];
        bool valid[C::chains], own[C::chains];
        uint64_t li[C::chains];
        uint32_t cm[C::chains];   // all ones for valid ranges: only they count
        // per chain: REG steps restart from Rc[j].e0, which is empty for lanes
        // past the last range (they read zero fill and must never count)
        Rows<WT, GR, REG> Rc[C::chains];
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            const uint64_t row = row0 + j * 32 + lane;
            valid[j] = row < a.rows;
            cm[j] = valid[j] ? ~0u : 0u;
            asm volatile("" : "+r"(cm[j]));   // keep the mask in a register (no per-byte recompute)
            Rc[j] = R;
            if constexpr (REG) {
#pragma unroll
                for (int w = 0; w < WT; ++w) Rc[j].e0[w] &= cm[j];
            }
            // K2's ownership: the first range starts in the start state, every
            // other one in SKIP (the empty set) until its first line boundary
            own[j] = FIXED ? valid[j] : row == 0;
            if (own[j]) set_e0<WT, GR, REG, XG>(R, E[j]);
            else set_empty(E[j]);
            li[j] = !RES ? 0 : FIXED ? row * (a.chunk / a.stride) : (valid[j] ? a.line_base[row] : 0);
        }
        uint32_t last[C::chains] = {};
        uint32_t sp = 0;   // fixed stride: byte offset in the current string (the same in every range)
        for (uint32_t col = 0; col < ncol; ++col) {
            const uint32_t st = col % C::stages;
            tma::mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
            phase ^= 1u << st;
            // (code size and compile time: only the one-word kernel unrolls the granules and words)
#pragma unroll(WT == 1 ? C::slice / 16 : 1)
            for (int g = 0; g < C::slice / 16; ++g) {
                uint4 v[C::chains];
#pragma unroll
                for (int j = 0; j < C::chains; ++j) {
                    const uint32_t r = j * 32 + lane;
                    v[j] = tma::lds128(stage[st] + r * C::slice + (tma::granule<C::slice>(r, g) << 4));
                }
#pragma unroll(REG ? 4 : 1)
                for (int w = 0; w < 4; ++w) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // fixed stride: the string end is at the same offset in every range (warp-uniform)
                        bool end_fixed = false;
                        if constexpr (FIXED) {
                            end_fixed = ++sp == a.stride;
                            if (end_fixed) sp = 0;
                        }
#pragma unroll
                        for (int j = 0; j < C::chains; ++j) {
                            const uint32_t x = tma::word_of(v[j], w);
                            if constexpr (FIXED) {
                                uint32_t c = 0, mm;
                                bstep<WT, GR, REG, XG>(a, R, E[j], row_of<WT>(a, x, k), 0u, mm, c);
                                if (end_fixed) {   // count A after the last byte, restart
                                    const uint32_t ok = (E[j][WT - 1] & cm[j]) >> 31;
                                    cnt += ok;
                                    if (RES && valid[j]) a.results[li[j]++] = static_cast<uint8_t>(ok);
                                    set_e0<WT, GR, REG, XG>(R, E[j]);
                                }
                            } else {
                                // the delimiter's table row (D = all ones) counts A and restarts E
                                const uint32_t abit = RES ? E[j][WT - 1] >> 31 : 0u;
                                uint32_t m;
                                bstep<WT, GR, REG, XG>(a, Rc[j], E[j], row_of<WT>(a, x, k), cm[j], m, cnt);
                                if (RES && m) {   // a line ended here: record it if owned
                                    if (own[j] && valid[j]) a.results[li[j]] = static_cast<uint8_t>(abit);
                                    ++li[j];
                                    own[j] = true;
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < C::chains; ++j) last[j] = v[j].w >> 24;
            }
            __syncwarp();
            if (lane == 0 && col + C::stages < ncol) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma::issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>((col + C::stages) * C::slice),
                                           static_cast<int32_t>(row0));
            }
        }
        if constexpr (!FIXED) {
            // the line straddling each range's end (or starting right after it)
            const uint32_t d = a.delim4 & 0xFFu;
#pragma unroll
            for (int j = 0; j < C::chains; ++j) {
                if (!valid[j]) continue;
                const uint64_t pos = (row0 + j * 32 + lane + 1) * a.chunk;
                const bool next_line = last[j] == d && pos < a.len;
                if (next_line) set_e0<WT, GR, REG, XG>(R, E[j]);
                // (counting only: a range that saw no line start holds the empty set, which
                // finish_line ends at once, so ownership needs no tracking)
                if (next_line || ((RES ? own[j] : true) && last[j] != d)) {
                    const uint32_t ok = finish_line<WT, GR, REG, XG>(a, R, E[j], pos);
                    cnt += ok;
                    if (RES) a.results[li[j]] = static_cast<uint8_t>(ok);
                }
            }
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    tma::publish_count(a.slot, a.count, a.accumulate != 0, cnt, a.bar_addr + C::warps * C::stages * 8 + 8);
}

}  // namespace
}  // namespace rxg

namespace rxg {
namespace {

// Delimiters per range (line mode with results): TMA rows, then the
// remainder pieces; one warp per range, coalesced 16-byte loads.
__global__ void __launch_bounds__(256) k_bits_range_delims(const uint8_t* __restrict__ text, uint64_t len,
                                                           uint32_t chunk, uint64_t rows, uint32_t rem_piece,
                                                           uint64_t nranges, uint32_t delim,
                                                           unsigned long long* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    const uint32_t d4 = delim * 0x01010101u;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nranges;
         i += nwarps) {
        const uint64_t c0 = i < rows ? i * chunk : rows * chunk + (i - rows) * rem_piece;
        const uint64_t c1 = min(c0 + (i < rows ? chunk : rem_piece), len);
        uint32_t n = 0;
        uint64_t pos = c0 + 16 * lane;
        for (; pos + 16 <= c1; pos += 512) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(text + pos));
            n += __popc(__vcmpeq4(v.x, d4)) + __popc(__vcmpeq4(v.y, d4)) + __popc(__vcmpeq4(v.z, d4)) +
                 __popc(__vcmpeq4(v.w, d4));
        }
        n /= 8;
        for (; pos < c1; ++pos) n += text[pos] == delim;
        n = __reduce_add_sync(0xFFFFFFFFu, n);
        if (lane == 0) out[i] = n;
    }
}

struct Split {
    uint64_t rows;
    uint32_t rem_piece, rem_pieces;
};

Split split_of(uint64_t len, uint32_t chunk, bool lines) {
    Split s{};
    s.rows = len / chunk;
    const uint64_t rem = len - s.rows * chunk;
    if (lines && rem) {
        s.rem_piece = static_cast<uint32_t>(((rem + 31) / 32 + 15) & ~uint64_t(15));
        if (s.rem_piece < 16) s.rem_piece = 16;
        s.rem_pieces = static_cast<uint32_t>((rem + s.rem_piece - 1) / s.rem_piece);
    }
    return s;
}

using ShapeR = Shape<24, 2, 32, 3>;   // registers (WT 2, 4)
using ShapeR1 = Shape<24, 4, 32, 2>;  // one word: four independent chains per lane hide the table loads
using ShapeS = Shape<16, 1, 32, 4>;   // shared-memory rows (WT 8, 16)

template <class C>
uint32_t stage_space(uint32_t table_bytes, BArgs& a) {
    const uint32_t base = kLtSmemBase;   // the dynamic window starts at 0x400
    a.tab = base;
    uint32_t p = (base + table_bytes + 1023) & ~1023u;
    for (int k = 0; k < C::warps * C::stages; ++k, p += C::stage_bytes) a.stage_addr[k] = p;
    a.bar_addr = (p + 7) & ~7u;
    return a.bar_addr + C::warps * C::stages * 8 + 8 + 4 * C::warps - base;
}

template <class C, int WT, int GR, bool REG, bool XG, bool FIXED>
int per_sm(uint32_t smem) {
    int n = 0;
    auto* k = k_bits_tma<C, WT, GR, REG, XG, FIXED, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, C::warps * 32, smem);
    return n < 1 ? 1 : n;
}

uint32_t unit_of(uint32_t slice, uint32_t stride) {   // chunk granularity: slice, and whole strings
    if (!stride) return slice;
    uint32_t a = slice, b = stride;
    while (b) {
        const uint32_t t = a % b;
        a = b;
        b = t;
    }
    const uint64_t l = static_cast<uint64_t>(slice) / a * stride;
    return l > (1u << 20) ? 0u : static_cast<uint32_t>(l);
}

template <class C, int WT, int GR, bool REG, bool XG, bool FIXED>
uint32_t auto_chunk(const BitsImage& b, uint64_t len, uint32_t stride) {
    BArgs a{};
    const uint32_t smem = stage_space<C>(static_cast<uint32_t>(b.t.img.size() * 4), a);
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t ranges =
        static_cast<uint64_t>(per_sm<C, WT, GR, REG, XG, FIXED>(smem)) * device_sm_count(dev) * C::warps * C::rows;
    const uint32_t unit = unit_of(C::slice, FIXED ? stride : 0);
    if (!unit) return 0;
    uint64_t c = (len + ranges - 1) / ranges;
    c = (c + unit - 1) / unit * unit;
    const uint64_t lo = ((4u * C::slice + unit - 1) / unit) * unit;
    if (c < lo) c = lo;
    if (c > (1u << 22)) c = (1u << 22) / unit * unit;
    return static_cast<uint32_t>(c);
}

template <class C, int WT, int GR, bool REG, bool XG, bool FIXED>
cudaError_t run(const BitsImage& b, const uint8_t* text, uint64_t len, int32_t delim, uint32_t stride, uint32_t chunk,
                unsigned long long* count, uint8_t* results, void* scratch, size_t scratch_bytes, CountSlot cs,
                cudaStream_t st) {
    if (len == 0) return cs.accumulate ? cudaSuccess : cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    if (chunk == 0) chunk = auto_chunk<C, WT, GR, REG, XG, FIXED>(b, len, stride);
    if (chunk == 0 || chunk % C::slice || (FIXED && chunk % stride)) return cudaErrorInvalidValue;
    BArgs a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    const Split sp = split_of(len, chunk, !FIXED);
    a.rows = sp.rows;
    a.tiles = (a.rows + C::rows - 1) / C::rows;
    a.rem_piece = sp.rem_piece;
    a.rem_pieces = sp.rem_pieces;
    a.stride = FIXED ? stride : 0;
    a.delim4 = FIXED ? 0u : static_cast<uint32_t>(delim) * 0x01010101u;
    a.n_groups = b.t.G;
    a.two = 2;
    a.img = static_cast<const uint4*>(b.d_img);
    a.img_words = static_cast<uint32_t>(b.t.img.size() / 4);
    a.regs_g = b.d_regs;
    const uint32_t smem = stage_space<C>(static_cast<uint32_t>(b.t.img.size() * 4), a);
    a.xg = a.tab + b.t.xg_off;
    a.count = count;
    a.slot = cs.p;
    a.accumulate = cs.accumulate ? 1 : 0;
    a.results = results;
    if (results && !FIXED) {
        const uint64_t nr = sp.rows + sp.rem_pieces;
        if (!scratch || scratch_bytes < bits_scratch_bytes(len, chunk, true, true)) return cudaErrorInvalidValue;
        auto* per = static_cast<unsigned long long*>(scratch);
        auto* base = per + nr;
        void* temp = base + nr;
        size_t temp_bytes = scratch_bytes - 2 * nr * sizeof(unsigned long long);
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t want = (nr + 7) / 8, cap = static_cast<uint64_t>(device_sm_count(dev)) * 8;
        k_bits_range_delims<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, st>>>(
            text, len, chunk, sp.rows, sp.rem_piece, nr, static_cast<uint32_t>(delim), per);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, per, base, static_cast<int64_t>(nr), st);
        if (e != cudaSuccess) return e;
        a.line_base = base;
    }
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (a.rows > 0 && tma::make_map(&map, text, a.rows, chunk, C::slice, C::rows) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const int ps = per_sm<C, WT, GR, REG, XG, FIXED>(smem);
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = static_cast<uint64_t>(ps) * device_sm_count(dev);
    const int grid = static_cast<int>(a.tiles == 0 ? 1 : (a.tiles < cap ? a.tiles : cap));
    if (results) {
        cudaFuncSetAttribute(k_bits_tma<C, WT, GR, REG, XG, FIXED, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        k_bits_tma<C, WT, GR, REG, XG, FIXED, true><<<grid, C::warps * 32, smem, st>>>(a, map);
    } else {
        k_bits_tma<C, WT, GR, REG, XG, FIXED, false><<<grid, C::warps * 32, smem, st>>>(a, map);
    }
    return cudaGetLastError();
}

struct ChunkF {
    const BitsImage& b;
    uint64_t len;
    uint32_t stride;
    template <class C, int WT, int GR, bool REG, bool XG, bool FIXED>
    uint32_t go() const { return auto_chunk<C, WT, GR, REG, XG, FIXED>(b, len, stride); }
};

struct LaunchF {
    const BitsImage& b;
    const uint8_t* text;
    uint64_t len;
    int32_t delim;
    uint32_t stride, chunk;
    unsigned long long* count;
    uint8_t* results;
    void* scratch;
    size_t scratch_bytes;
    CountSlot cs;
    cudaStream_t st;
    template <class C, int WT, int GR, bool REG, bool XG, bool FIXED>
    cudaError_t go() const {
        return run<C, WT, GR, REG, XG, FIXED>(b, text, len, delim, stride, chunk, count, results, scratch, scratch_bytes,
                                          cs, st);
    }
};

template <class F>
auto dispatch(const BitsImage& b, bool fixed, F f) {
    const int WT = b.t.WT;
    const bool xg = b.t.G > b.t.GR && b.t.WT <= 4;   // (the broadcast kernels loop over every group)
#define RXG_BITS_CASE(W, S, REG)                                                                          \
    if (WT == W) {                                                                                        \
        if (fixed) return xg ? f.template go<S, W, 2, REG, true, true>() : f.template go<S, W, 2, REG, false, true>(); \
        return xg ? f.template go<S, W, 2, REG, true, false>() : f.template go<S, W, 2, REG, false, false>();         \
    }
    RXG_BITS_CASE(1, ShapeR, true)
    RXG_BITS_CASE(2, ShapeR, true)
    RXG_BITS_CASE(4, ShapeR, true)
    RXG_BITS_CASE(8, ShapeS, false)
    RXG_BITS_CASE(16, ShapeS, false)
#undef RXG_BITS_CASE
    return f.template go<ShapeR, 1, 2, true, false, false>();   // unreachable for ok tables
}

}  // namespace

size_t bits_scratch_bytes(uint64_t len, uint32_t chunk, bool lines, bool results) {
    if (!lines || !results || chunk == 0) return 0;
    const Split sp = split_of(len, chunk, true);
    const uint64_t nr = sp.rows + sp.rem_pieces;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<int64_t>(nr));
    return 2 * nr * sizeof(unsigned long long) + temp + 256;
}

uint32_t bits_chunk(const BitsImage& b, uint64_t len, int32_t delimiter, uint32_t stride, uint32_t chunk) {
    if (chunk) return chunk;
    return dispatch(b, delimiter < 0, ChunkF{b, len, stride});
}

cudaError_t launch_bits(const BitsImage& b, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                        uint32_t chunk, unsigned long long* count, uint8_t* results, void* scratch,
                        size_t scratch_bytes, CountSlot cs, cudaStream_t st) {
    if (!b.t.ok) return cudaErrorInvalidValue;
    return dispatch(b, delimiter < 0, LaunchF{b, text, len, delimiter, stride, chunk, count, results, scratch,
                                              scratch_bytes, cs, st});
}

}  // namespace rxg
