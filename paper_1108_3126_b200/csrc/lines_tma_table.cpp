// Absolute-address shared-memory layout for the TMA line kernel
// (kernels_lines_tma.cu). Rows are raw-byte indexed u16 entries (4-byte
// column stride) holding the absolute shared address of the next row, so one
// IMAD + one LDS advance a string by one byte.
//
//   [0x400 .. lo_addr)        stage-ring slots (1 KB, 128 B aligned)
//   [lo_addr .. 0x8000)       main rows: DFA states 0..S-1, SKIP, VOID (absorbing,
//                             for lanes whose range lies past the input)
//   [0x8000]                  START_A (copy of the start row, entered on an
//                             accepted line end; bit 15 set)
//   [main + tail_delta ..)    tail copies of states 0..S-1, then TERM_A, TERM_R
//   [..]                      remaining stage slots, then the mbarriers
//
// Bank placement: byte b of a row at word offset o sits in bank (o + b) mod 32.
// Each main row gets its own o (rows are addressed absolutely, so the choice
// is free): greedily, hottest row first, the o that minimises the expected
// number of lanes colliding with already placed rows under the sampled
// state x byte frequencies (lt_sample_freq). Placement changes speed only,
// never results.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>

#include "options.hpp"
#include "lines_tma.hpp"

namespace rxg {

namespace {

void put16(std::vector<uint8_t>& img, uint32_t off, uint32_t v) {
    const uint16_t x = static_cast<uint16_t>(v);
    std::memcpy(&img[off], &x, 2);
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

LtTable make_direct_table(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq,
                          uint32_t c);

}  // namespace

std::vector<double> lt_sample_freq(const Program& p, const Dfa& d, uint8_t delim, const uint8_t* sample,
                                   uint64_t len) {
    // rows: states 0..S-1, SKIP (S), VOID (S+1), START_A (S+2). START_A takes
    // the byte after every accepted line end. SKIP is estimated: a range
    // walks about half a line before its first delimiter, and ranges of a
    // large input are a few KB (one wave of ~340k ranges per GB), so SKIP's
    // share of the steps is about (mean line length / 2) / 4 KB.
    const size_t S = static_cast<size_t>(d.n_states);
    std::vector<double> f((S + 3) * 256, 0.0);
    int32_t s = d.start;
    bool after_acc = false;
    uint64_t lines = 0;
    for (uint64_t i = 0; i < len; ++i) {
        const uint8_t b = sample[i];
        f[(after_acc ? S + 2 : static_cast<size_t>(s)) * 256 + b] += 1.0;
        after_acc = b == delim && d.accept[static_cast<size_t>(s)] != 0;
        lines += b == delim;
        s = b == delim ? d.start : d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + p.byte_class[b]];
    }
    const double mean_line = static_cast<double>(len) / static_cast<double>(lines ? lines : 1);
    double skip_share = std::min(0.5, mean_line / 2.0 / 4096.0);
    if (const char* e = rxg::option("RXG_SKIP_SHARE")) skip_share = std::atof(e);   // A/B override (tools)
    for (uint64_t i = 0; i < len; ++i) f[S * 256 + sample[i]] += skip_share;
    return f;
}

uint32_t lt_sync_lookback(const Program& p, const Dfa& d, const uint8_t* sample, uint64_t len) {
    // the true state before every byte of the sample
    std::vector<int32_t> st(len + 1);
    st[0] = d.start;
    for (uint64_t i = 0; i < len; ++i)
        st[i + 1] = d.next[static_cast<size_t>(st[i]) * static_cast<size_t>(d.n_classes) + p.byte_class[sample[i]]];
    for (uint32_t k : {16u, 32u}) {
        uint64_t tried = 0, wrong = 0;
        for (uint64_t pos = 64; pos <= len; pos += 61) {
            int32_t g = d.start;
            for (uint64_t i = pos - k; i < pos; ++i)
                g = d.next[static_cast<size_t>(g) * static_cast<size_t>(d.n_classes) + p.byte_class[sample[i]]];
            ++tried;
            wrong += g != st[pos];
        }
        if (tried >= 64 && wrong * 1000 <= tried) return k;   // at most 0.1% of ranges repaired
    }
    return 64;
}

std::vector<double> lt_sample_freq_plain(const Program& p, const Dfa& d, const uint8_t* sample, uint64_t len) {
    std::vector<double> f(static_cast<size_t>(d.n_states) * 256, 0.0);
    int32_t s = d.start;
    for (uint64_t i = 0; i < len; ++i) {
        f[static_cast<size_t>(s) * 256 + sample[i]] += 1.0;
        s = d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + p.byte_class[sample[i]]];
    }
    return f;
}

// Direct layouts: row r holds the u16 entry for byte b at base_r + c*b, c the
// column stride in bytes (even). The entries of one row occupy every other
// half-word of a c*256-byte span, so g = c/2 rows interleave in one span at
// 2-byte offsets (a "group"). Lanes of one group reading the same byte read
// the same or the next word: never a bank conflict. With c = 4 the entry
// for byte b is word b, so bytes 32 apart ('a'/'A', 'e'/'E', ' '/'@') share a
// bank; c = 6 or 10 spread bytes over banks floor(c*b/4) mod 32 instead.
// The stride is chosen from sampled state x byte frequencies (the expected
// colliding mass of the two hottest rows); groups are filled hottest rows
// first, then each group gets the bank offset that collides least with the
// groups already placed. Placement changes speed only, never results.
namespace {

uint32_t col_word(uint32_t c, uint32_t h, uint32_t b) { return (2u * h + c * b) / 4u; }

std::vector<std::array<double, 32>> bank_hist(const std::vector<double>* f, uint32_t nrows, uint32_t c,
                                              std::vector<double>& tot) {
    std::vector<std::array<double, 32>> H(nrows);
    tot.assign(nrows, 0.0);
    for (uint32_t r = 0; r < nrows; ++r) {
        H[r].fill(0.0);
        if (!f) continue;
        for (uint32_t b = 0; b < 256; ++b) {
            const size_t i = static_cast<size_t>(r) * 256u + b;
            const double x = i < f->size() ? (*f)[i] : 0.0;
            H[r][col_word(c, 0, b) & 31u] += x;
            tot[r] += x;
        }
    }
    return H;
}

}  // namespace

uint32_t lt_choose_col_bytes(const std::vector<double>* f, uint32_t nrows) {
    if (const char* e = rxg::option("RXG_COL_BYTES")) {   // A/B override (tools)
        const uint32_t v = static_cast<uint32_t>(std::atoi(e));
        if (v >= 4 && v % 2 == 0 && v <= 14) return v;
    }
    if (!f) return kLtColBytes;
    std::vector<double> tot(nrows, 0.0);
    for (uint32_t r = 0; r < nrows; ++r)
        for (uint32_t b = 0; b < 256; ++b) {
            const size_t i = static_cast<size_t>(r) * 256u + b;
            tot[r] += i < f->size() ? (*f)[i] : 0.0;
        }
    std::vector<uint32_t> order(nrows);
    for (uint32_t r = 0; r < nrows; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return tot[a] > tot[b]; });
    const uint32_t top = std::min<uint32_t>(2, nrows);
    uint32_t best_c = kLtColBytes;
    double best = -1.0;
    for (uint32_t c : {4u, 6u, 10u}) {
        // colliding mass: (row h, byte b) vs (row h', byte b') in one group,
        // different words in the same bank
        double cost = 0.0;
        for (uint32_t i = 0; i < top; ++i)
            for (uint32_t j = 0; j < top; ++j)
                for (uint32_t b = 0; b < 256; ++b) {
                    const double x = (*f)[static_cast<size_t>(order[i]) * 256u + b];
                    if (x == 0.0) continue;
                    const uint32_t wa = col_word(c, i, b);
                    for (uint32_t b2 = 0; b2 < 256; ++b2) {
                        const double y = (*f)[static_cast<size_t>(order[j]) * 256u + b2];
                        if (y == 0.0) continue;
                        const uint32_t wb = col_word(c, j, b2);
                        if (wa != wb && ((wa ^ wb) & 31u) == 0) cost += x * y;
                    }
                }
        if (best < 0.0 || cost < best * 0.98) {   // a larger stride must win clearly
            best = cost;
            best_c = c;
        }
    }
    return best_c;
}

RowPlacement lt_place_groups(const std::vector<double>* f, uint32_t nrows, uint32_t c, bool group_rows) {
    RowPlacement pl;
    pl.col_bytes = c;
    pl.pair.assign(nrows, 0);
    pl.half.assign(nrows, 0);
    std::vector<double> tot;
    const std::vector<std::array<double, 32>> H = bank_hist(f, nrows, c, tot);
    std::vector<uint32_t> order(nrows);
    for (uint32_t r = 0; r < nrows; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return tot[a] > tot[b]; });
    const uint32_t per = group_rows && !rxg::option("RXG_NO_ROW_PAIRS") ? c / 2u : 1u;   // env: A/B switch (tools)
    pl.npairs = (nrows + per - 1) / per;
    std::vector<std::array<double, 32>> HP(pl.npairs);
    std::vector<double> tp(pl.npairs, 0.0);
    for (uint32_t q = 0; q < pl.npairs; ++q) HP[q].fill(0.0);
    for (uint32_t i = 0; i < nrows; ++i) {
        const uint32_t r = order[i], q = i / per;
        pl.pair[r] = q;
        pl.half[r] = i % per;
        for (int k = 0; k < 32; ++k) HP[q][static_cast<size_t>(k)] += H[r][static_cast<size_t>(k)];
        tp[q] += tot[r];
    }
    pl.pair_off.assign(pl.npairs, 0);
    std::vector<uint32_t> placed;
    for (uint32_t q = 0; q < pl.npairs; ++q) {   // groups are already in hotness order
        if (tp[q] == 0.0) {
            pl.pair_off[q] = (q * 9u) & 31u;
            continue;
        }
        double best = -1.0;
        uint32_t bo = 0;
        for (uint32_t o = 0; o < 32; ++o) {
            double cc = 0.0;
            for (uint32_t q2 : placed)
                for (uint32_t k = 0; k < 32; ++k) cc += HP[q][k] * HP[q2][(k + o + 32 - pl.pair_off[q2]) & 31u];
            if (best < 0.0 || cc < best) {
                best = cc;
                bo = o;
            }
        }
        pl.pair_off[q] = bo;
        placed.push_back(q);
    }
    return pl;
}

namespace {

// Row numbering for the class layout. Row r starts at word (base + r*rb/4)
// with rb/4 odd, so its bank offset cycles through all 32 values as r does:
// choosing a row index for a state chooses its bank offset. Hot states are
// numbered greedily (hottest first) into the offset class that collides least
// with the already numbered hot states under the sampled class frequencies.
std::vector<uint32_t> number_states(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq,
                                    uint32_t nmain, uint32_t base_word, uint32_t rb_words, uint32_t delim_col,
                                    uint32_t range_x = 0, uint32_t range_k = 0) {
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    std::vector<uint32_t> row(nmain);
    for (uint32_t s = 0; s < nmain; ++s) row[s] = s;
    if (!freq || freq->size() < static_cast<size_t>(S) * 256) return row;
    auto off_of = [&](uint32_t r) { return (base_word + r * rb_words) & 31u; };
    // bank histogram of each state in a row at offset 0: column c sits in word c/2
    // (SKIP, row S, too when the sample covers it: lt_sample_freq estimates it)
    const uint32_t NS = freq->size() >= static_cast<size_t>(S + 1) * 256 && nmain > S ? S + 1 : S;
    std::vector<std::array<double, 32>> H(NS);
    std::vector<double> tot(NS, 0.0);
    for (uint32_t s = 0; s < NS; ++s) {
        H[s].fill(0.0);
        for (int b = 0; b < 256; ++b) {
            const double x = (*freq)[static_cast<size_t>(s) * 256 + static_cast<size_t>(b)];
            if (x == 0.0) continue;
            const uint32_t c = range_k ? std::min<uint32_t>(static_cast<uint32_t>(b) ^ range_x, range_k)
                                       : (b == delim ? delim_col : p.byte_class[b]);
            H[s][(c / 2) & 31u] += x;
            tot[s] += x;
        }
    }
    std::vector<uint32_t> order(NS);
    for (uint32_t s = 0; s < NS; ++s) order[s] = s;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return tot[a] > tot[b]; });
    // free rows per bank offset
    std::array<std::vector<uint32_t>, 32> free_rows;
    for (uint32_t r = nmain; r-- > 0;) free_rows[off_of(r)].push_back(r);   // pop_back yields the lowest
    std::vector<uint32_t> hot_state, hot_off;
    std::vector<bool> placed(nmain, false);
    constexpr size_t kHot = 64;
    for (uint32_t s : order) {
        if (tot[s] == 0.0) break;
        double best = -1.0;
        uint32_t bo = 0;
        for (uint32_t o = 0; o < 32; ++o) {
            if (free_rows[o].empty()) continue;
            double c = 0.0;
            for (size_t i = 0; i < hot_state.size(); ++i)
                for (uint32_t k = 0; k < 32; ++k) c += H[s][k] * H[hot_state[i]][(k + o + 32 - hot_off[i]) & 31u];
            if (best < 0.0 || c < best) {
                best = c;
                bo = o;
            }
        }
        row[s] = free_rows[bo].back();
        free_rows[bo].pop_back();
        placed[s] = true;
        if (hot_state.size() < kHot) {
            hot_state.push_back(s);
            hot_off.push_back(bo);
        }
    }
    // cold states, SKIP and VOID take the remaining rows in order
    std::vector<uint32_t> rest;
    for (auto& v : free_rows) rest.insert(rest.end(), v.begin(), v.end());
    std::sort(rest.begin(), rest.end());
    size_t k = 0;
    for (uint32_t s = 0; s < nmain; ++s)
        if (!placed[s]) row[s] = rest[k++];
    return row;
}

// Class layout (large DFAs): rows indexed by byte class, u16 row-index entries.
// Range-clamped columns for the class layout: column = min(byte ^ x, k), so
// no class map is read per byte (one IMNMX instead of an LDS). Every byte
// that matters (a class other than 0, or the delimiter) must land below k;
// column k collects the class-0 bytes. Returns k = 0 when no x gives at most
// `max_cols` columns.
uint32_t range_cols(const Program& p, uint8_t delim, uint32_t max_cols, uint32_t* x_out, bool with_delim = true) {
    uint32_t best_k = 0, best_x = 0;
    for (uint32_t x = 0; x < 256; ++x) {
        uint32_t hi = 0;
        for (uint32_t b = 0; b < 256; ++b)
            if ((with_delim && b == delim) || p.byte_class[b] != 0) hi = std::max(hi, b ^ x);
        const uint32_t k = hi + 1;
        if (k + 1 <= max_cols && (best_k == 0 || k < best_k)) {
            best_k = k;
            best_x = x;
        }
    }
    *x_out = best_x;
    return best_k;
}

LtTable make_class_table(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq,
                         uint32_t range_x = 0, uint32_t range_k = 0) {
    LtTable t;
    t.cls = true;
    t.range_x = range_x;
    t.range_k = range_k;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    // class layout: the byte classes + the delimiter column; range layout: k + 1 columns
    const uint32_t ncols = range_k ? range_k + 1 : static_cast<uint32_t>(p.n_classes) + 1;
    const uint32_t delim_col = range_k ? (static_cast<uint32_t>(delim) ^ range_x) : ncols - 1;
    auto class_of_col = [&](uint32_t c) -> int32_t {   // -1: the delimiter column
        if (!range_k) return c == delim_col ? -1 : static_cast<int32_t>(c);
        if (c == range_k) return 0;
        const uint32_t b = c ^ range_x;
        return b == delim ? -1 : static_cast<int32_t>(p.byte_class[b]);
    };
    uint32_t rb = align_up(ncols * 2u, 4u);
    if (((rb / 4u) & 1u) == 0) rb += 4;   // odd word stride: consecutive rows rotate banks
    t.row_bytes = rb;
    uint32_t k = 0;
    while ((1u << k) < S + 2) ++k;       // states, SKIP, VOID below START_A
    t.acc_shift = k;
    const uint32_t acc = 1u << k;
    const uint32_t nrows = acc + 1 + (S + 2) + 2;   // START_A, tail copies of the S+2 main rows, TERM_A, TERM_R
    if (nrows > 0xFFFFu) return t;
    t.cmap_addr = kLtSmemBase;
    const uint32_t rows_addr = kLtSmemBase + 1024;
    t.lo_addr = kLtSmemBase;
    t.lo_bytes = align_up(1024 + nrows * rb, 16);
    if (kLtSmemBase + t.lo_bytes > 200u * 1024u) return t;
    t.lo.assign(t.lo_bytes, 0);
    t.hi_addr = kLtSmemBase + t.lo_bytes;
    t.hi_bytes = 0;
    t.hole_lo = align_up(rows_addr + (S + 2) * rb, 256);
    t.hole_hi = rows_addr + acc * rb;
    // class map: absolute address of each byte's column in row 0
    for (int b = 0; b < 256; ++b) {
        const uint32_t col = b == delim ? delim_col : p.byte_class[b];
        const uint32_t v = rows_addr + col * 2u;
        std::memcpy(&t.lo[static_cast<size_t>(b) * 4], &v, 4);
    }
    auto put = [&](uint32_t row, uint32_t col, uint32_t v) { put16(t.lo, 1024 + row * rb + col * 2u, v); };
    const std::vector<uint32_t> R = number_states(p, d, delim, freq, S + 2, rows_addr / 4u, rb / 4u, delim_col,
                                                  range_x, range_k);
    const uint32_t skip = R[S], vd = R[S + 1], tail0 = acc + 1, term_a = acc + 1 + S + 2, term_r = term_a + 1;
    t.start = R[static_cast<uint32_t>(d.start)];
    t.skip = skip;
    t.void_row = vd;
    t.tail_delta = tail0;
    t.term_acc = term_a;
    t.term_rej = term_r;
    for (uint32_t s = 0; s < S; ++s) {
        const bool ac = d.accept[s] != 0;
        const uint32_t r = R[s];
        for (uint32_t c = 0; c < ncols; ++c) {
            const int32_t cl = class_of_col(c);
            if (cl < 0) {
                put(r, c, ac ? acc : t.start);
                put(tail0 + r, c, ac ? term_a : term_r);
            } else {
                const uint32_t nx = R[static_cast<uint32_t>(d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + static_cast<uint32_t>(cl)])];
                put(r, c, nx);
                put(tail0 + r, c, tail0 + nx);
            }
        }
    }
    for (uint32_t c = 0; c < ncols; ++c) {
        put(skip, c, class_of_col(c) < 0 ? t.start : skip);
        put(vd, c, vd);
        put(term_a, c, term_a);
        put(term_r, c, term_r);
        put(acc, c, 0);
    }
    std::memcpy(&t.lo[1024 + acc * rb], &t.lo[1024 + t.start * rb], rb);   // START_A = start row
    t.smem_table_end = kLtSmemBase + t.lo_bytes;
    t.ok = true;
    return t;
}

}  // namespace

LtTable make_lines_tma_table(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq,
                             bool force_class) {
    force_class = force_class || rxg::option("RXG_FORCE_CLASS") != nullptr;   // tests: class layouts on small DFAs
    if (force_class || d.n_states > kLtDirectMaxStates) {
        // range-clamped columns when they fit (no class-map lookup per byte)
        uint32_t x = 0;
        const uint32_t k = rxg::option("RXG_NO_RANGE_LAYOUT") ? 0 : range_cols(p, delim, 128, &x);
        if (k) {
            LtTable t = make_class_table(p, d, delim, freq, x, k);
            // the range kernel's 96 KB stage ring goes into the unused rows first
            const uint32_t hole = t.hole_hi > t.hole_lo ? (t.hole_hi - t.hole_lo) / 2048u * 2048u : 0u;
            const uint32_t ring = 96u * 1024u;
            if (t.ok && t.lo_bytes + (ring > hole ? ring - hole : 0u) + 4096u <= 224u * 1024u) return t;
        }
        return make_class_table(p, d, delim, freq);
    }
    const uint32_t c = lt_choose_col_bytes(freq, static_cast<uint32_t>(d.n_states) + 2);
    LtTable t = make_direct_table(p, d, delim, freq, c);
    if (!t.ok && c != kLtColBytes) t = make_direct_table(p, d, delim, freq, kLtColBytes);
    return t.ok ? t : make_class_table(p, d, delim, freq);   // the direct rows did not fit below 64 KB
}

namespace {

// Main rows (states 0..S-1, SKIP (S), VOID (S+1)) in groups sharing column
// words, each group at a chosen bank offset; column stride c.
LtTable make_direct_table(const Program& p, const Dfa& d, uint8_t delim, const std::vector<double>* freq,
                          uint32_t c) {
    LtTable t;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    const RowPlacement pl = lt_place_groups(freq, S + 2, c, true);
    if (pl.npairs * (256u * c + 128u) + kLtSmemBase > kLtAccAddr) return t;
    const uint32_t R = 256u * c;
    t.col_bytes = c;
    // START_A (counted: the only main-loop row at >= 0x8000) at the bank offset
    // that collides least with the groups under the sampled bytes after
    // accepted line ends
    uint32_t acc_off = 0;
    if (freq && freq->size() >= static_cast<size_t>(S + 3) * 256) {
        std::vector<double> tot;
        const auto H = bank_hist(freq, S + 3, c, tot);
        std::vector<std::array<double, 32>> HG(pl.npairs);
        for (auto& h : HG) h.fill(0.0);
        for (uint32_t r = 0; r < S + 2; ++r)
            for (int k = 0; k < 32; ++k) HG[pl.pair[r]][static_cast<size_t>(k)] += H[r][static_cast<size_t>(k)];
        double best = -1.0;
        for (uint32_t o = 0; o < 32; ++o) {
            double cc = 0.0;
            for (uint32_t q = 0; q < pl.npairs; ++q)
                for (uint32_t k = 0; k < 32; ++k) cc += H[S + 2][k] * HG[q][(k + o + 32 - pl.pair_off[q]) & 31u];
            if (best < 0.0 || cc < best) {
                best = cc;
                acc_off = o;
            }
        }
    }
    const uint32_t acc_row = kLtAccAddr + 4u * acc_off;
    t.lo_addr = (kLtAccAddr - pl.npairs * (R + 128u)) & ~127u;
    std::vector<uint32_t> paddr(pl.npairs), addr(S + 2);
    uint32_t cur = t.lo_addr;
    for (uint32_t q = 0; q < pl.npairs; ++q) {
        paddr[q] = cur + ((pl.pair_off[q] * 4u + 128u - (cur & 127u)) & 127u);
        cur = paddr[q] + R;
    }
    for (uint32_t r = 0; r < S + 2; ++r) addr[r] = paddr[pl.pair[r]] + 2u * pl.half[r];
    if (cur > kLtAccAddr) return t;
    // upper region: START_A at 0x8000, tail copies at main + tail_delta, TERM rows
    t.tail_delta = align_up(acc_row + R - t.lo_addr, 128);
    t.term_acc = align_up(cur + t.tail_delta, 4);
    t.term_rej = t.term_acc + R;
    const uint32_t hi_end = t.term_rej + R;
    if (hi_end > 0x10000u) return t;
    t.lo_bytes = align_up(kLtAccAddr - t.lo_addr, 16);
    t.hi_addr = kLtAccAddr;
    t.hi_bytes = align_up(hi_end - kLtAccAddr, 16);
    t.lo.assign(t.lo_bytes, 0);
    t.hi.assign(t.hi_bytes, 0);
    auto main_row = [&](uint32_t s) { return addr[s]; };
    auto tail_row = [&](uint32_t s) { return addr[s] + t.tail_delta; };
    t.start = main_row(static_cast<uint32_t>(d.start));
    t.skip = main_row(S);
    t.void_row = main_row(S + 1);
    auto next = [&](uint32_t s, int b) {
        return static_cast<uint32_t>(d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + p.byte_class[b]]);
    };
    auto put_lo = [&](uint32_t row, int b, uint32_t v) { put16(t.lo, row - t.lo_addr + c * static_cast<uint32_t>(b), v); };
    auto put_hi = [&](uint32_t row, int b, uint32_t v) { put16(t.hi, row - kLtAccAddr + c * static_cast<uint32_t>(b), v); };
    for (uint32_t s = 0; s < S; ++s) {
        const bool acc = d.accept[s] != 0;
        for (int b = 0; b < 256; ++b) {
            if (b == delim) {
                put_lo(main_row(s), b, acc ? acc_row : t.start);
                put_hi(tail_row(s), b, acc ? t.term_acc : t.term_rej);
            } else {
                put_lo(main_row(s), b, main_row(next(s, b)));
                put_hi(tail_row(s), b, tail_row(next(s, b)));
            }
        }
    }
    for (int b = 0; b < 256; ++b) {
        put_lo(t.skip, b, b == delim ? t.start : t.skip);
        put_lo(t.void_row, b, t.void_row);
        put_hi(t.term_acc, b, t.term_acc);
        put_hi(t.term_rej, b, t.term_rej);
    }
    for (int b = 0; b < 256; ++b) {   // START_A = the start row (low halves of its own words)
        uint16_t v;
        std::memcpy(&v, &t.lo[t.start - t.lo_addr + c * static_cast<uint32_t>(b)], 2);
        put_hi(acc_row, b, v);
    }

    t.smem_table_end = kLtAccAddr + t.hi_bytes;
    t.ok = true;
    return t;
}

}  // namespace

LtTable make_chunk_tma_table(const Program& p, const Dfa& d, const std::vector<double>* freq) {
    LtTable t;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    auto next = [&](uint32_t s, uint32_t c) {
        return static_cast<uint32_t>(d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + c]);
    };
    t.lo_addr = kLtSmemBase;
    if (static_cast<int32_t>(S) <= kLtPackedMaxStates && !rxg::option("RXG_NO_PACKED")) {
        // packed: the step is a variable shift of one per-byte word (no dependent
        // table load on the state chain), the word read from the lane's own bank
        t.packed = true;
        t.lo_bytes = 256u * 128u;
        t.lo.assign(t.lo_bytes, 0);
        for (uint32_t b = 0; b < 256; ++b) {
            uint32_t w = 0;
            for (uint32_t s = 0; s < S; ++s) w |= (5u * next(s, p.byte_class[b])) << (5u * s);
            for (uint32_t l = 0; l < 32; ++l) std::memcpy(&t.lo[b * 128u + l * 4u], &w, 4);
        }
        for (uint32_t s = 0; s < S; ++s) t.acc_mask |= static_cast<uint32_t>(d.accept[s] != 0) << s;
        t.start = 5u * static_cast<uint32_t>(d.start);
        // a byte class whose step has a cycle of length >= 2 (a permutation of
        // some states): runs of it keep every lookback guess ambiguous
        bool cycles = false;
        for (int32_t c = 0; c < d.n_classes && !cycles; ++c)
            for (uint32_t s0 = 0; s0 < S && !cycles; ++s0) {
                uint32_t x = s0;
                for (uint32_t k = 1; k <= S; ++k) {
                    x = next(x, static_cast<uint32_t>(c));
                    if (x == s0) {
                        cycles = k >= 2;
                        break;
                    }
                }
            }
        if (const char* e = rxg::option("RXG_CHUNK_FN")) cycles = std::atoi(e) != 0;   // force on / off (tests, A/B)
        t.fn_states = cycles ? S : 0u;
    } else if (S <= kLtChunkDirectMaxStates) {
        // direct: rows of 256 four-byte columns at chosen bank offsets
        // direct: rows of 256 four-byte columns at chosen bank offsets; a row's
        // accept flag follows its columns. (Row pairs measured slower here:
        // config (e) 2.96 vs 3.25 TB/s with fewer bank conflicts; unpaired.)
        const uint32_t R = kLtRowBytes;
        const RowPlacement pl = lt_place_groups(freq, S, kLtColBytes, false);
        std::vector<uint32_t> paddr(pl.npairs), addr(S);
        uint32_t cur = kLtSmemBase;
        for (uint32_t q = 0; q < pl.npairs; ++q) {
            paddr[q] = cur + ((pl.pair_off[q] * 4u + 128u - (cur & 127u)) & 127u);
            cur = paddr[q] + R + 4u;
        }
        for (uint32_t r = 0; r < S; ++r) addr[r] = paddr[pl.pair[r]] + 2u * pl.half[r];
        if (cur > 0x10000u) return t;
        t.lo_bytes = align_up(cur - kLtSmemBase, 16);
        t.lo.assign(t.lo_bytes, 0);
        for (uint32_t s = 0; s < S; ++s) {
            for (int b = 0; b < 256; ++b)
                put16(t.lo, addr[s] - kLtSmemBase + kLtColBytes * static_cast<uint32_t>(b), addr[next(s, p.byte_class[b])]);
            put16(t.lo, addr[s] - kLtSmemBase + R, d.accept[s]);
        }
        t.start = addr[static_cast<uint32_t>(d.start)];
        t.acc_off = R;
    } else {
        t.cls = true;
        // range-clamped columns (no class map lookup) when the bytes that matter fit
        uint32_t rx = 0;
        const uint32_t rk = rxg::option("RXG_NO_RANGE_LAYOUT") ? 0 : range_cols(p, 0xFF, 128, &rx, false);
        t.range_x = rx;
        t.range_k = rk;
        auto class_of_col = [&](uint32_t c) -> uint32_t {
            if (!rk) return c;
            return c >= rk ? 0u : p.byte_class[c ^ rx];
        };
        const uint32_t ncols = (rk ? rk + 1 : static_cast<uint32_t>(p.n_classes)) + 1;   // + the accept column
        uint32_t rb = align_up(ncols * 2u, 4u);
        if (((rb / 4u) & 1u) == 0) rb += 4;
        t.row_bytes = rb;
        t.cmap_addr = kLtSmemBase;
        const uint32_t rows_addr = kLtSmemBase + 1024;
        t.lo_bytes = align_up(1024 + S * rb, 16);
        if (kLtSmemBase + t.lo_bytes > 160u * 1024u || S > 0xFFFFu) return t;
        t.lo.assign(t.lo_bytes, 0);
        for (int b = 0; b < 256; ++b) {
            const uint32_t v = rows_addr + static_cast<uint32_t>(p.byte_class[b]) * 2u;
            std::memcpy(&t.lo[static_cast<size_t>(b) * 4], &v, 4);
        }
        std::vector<uint32_t> R(S);
        if (freq) {
            std::vector<double> f2(static_cast<size_t>(S) * 256);
            std::copy(freq->begin(), freq->begin() + static_cast<std::ptrdiff_t>(f2.size()), f2.begin());
            R = number_states(p, d, 0xFF, &f2, S, rows_addr / 4u, rb / 4u, ncols, rx, rk);   // no delimiter column
        } else {
            for (uint32_t s = 0; s < S; ++s) R[s] = s;
        }
        for (uint32_t s = 0; s < S; ++s) {
            for (uint32_t c = 0; c + 1 < ncols; ++c) put16(t.lo, 1024 + R[s] * rb + c * 2u, R[next(s, class_of_col(c))]);
            put16(t.lo, 1024 + R[s] * rb + (ncols - 1) * 2u, d.accept[s]);
        }
        t.start = R[static_cast<uint32_t>(d.start)];
        t.acc_off = (ncols - 1) * 2u;
    }
    t.hi_addr = kLtSmemBase + t.lo_bytes;
    t.hi_bytes = 0;
    t.smem_table_end = kLtSmemBase + t.lo_bytes;
    t.ok = true;
    return t;
}

uint32_t lt_step(const LtTable& t, uint32_t s, uint8_t byte) {
    uint16_t v;
    if (t.cls) {
        uint32_t colabs;
        if (t.range_k) colabs = kLtSmemBase + 1024 + 2u * std::min<uint32_t>(static_cast<uint32_t>(byte) ^ t.range_x, t.range_k);
        else std::memcpy(&colabs, &t.lo[static_cast<size_t>(byte) * 4], 4);
        std::memcpy(&v, &t.lo[s * t.row_bytes + colabs - t.lo_addr], 2);
        return v;
    }
    if (s < kLtAccAddr) std::memcpy(&v, &t.lo[s - t.lo_addr + t.col_bytes * byte], 2);
    else std::memcpy(&v, &t.hi[s - kLtAccAddr + t.col_bytes * byte], 2);
    return v;
}

uint32_t lt_chunk_step(const LtTable& t, uint32_t s, uint8_t byte) {
    if (t.packed) {
        uint32_t w;
        std::memcpy(&w, &t.lo[static_cast<size_t>(byte) * 128u], 4);
        return (w >> (s & 31u)) & 31u;
    }
    uint16_t v;
    if (t.cls) {
        uint32_t colabs;
        if (t.range_k) colabs = kLtSmemBase + 1024 + 2u * std::min<uint32_t>(static_cast<uint32_t>(byte) ^ t.range_x, t.range_k);
        else std::memcpy(&colabs, &t.lo[static_cast<size_t>(byte) * 4], 4);
        std::memcpy(&v, &t.lo[s * t.row_bytes + colabs - t.lo_addr], 2);
        return v;
    }
    std::memcpy(&v, &t.lo[s - t.lo_addr + kLtColBytes * byte], 2);
    return v;
}

bool lt_chunk_accept(const LtTable& t, uint32_t s) {
    if (t.packed) return (t.acc_mask >> ((s & 31u) / 5u)) & 1u;
    uint16_t v;
    const uint32_t addr = t.cls ? kLtSmemBase + 1024 + s * t.row_bytes + t.acc_off : s + t.acc_off;
    std::memcpy(&v, &t.lo[addr - t.lo_addr], 2);
    return v != 0;
}

}  // namespace rxg
