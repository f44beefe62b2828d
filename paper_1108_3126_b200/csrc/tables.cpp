// Shared-memory DFA images. See tables.hpp.
#include "tables.hpp"

#include <cstring>
#include <stdexcept>

namespace rxg {

namespace {

// Raw-byte rows cost 257 entries per state; above this budget the rows are
// indexed by byte class instead (one extra class-map load per byte).
constexpr uint32_t kDirectBudget = 96 * 1024;

void put(KTable& t, uint32_t off, uint32_t v) {
    if (t.esize == 2) {
        if (v > 0xFFFFu) throw std::logic_error("table entry overflow");
        const uint16_t x = static_cast<uint16_t>(v);
        std::memcpy(&t.img[off], &x, 2);
    } else {
        std::memcpy(&t.img[off], &v, 4);
    }
}

uint32_t get(const KTable& t, uint32_t off) {
    if (t.esize == 2) {
        uint16_t x;
        std::memcpy(&x, &t.img[off], 2);
        return x;
    }
    uint32_t v;
    std::memcpy(&v, &t.img[off], 4);
    return v;
}

uint32_t col_of(const KTable& t, uint8_t byte) { return t.cls ? t.img[t.cls_off + byte] : byte; }

uint32_t pad16(uint32_t x) { return (x + 15u) & ~15u; }

}  // namespace

uint32_t ktable_step(const KTable& t, uint32_t off, uint8_t byte) {
    return get(t, off + col_of(t, byte) * static_cast<uint32_t>(t.esize));
}

uint32_t ktable_accept(const KTable& t, uint32_t off) {
    return get(t, off + static_cast<uint32_t>(t.ncols) * static_cast<uint32_t>(t.esize));
}

KTable make_plain_table(const Program& p, const Dfa& d, bool force_class) {
    KTable t;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    t.n_states = d.n_states;
    t.accept = d.accept;
    t.cls = force_class || S * 257u * 2u > kDirectBudget;
    t.ncols = t.cls ? p.n_classes : 256;
    for (int es : {2, 4}) {
        t.esize = es;
        t.row_bytes = static_cast<uint32_t>(t.ncols + 1) * static_cast<uint32_t>(es);
        if (es == 4 || S * t.row_bytes <= 0x10000u) break;
    }
    const uint32_t rows = S * t.row_bytes;
    t.cls_off = t.cls ? pad16(rows) : 0;
    t.img.assign(pad16(t.cls ? t.cls_off + 256 : rows), 0);
    if (t.cls)
        for (int b = 0; b < 256; ++b) t.img[t.cls_off + static_cast<uint32_t>(b)] = p.byte_class[b];
    auto row = [&](int32_t s) { return static_cast<uint32_t>(s) * t.row_bytes; };
    for (int32_t s = 0; s < d.n_states; ++s) {
        for (int c = 0; c < t.ncols; ++c) {
            const int32_t cls = t.cls ? c : p.byte_class[c];
            const int32_t nx = d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + static_cast<size_t>(cls)];
            put(t, row(s) + static_cast<uint32_t>(c * t.esize), row(nx));
        }
        put(t, row(s) + static_cast<uint32_t>(t.ncols * t.esize), d.accept[static_cast<size_t>(s)]);
        t.state_of_row.push_back(static_cast<uint32_t>(s));
    }
    t.start = row(d.start);
    t.dead = row(d.dead);
    return t;
}

KTable make_line_table(const Program& p, const Dfa& d, uint8_t delim, bool force_class) {
    KTable t;
    t.delimited = true;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    t.n_states = d.n_states;
    t.accept = d.accept;
    // rows: S main + SKIP, START_A, S tail + TERM_A + TERM_R
    const uint32_t nrows_est = 2 * S + 4;
    t.cls = force_class || nrows_est * 257u * 2u > kDirectBudget;
    t.ncols = t.cls ? p.n_classes + 1 : 256;
    t.delim_col = t.cls ? static_cast<uint32_t>(p.n_classes) : delim;
    for (int es : {2, 4}) {
        t.esize = es;
        t.row_bytes = static_cast<uint32_t>(t.ncols + 1) * static_cast<uint32_t>(es);
        const uint32_t main_bytes = (S + 1) * t.row_bytes;
        t.acc_shift = 0;
        while ((1u << t.acc_shift) < main_bytes) ++t.acc_shift;
        t.acc_row = 1u << t.acc_shift;
        const uint32_t tail_base = t.acc_row + t.row_bytes;
        t.tail_delta = tail_base;
        t.term_acc = tail_base + S * t.row_bytes;
        t.term_rej = t.term_acc + t.row_bytes;
        if (es == 4 || t.term_rej <= 0xFFFFu) break;
    }
    const uint32_t rows_end = t.term_rej + t.row_bytes;
    t.cls_off = t.cls ? pad16(rows_end) : 0;
    t.img.assign(pad16(t.cls ? t.cls_off + 256 : rows_end), 0);
    if (t.cls) {
        for (int b = 0; b < 256; ++b) t.img[t.cls_off + static_cast<uint32_t>(b)] = p.byte_class[b];
        t.img[t.cls_off + delim] = static_cast<uint8_t>(t.delim_col);
    }
    auto mrow = [&](int32_t s) { return static_cast<uint32_t>(s) * t.row_bytes; };
    auto trow = [&](int32_t s) { return t.tail_delta + static_cast<uint32_t>(s) * t.row_bytes; };
    t.skip = S * t.row_bytes;
    t.start = mrow(d.start);
    t.dead = mrow(d.dead);
    const uint32_t es = static_cast<uint32_t>(t.esize);
    const uint32_t endc = static_cast<uint32_t>(t.ncols) * es;
    auto next_of = [&](int32_t s, int c) -> int32_t {
        const int32_t cls = t.cls ? c : p.byte_class[c];
        return d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + static_cast<size_t>(cls)];
    };
    for (int32_t s = 0; s < d.n_states; ++s) {
        const bool acc = d.accept[static_cast<size_t>(s)] != 0;
        for (int c = 0; c < t.ncols; ++c) {
            const uint32_t cb = static_cast<uint32_t>(c) * es;
            if (static_cast<uint32_t>(c) == t.delim_col) {
                put(t, mrow(s) + cb, acc ? t.acc_row : t.start);
                put(t, trow(s) + cb, acc ? t.term_acc : t.term_rej);
            } else {
                const int32_t nx = next_of(s, c);
                put(t, mrow(s) + cb, mrow(nx));
                put(t, trow(s) + cb, trow(nx));
            }
        }
        put(t, mrow(s) + endc, acc);
        put(t, trow(s) + endc, acc);
        t.state_of_row.push_back(static_cast<uint32_t>(s));
    }
    // SKIP: swallow until the first delimiter, then start a line (uncounted).
    for (int c = 0; c < t.ncols; ++c)
        put(t, t.skip + static_cast<uint32_t>(c) * es, static_cast<uint32_t>(c) == t.delim_col ? t.start : t.skip);
    // START_A: same transitions as the start state.
    std::memcpy(&t.img[t.acc_row], &t.img[t.start], t.row_bytes);
    // terminal rows absorb everything; their accept column records the line result
    for (int c = 0; c < t.ncols; ++c) {
        put(t, t.term_acc + static_cast<uint32_t>(c) * es, t.term_acc);
        put(t, t.term_rej + static_cast<uint32_t>(c) * es, t.term_rej);
    }
    put(t, t.term_acc + endc, 1);
    put(t, t.term_rej + endc, 0);
    return t;
}

}  // namespace rxg
