// Absolute-address shared-memory layout for the TMA line kernel
// (kernels_lines_tma.cu). Rows are raw-byte indexed u16 entries holding the
// absolute shared address of the next row, so one IMAD + one LDS advance a
// string by one byte.
//
//   [0x400 .. lo_addr)        stage-ring slots (2 KB, 1 KB aligned)
//   [lo_addr .. 0x8000)       main rows: DFA states 0..S-1, SKIP, VOID (absorbing,
//                             for lanes whose range lies past the input)
//   [0x8000]                  START_A (copy of the start row, entered on an
//                             accepted line end; bit 15 set)
//   [0x8000 + 548 ..)         tail copies of states 0..S-1, TERM_A, TERM_R
//   [..]                      remaining stage slots, then the mbarriers
#include <cstring>

#include "lines_tma.hpp"

namespace rxg {

namespace {

void put16(std::vector<uint8_t>& img, uint32_t off, uint32_t v) {
    const uint16_t x = static_cast<uint16_t>(v);
    std::memcpy(&img[off], &x, 2);
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

}  // namespace

LtTable make_lines_tma_table(const Program& p, const Dfa& d, uint8_t delim) {
    LtTable t;
    const uint32_t S = static_cast<uint32_t>(d.n_states);
    const uint32_t R = kLtRowBytes;
    const uint32_t main_bytes = (S + 2) * R;   // + SKIP + VOID
    if (main_bytes + kLtSmemBase > kLtAccAddr) return t;
    const uint32_t upper_bytes = (S + 3) * R;
    if (kLtAccAddr + upper_bytes > 0x10000u) return t;
    t.lo_addr = (kLtAccAddr - main_bytes) & ~15u;
    t.lo_bytes = align_up(kLtAccAddr - t.lo_addr, 16);
    t.hi_addr = kLtAccAddr;
    t.hi_bytes = align_up(upper_bytes, 16);
    t.lo.assign(t.lo_bytes, 0);
    t.hi.assign(t.hi_bytes, 0);
    auto main_row = [&](uint32_t s) { return t.lo_addr + s * R; };
    auto tail_row = [&](uint32_t s) { return kLtAccAddr + R + s * R; };
    t.start = main_row(static_cast<uint32_t>(d.start));
    t.skip = main_row(S);
    t.void_row = main_row(S + 1);
    t.tail_delta = tail_row(0) - main_row(0);
    t.term_acc = tail_row(S);
    t.term_rej = tail_row(S + 1);
    auto next = [&](uint32_t s, int b) {
        return static_cast<uint32_t>(d.next[static_cast<size_t>(s) * static_cast<size_t>(d.n_classes) + p.byte_class[b]]);
    };
    for (uint32_t s = 0; s < S; ++s) {
        const bool acc = d.accept[s] != 0;
        for (int b = 0; b < 256; ++b) {
            const uint32_t mo = main_row(s) - t.lo_addr + 2u * static_cast<uint32_t>(b);
            const uint32_t to = tail_row(s) - kLtAccAddr + 2u * static_cast<uint32_t>(b);
            if (b == delim) {
                put16(t.lo, mo, acc ? kLtAccAddr : t.start);
                put16(t.hi, to, acc ? t.term_acc : t.term_rej);
            } else {
                put16(t.lo, mo, main_row(next(s, b)));
                put16(t.hi, to, tail_row(next(s, b)));
            }
        }
    }
    for (int b = 0; b < 256; ++b) {
        put16(t.lo, t.skip - t.lo_addr + 2u * static_cast<uint32_t>(b), b == delim ? t.start : t.skip);
        put16(t.lo, t.void_row - t.lo_addr + 2u * static_cast<uint32_t>(b), t.void_row);
        put16(t.hi, t.term_acc - kLtAccAddr + 2u * static_cast<uint32_t>(b), t.term_acc);
        put16(t.hi, t.term_rej - kLtAccAddr + 2u * static_cast<uint32_t>(b), t.term_rej);
    }
    std::memcpy(&t.hi[0], &t.lo[t.start - t.lo_addr], R);   // START_A = start row

    // stage slots: first in the gap below the main rows, then after the upper rows
    int slot = 0;
    for (uint32_t a = kLtSmemBase; a + kLtStageBytes <= t.lo_addr && slot < kLtWarps * kLtStages; a += kLtStageBytes)
        t.stage_addr[slot++] = a;
    uint32_t a = align_up(kLtAccAddr + t.hi_bytes, 1024);
    for (; slot < kLtWarps * kLtStages; ++slot, a += kLtStageBytes) t.stage_addr[slot] = a;
    t.bar_addr = align_up(a, 8);
    t.smem_bytes = t.bar_addr + kLtWarps * kLtStages * 8 - kLtSmemBase;
    t.ok = true;
    return t;
}

uint32_t lt_step(const LtTable& t, uint32_t s, uint8_t byte) {
    uint16_t v;
    if (s < kLtAccAddr) std::memcpy(&v, &t.lo[s - t.lo_addr + 2u * byte], 2);
    else std::memcpy(&v, &t.hi[s - kLtAccAddr + 2u * byte], 2);
    return v;
}

}  // namespace rxg
