// Shared-memory bank model of the line kernel's table step (k_lines_tma,
// class layouts) on a config's text: per warp-wide LDS, wavefronts = the most
// distinct 4-byte words any one bank is asked for. Scores table layouts on the
// host before they are built. Tool, not product.
//
//   bank_sim CONFIG [HOT...]   (CONFIG a-e; HOT: hot-row counts to model)
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "frontend.hpp"
#include "lines_tma.hpp"
#include "program.hpp"
#include "synth.hpp"

using namespace rxg;

int main(int argc, char** argv) {
    const char cfg = argc > 1 ? argv[1][0] : 'd';
    const std::string pat = synth_pattern(cfg);
    Program p = build_program(compile(parse(pat)));
    Dfa d;
    if (!build_dfa(p, 16384, d)) return 1;
    minimize_dfa(d);
    const uint64_t n = 64ull << 20;
    std::vector<uint8_t> text(n);
    const uint64_t got = synth_input(cfg, 0, text.data(), n);
    text.resize(got);
    const std::vector<double> freq = lt_sample_freq(p, d, '\n', text.data(), std::min<uint64_t>(got, 1u << 20));
    LtTable t = make_lines_tma_table(p, d, '\n', &freq);
    std::printf("config %c: %d states, %d classes, cls %d range_k %u range_x %u row_bytes %u acc_shift %u\n", cfg,
                d.n_states, d.n_classes, t.cls, t.range_k, t.range_x, t.row_bytes, t.acc_shift);
    const uint32_t rows_addr = kLtSmemBase + 1024;
    auto col_of = [&](uint8_t b) { return std::min<uint32_t>(b ^ t.range_x, t.range_k); };
    // walk: warps of 32 lanes, lane l at range (w*32 + l) * chunk, SKIP entry
    const uint32_t chunk = 7168, steps = 2048;
    const uint32_t warps = static_cast<uint32_t>(std::min<uint64_t>(400, got / (32ull * chunk)));
    std::vector<std::vector<uint32_t>> S(warps * 32), B(warps * 32);
    std::map<uint32_t, uint64_t> visits;
    for (uint32_t w = 0; w < warps; ++w)
        for (uint32_t l = 0; l < 32; ++l) {
            const uint64_t at = (static_cast<uint64_t>(w) * 32 + l) * chunk;
            uint32_t s = at == 0 ? t.start : t.skip;
            auto& sv = S[w * 32 + l];
            auto& bv = B[w * 32 + l];
            for (uint32_t k = 0; k < steps; ++k) {
                const uint8_t b = text[at + k];
                sv.push_back(s);
                bv.push_back(b);
                ++visits[s];
                s = lt_step(t, s, b);
            }
        }
    std::vector<std::pair<uint64_t, uint32_t>> hot;
    for (auto& kv : visits) hot.push_back({kv.second, kv.first});
    std::sort(hot.rbegin(), hot.rend());
    const double total = static_cast<double>(warps) * 32 * steps;
    double cum = 0;
    std::printf("hottest rows (share, cumulative):");
    for (size_t i = 0; i < std::min<size_t>(hot.size(), 40); ++i) {
        cum += hot[i].first / total;
        if (i < 8 || i % 8 == 7) std::printf(" %zu:%.3f", i + 1, cum);
    }
    std::printf("\n");
    auto score = [&](auto word_of) {
        double wf = 0;
        for (uint32_t w = 0; w < warps; ++w)
            for (uint32_t k = 0; k < steps; ++k) {
                std::set<uint32_t> words[32];
                for (uint32_t l = 0; l < 32; ++l) {
                    const uint32_t wd = word_of(S[w * 32 + l][k], B[w * 32 + l][k], l);
                    words[wd & 31].insert(wd);
                }
                size_t m = 0;
                for (auto& x : words) m = std::max(m, x.size());
                wf += static_cast<double>(m);
            }
        return wf / (static_cast<double>(warps) * steps);
    };
    std::printf("current layout: %.3f wavefronts / warp step\n",
                score([&](uint32_t s, uint8_t b, uint32_t) { return (rows_addr + s * t.row_bytes + 2 * col_of(b)) >> 2; }));
    // Local search on the row numbering (the builder's greedy placement is the
    // start): swap two main rows when the pairwise same-bank mass
    // sum_{s != s'} P(s, c) P(s', c') [bank(s, c) == bank(s', c')] drops.
    {
        const uint32_t rbw = t.row_bytes / 4, base = rows_addr / 4;
        const uint32_t nmain = static_cast<uint32_t>(d.n_states) + 2;
        std::vector<std::array<double, 32>> Hs(nmain);   // word-offset histogram per current row (offset 0 row)
        for (auto& h : Hs) h.fill(0.0);
        for (uint32_t w = 0; w < warps * 32; ++w)
            for (uint32_t k = 0; k < steps; ++k) {
                const uint32_t s = S[w][k];
                if (s < nmain) Hs[s][(col_of(B[w][k]) / 2) & 31u] += 1.0 / total;
            }
        std::vector<uint32_t> row(nmain);
        for (uint32_t r = 0; r < nmain; ++r) row[r] = r;
        auto off = [&](uint32_t r) { return (base + r * rbw) & 31u; };
        auto pair_cost = [&](uint32_t a, uint32_t oa, uint32_t b, uint32_t ob) {
            double c = 0;
            for (uint32_t k = 0; k < 32; ++k) c += Hs[a][k] * Hs[b][(k + oa + 64 - ob) & 31u];
            return c;
        };
        auto cost_of = [&](uint32_t a, uint32_t oa, uint32_t skip) {   // row a at offset oa against all others
            double c = 0;
            for (uint32_t b = 0; b < nmain; ++b)
                if (b != a && b != skip) c += pair_cost(a, oa, b, off(row[b]));
            return c;
        };
        for (int pass = 0; pass < 4; ++pass) {
            int swaps = 0;
            for (uint32_t a = 0; a < nmain; ++a)
                for (uint32_t b = a + 1; b < nmain; ++b) {
                    const uint32_t oa = off(row[a]), ob = off(row[b]);
                    if (oa == ob) continue;
                    const double now = cost_of(a, oa, b) + cost_of(b, ob, a);
                    const double sw = cost_of(a, ob, b) + cost_of(b, oa, a);
                    if (sw < now - 1e-12) {
                        std::swap(row[a], row[b]);
                        ++swaps;
                    }
                }
            std::printf("local search pass %d: %d swaps\n", pass, swaps);
            if (!swaps) break;
        }
        std::printf("renumbered layout: %.3f wavefronts / warp step\n",
                    score([&](uint32_t s, uint8_t b, uint32_t) {
                        const uint32_t r = s < nmain ? row[s] : s;
                        return (rows_addr + r * t.row_bytes + 2 * col_of(b)) >> 2;
                    }));
    }
    // Absorbing hot state: lanes in a state whose every non-delimiter byte
    // leads back to itself skip the table load (predicated off). (Config (d)'s
    // accepting state is absorbing only over the pattern's alphabet: bytes of
    // class 0 lead to the dead state, so an exact skip also needs a per-word
    // alphabet test; the two compares alone measured +2% on (d).)
    {
        const uint32_t h0 = hot[0].second;
        bool absorbing = true;
        for (int b = 0; b < 256 && absorbing; ++b)
            if (b != '\n' && lt_step(t, h0, static_cast<uint8_t>(b)) != h0) absorbing = false;
        std::printf("hottest row %u (share %.3f) absorbing: %d\n", h0, hot[0].first / total, absorbing);
        if (absorbing) {
            double wf = 0;
            for (uint32_t w = 0; w < warps; ++w)
                for (uint32_t k = 0; k < steps; ++k) {
                    std::set<uint32_t> words[32];
                    for (uint32_t l = 0; l < 32; ++l) {
                        const uint32_t s0 = S[w * 32 + l][k];
                        const uint8_t b = B[w * 32 + l][k];
                        if (s0 == h0 && b != '\n') continue;
                        const uint32_t wd = (rows_addr + s0 * t.row_bytes + 2 * col_of(b)) >> 2;
                        words[wd & 31].insert(wd);
                    }
                    size_t m = 0;
                    for (auto& x : words) m = std::max(m, x.size());
                    wf += static_cast<double>(m);
                }
            std::printf("absorbing row skipped: %.3f wavefronts / warp step\n", wf / (static_cast<double>(warps) * steps));
        }
    }
    // Hot rows lane-replicated over a compact column set (the columns with a
    // sampled share >= 0.5% in the hot rows), the rest through the cold rows.
    for (size_t H : {8u, 16u, 24u, 32u}) {
        std::map<uint32_t, uint32_t> hidx;
        for (size_t j = 0; j < std::min(H, hot.size()); ++j) hidx[hot[j].second] = static_cast<uint32_t>(j);
        std::map<uint32_t, double> colw;
        double hs = 0;
        for (uint32_t w = 0; w < warps * 32; ++w)
            for (uint32_t k = 0; k < steps; ++k)
                if (hidx.count(S[w][k])) {
                    colw[col_of(B[w][k])] += 1;
                    hs += 1;
                }
        std::map<uint32_t, uint32_t> cidx;
        for (auto& kv : colw)
            if (kv.second >= 0.005 * hs) cidx[kv.first] = static_cast<uint32_t>(cidx.size());
        const uint32_t cw = static_cast<uint32_t>((cidx.size() + 1) / 2);
        std::printf("hot %2zu compact cols %zu (%u words): %.1f KB, %.3f wavefronts\n", H, cidx.size(), cw, H * cw * 128 / 1024.0,
                    score([&](uint32_t s0, uint8_t b, uint32_t l) {
                        auto it = hidx.find(s0);
                        auto ic = cidx.find(col_of(b));
                        if (it != hidx.end() && ic != cidx.end()) return 0x20000u + (it->second * cw + ic->second / 2) * 32 + l;
                        return (rows_addr + s0 * t.row_bytes + 2 * col_of(b)) >> 2;
                    }));
    }
    // Paired rows: two states share each column word (u16 halves), rows of
    // (k + 1) words at an odd stride; states paired in hotness order.
    {
        std::map<uint32_t, uint32_t> pair_of;
        uint32_t np = 0;
        for (size_t j = 0; j < hot.size(); ++j) pair_of[hot[j].second] = static_cast<uint32_t>(j / 2);
        np = static_cast<uint32_t>((hot.size() + 1) / 2);
        uint32_t pw = t.range_k + 1;
        if ((pw & 1u) == 0) ++pw;
        std::printf("paired rows (%u pairs, %u words each): %.3f wavefronts / warp step\n", np, pw,
                    score([&](uint32_t s, uint8_t b, uint32_t) {
                        auto it = pair_of.find(s);
                        const uint32_t pr = it != pair_of.end() ? it->second : np + s;
                        return 0x1000u + pr * pw + col_of(b);
                    }));
    }
    for (int i = 2; i < argc; ++i) {
        const size_t H = static_cast<size_t>(std::atoi(argv[i]));
        std::map<uint32_t, uint32_t> hidx;
        for (size_t j = 0; j < std::min(H, hot.size()); ++j) hidx[hot[j].second] = static_cast<uint32_t>(j);
        const uint32_t hot_base = 0x20000;   // lane-replicated rows: word (h * cols + col) * 32 + lane
        const uint32_t cw = (t.range_k + 2) / 2;
        double share = 0;
        for (size_t j = 0; j < std::min(H, hot.size()); ++j) share += hot[j].first / total;
        std::printf("hot %3zu (%.3f of steps, %6.1f KB replicated): %.3f wavefronts\n", H, share,
                    H * cw * 128 / 1024.0, score([&](uint32_t s, uint8_t b, uint32_t l) {
                        auto it = hidx.find(s);
                        if (it != hidx.end()) return hot_base + (it->second * cw + col_of(b) / 2) * 32 + l;
                        return (rows_addr + s * t.row_bytes + 2 * col_of(b)) >> 2;
                    }));
    }
    return 0;
}
