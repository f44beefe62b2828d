// Synthetic workloads. See synth.hpp.
#include "synth.hpp"

#include <algorithm>
#include <cstring>
#include <random>
#include <stdexcept>

namespace rxg {

std::vector<std::string> synth_keywords(int total_len, uint64_t seed) {
    std::mt19937_64 r(seed);
    std::vector<std::string> kws;
    int total = 0;
    while (total < total_len) {
        int len = 3 + static_cast<int>(r() % 6);
        len = std::min(len, total_len - total);
        std::string k;
        for (int i = 0; i < len; ++i) k += static_cast<char>('a' + r() % 26);
        kws.push_back(std::move(k));
        total += len;
    }
    return kws;
}

namespace {

std::string alt_of(const std::vector<std::string>& items) {
    std::string s;
    for (size_t i = 0; i < items.size(); ++i) {
        if (i) s += '|';
        s += items[i];
    }
    return s;
}

const char* kS9 = "(a|b|c|d|e|f|g|h| )";

std::string s27() {
    std::string s = "(";
    for (char c = 'a'; c <= 'z'; ++c) {
        s += c;
        s += '|';
    }
    s += " )";
    return s;
}

constexpr uint64_t kLinesC = 10'000'000;
constexpr uint64_t kSizeA = 1ull << 20;
constexpr uint64_t kSizeB = 32'000'000;
constexpr uint64_t kSizeD = 1ull << 30;
constexpr uint64_t kSizeE = 1ull << 28;

uint64_t canonical_seed(char c) {
    switch (c) {
    case 'a': case 'A': return 1;
    case 'c': return 3;
    case 'd': return 11;
    case 'e': return 5;
    default: return 0;
    }
}

}  // namespace

std::string synth_pattern(char config) {
    switch (config) {
    case 'a':
    case 'A':
        return "(a|b)*abb";
    case 'b': {
        std::string s;
        for (int i = 0; i < 32; ++i) s += "(a|())";
        for (int i = 0; i < 32; ++i) s += "a";
        return s;
    }
    case 'c':
        return std::string("(") + kS9 + "*(ERROR|WARN|FAIL)" + kS9 + "*)*";
    case 'd': {
        const std::string s = s27();
        return "(" + s + "*(" + alt_of(synth_keywords(457, 7)) + ")" + s + "*)*";
    }
    case 'e': {
        std::vector<std::string> items = synth_keywords(2018, 7);
        for (char c = 'a'; c <= 'z'; ++c) items.emplace_back(1, c);
        items.emplace_back(" ");
        return "(" + alt_of(items) + ")*abb";
    }
    default:
        throw std::invalid_argument("unknown config");
    }
}

uint64_t synth_input_size(char config) {
    switch (config) {
    case 'a': case 'A': return kSizeA;
    case 'b': return kSizeB;
    case 'c': return kLinesC * 116;   // upper bound: 110 chars + keyword (<=5) + '\n'
    case 'd': return kSizeD;
    case 'e': return kSizeE;
    default: throw std::invalid_argument("unknown config");
    }
}

uint64_t synth_input(char config, uint64_t seed, uint8_t* out, uint64_t n) {
    std::mt19937_64 r(seed ? seed : canonical_seed(config));
    switch (config) {
    case 'a':
    case 'A': {
        for (uint64_t i = 0; i < n; ++i) out[i] = (r() & 1) ? 'a' : 'b';
        if (n >= 3) std::memcpy(out + n - 3, "abb", 3);
        if (config == 'A' && n >= 1) out[n - 1] = 'a';
        return n;
    }
    case 'b': {
        std::memset(out, 'a', n);
        return n;
    }
    case 'c': {
        static const char* kw[3] = {"ERROR", "WARN", "FAIL"};
        static const char alpha[] = "abcdefgh ";
        uint64_t at = 0;
        char line[128];
        for (uint64_t k = 0; k < kLinesC; ++k) {
            const int len = 90 + static_cast<int>(r() % 21);
            uint64_t bits = r();
            for (int i = 0; i < len; ++i) {
                if (i % 20 == 0 && i) bits = r();
                line[i] = alpha[bits % 9];
                bits /= 9;
            }
            int total = len;
            if (r() % 4 == 0) {
                const char* w = kw[r() % 3];
                const int wl = static_cast<int>(std::strlen(w));
                const int pos = static_cast<int>(r() % static_cast<uint64_t>(len + 1));
                std::memmove(line + pos + wl, line + pos, static_cast<size_t>(len - pos));
                std::memcpy(line + pos, w, static_cast<size_t>(wl));
                total += wl;
            }
            line[total++] = '\n';
            if (at + static_cast<uint64_t>(total) > n) break;
            std::memcpy(out + at, line, static_cast<size_t>(total));
            at += static_cast<uint64_t>(total);
        }
        return at;
    }
    case 'd': {
        // ~1 KiB lines of lowercase words (2-9 letters) separated by single
        // spaces; the final line is truncated so the stream is exactly n bytes.
        uint64_t at = 0;
        std::string line;
        while (at < n) {
            line.clear();
            for (;;) {
                const int wl = 2 + static_cast<int>(r() % 8);
                const size_t need = line.size() + (line.empty() ? 0 : 1) + static_cast<size_t>(wl);
                if (need > 1023) break;
                if (!line.empty()) line += ' ';
                for (int i = 0; i < wl; ++i) line += static_cast<char>('a' + r() % 26);
            }
            line += '\n';
            const uint64_t room = n - at;
            if (line.size() > room) {
                line.resize(static_cast<size_t>(room));
                line.back() = '\n';
            }
            std::memcpy(out + at, line.data(), line.size());
            at += line.size();
        }
        return at;
    }
    case 'e': {
        for (uint64_t i = 0; i < n; ++i)
            out[i] = (r() % 6 == 0) ? ' ' : static_cast<uint8_t>('a' + r() % 26);
        if (n >= 3) std::memcpy(out + n - 3, "abb", 3);
        return n;
    }
    default:
        throw std::invalid_argument("unknown config");
    }
}

}  // namespace rxg
