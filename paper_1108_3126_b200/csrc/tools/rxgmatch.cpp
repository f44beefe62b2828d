// rxgmatch — the `rxvm match` front end (reference tools/rxvm.cpp:74-115) on
// the GPU batch path.
//
//   rxgmatch [--count] [--device N] PATTERN [INPUT...]
//
// With INPUT arguments: exit 0 if any input matches, 1 if none, 2 on error.
// Without: every stdin line (std::getline: '\n' stripped, '\r' kept, a final
// unterminated line counts) is a candidate; matching lines are echoed in
// order; same exit codes. Lines are matched in one device pass
// (rxg_match_batch_host) instead of one engine call per line. As in the
// reference, a line that is not valid UTF-8 is an error (exit 2) after the
// matching lines before it have been printed.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <iterator>
#include <string>
#include <vector>

#include "rxg.h"

namespace {

constexpr int kMatch = 0, kNoMatch = 1, kError = 2;   // rxvm.cpp:30-32

// Offset of the first invalid UTF-8 sequence in [p, p+n), or n.
size_t utf8_invalid_at(const unsigned char* p, size_t n) {
    size_t i = 0;
    while (i < n) {
        const unsigned b0 = p[i];
        if (b0 < 0x80) {
            ++i;
            continue;
        }
        int len;
        unsigned cp;
        if ((b0 & 0xE0) == 0xC0) { len = 2; cp = b0 & 0x1F; }
        else if ((b0 & 0xF0) == 0xE0) { len = 3; cp = b0 & 0x0F; }
        else if ((b0 & 0xF8) == 0xF0) { len = 4; cp = b0 & 0x07; }
        else return i;
        if (i + static_cast<size_t>(len) > n) return i;
        for (int k = 1; k < len; ++k) {
            if ((p[i + k] & 0xC0) != 0x80) return i;
            cp = (cp << 6) | (p[i + k] & 0x3F);
        }
        static const unsigned kMin[5] = {0, 0, 0x80, 0x800, 0x10000};
        if (cp < kMin[len] || cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return i;
        i += static_cast<size_t>(len);
    }
    return n;
}

int usage() {
    std::fprintf(stderr, "usage: rxgmatch [--count] [--device N] PATTERN [INPUT...]\n");
    return kError;
}

}  // namespace

int main(int argc, char** argv) {
    bool count_only = false;
    int device = 0;
    int i = 1;
    for (; i < argc && argv[i][0] == '-' && argv[i][1] == '-'; ++i) {
        if (!std::strcmp(argv[i], "--count")) count_only = true;
        else if (!std::strcmp(argv[i], "--device") && i + 1 < argc) device = std::atoi(argv[++i]);
        else return usage();
    }
    if (i >= argc) return usage();
    const std::string pattern = argv[i++];
    int32_t n = 0;
    size_t pos = 0;
    if (rxg_parse_compile(pattern.data(), pattern.size(), nullptr, nullptr, 0, &n, &pos) != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", rxg_last_error());
        return kError;
    }
    rxg_heap* h = nullptr;
    if (rxg_heap_create_pattern(pattern.data(), pattern.size(), device, &h) != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", rxg_last_error());
        return kError;
    }
    // candidates: the INPUT arguments as lines of one buffer, or stdin
    std::string buf;
    const bool from_args = i < argc;
    if (from_args) {
        for (; i < argc; ++i) {
            if (std::strchr(argv[i], '\n')) {   // an argument is one candidate; keep it a single line
                std::fprintf(stderr, "rxvm: newline inside an INPUT argument is not supported\n");
                rxg_heap_destroy(h);
                return kError;
            }
            buf += argv[i];
            buf += '\n';
        }
    } else {
        buf.assign(std::istreambuf_iterator<char>(std::cin), std::istreambuf_iterator<char>());
    }
    // line table (std::getline semantics)
    std::vector<size_t> starts;
    for (size_t at = 0; at < buf.size();) {
        starts.push_back(at);
        const void* nl = std::memchr(buf.data() + at, '\n', buf.size() - at);
        at = nl ? static_cast<size_t>(static_cast<const char*>(nl) - buf.data()) + 1 : buf.size();
    }
    const size_t lines = starts.size();
    auto line_end = [&](size_t k) {   // exclusive end, the '\n' stripped
        if (k + 1 < lines) return starts[k + 1] - 1;
        return buf.back() == '\n' ? buf.size() - 1 : buf.size();
    };
    // first line that is not valid UTF-8 (the reference throws there)
    size_t bad_line = lines;
    {
        const size_t bad = utf8_invalid_at(reinterpret_cast<const unsigned char*>(buf.data()), buf.size());
        if (bad < buf.size())
            for (size_t k = 0; k < lines; ++k)
                if (starts[k] <= bad && (k + 1 == lines || bad < starts[k + 1])) bad_line = k;
    }
    std::vector<uint8_t> res(lines + 1, 0);
    uint64_t matches = 0;
    if (rxg_match_batch_host(h, reinterpret_cast<const uint8_t*>(buf.data()), buf.size(), '\n', 0, &matches,
                             res.data()) != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", rxg_last_error());
        rxg_heap_destroy(h);
        return kError;
    }
    rxg_heap_destroy(h);
    bool any = false;
    uint64_t shown = 0;
    for (size_t k = 0; k < lines && k < bad_line; ++k) {
        if (!res[k]) continue;
        any = true;
        ++shown;
        if (!from_args && !count_only) {
            const size_t e = line_end(k);
            std::fwrite(buf.data() + starts[k], 1, e - starts[k], stdout);
            std::fputc('\n', stdout);
        }
    }
    if (count_only) std::printf("%llu\n", static_cast<unsigned long long>(shown));
    if (bad_line < lines) {
        std::fflush(stdout);
        std::fprintf(stderr, "rxvm: invalid UTF-8 in line %zu\n", bad_line + 1);
        return kError;
    }
    return any ? kMatch : kNoMatch;
}
