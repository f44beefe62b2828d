// rxgmatch — the `rxvm match` front end (reference tools/rxvm.cpp:74-115) on
// the GPU batch path.
//
//   rxgmatch [--count] [--device N] PATTERN [INPUT...]
//
// With INPUT arguments: exit 0 if any input matches, 1 if none, 2 on error.
// Without: every stdin line (std::getline: '\n' stripped, '\r' kept, a final
// unterminated line counts) is a candidate; matching lines are echoed in
// order; same exit codes. Lines are matched in one device pass
// (rxg_match_batch_host_ex) instead of one engine call per line, with the
// device UTF-8 check fused into it. As in the reference, a line that is not
// valid UTF-8 is an error (exit 2, "rxvm: invalid UTF-8 at byte N" with N
// inside that line, the runtime_error of decode_utf8) after the matching
// lines before it have been printed.
#include <algorithm>
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
    std::vector<uint8_t> res(lines + 1, 0);
    uint64_t matches = 0, bad = UINT64_MAX;
    if (rxg_match_batch_host_ex(h, reinterpret_cast<const uint8_t*>(buf.data()), buf.size(), '\n', 0, &matches,
                                res.data(), &bad) != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", rxg_last_error());
        rxg_heap_destroy(h);
        return kError;
    }
    rxg_heap_destroy(h);
    // first line that is not valid UTF-8 (the reference throws there)
    size_t bad_line = lines;
    if (bad != UINT64_MAX) bad_line = static_cast<size_t>(std::upper_bound(starts.begin(), starts.end(), bad) - starts.begin()) - 1;
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
        std::fprintf(stderr, "rxvm: invalid UTF-8 at byte %llu\n",
                     static_cast<unsigned long long>(bad - starts[bad_line]));
        return kError;
    }
    return any ? kMatch : kNoMatch;
}
