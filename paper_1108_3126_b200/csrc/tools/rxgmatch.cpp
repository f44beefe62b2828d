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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cerrno>
#include <memory>
#include <thread>

#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "rxg.h"

namespace {

constexpr int kMatch = 0, kNoMatch = 1, kError = 2;   // rxvm.cpp:30-32

// RXGMATCH_TIMES=1: phase times on stderr (tools/rxgmatch_e2e.sh)
struct Phases {
    bool on = std::getenv("RXGMATCH_TIMES") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "rxgmatch %-8s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// The candidate buffer: stdin mapped when it is a regular file (no copy; the
// pages fault in on the threads that first touch them), else read in blocks.
struct Input {
    const char* data = "";
    size_t size = 0;
    std::string own;
    void* map = nullptr;
    size_t map_len = 0;

    bool read_stdin() {
        struct stat st {};
        if (fstat(0, &st) == 0 && S_ISREG(st.st_mode) && st.st_size > 0) {
            const off_t at = lseek(0, 0, SEEK_CUR);
            if (at >= 0 && at < st.st_size) {
                void* m = mmap(nullptr, static_cast<size_t>(st.st_size), PROT_READ, MAP_PRIVATE, 0, 0);
                if (m != MAP_FAILED) {
                    madvise(m, static_cast<size_t>(st.st_size), MADV_SEQUENTIAL);
                    map = m;
                    map_len = static_cast<size_t>(st.st_size);
                    data = static_cast<const char*>(m) + at;
                    size = static_cast<size_t>(st.st_size - at);
                    return true;
                }
            }
        }
        constexpr size_t kBlock = 16u << 20;
        for (;;) {
            const size_t at = own.size();
            own.resize(at + kBlock);
            ssize_t got;
            do got = ::read(0, &own[at], kBlock);
            while (got < 0 && errno == EINTR);
            if (got < 0) return false;
            own.resize(at + static_cast<size_t>(got));
            if (got == 0) break;
        }
        data = own.data();
        size = own.size();
        return true;
    }
    ~Input() {
        if (map) munmap(map, map_len);
    }
};

// A run of whole lines [lo, hi) of the buffer.
struct Piece {
    size_t lo = 0, hi = 0;
    uint64_t lines = 0, first = 0, shown = 0;
    std::string out;

    void count(const char* d, size_t n) {
        lines = 0;
        for (size_t at = lo; at < hi;) {
            ++lines;
            const void* nl = std::memchr(d + at, '\n', hi - at);
            at = nl ? static_cast<size_t>(static_cast<const char*>(nl) - d) + 1 : hi;
        }
        (void)n;
    }
    void emit(const char* d, size_t n, const uint8_t* res, uint64_t bad, bool echo) {
        uint64_t k = first;
        for (size_t at = lo; at < hi; ++k) {
            const void* nl = std::memchr(d + at, '\n', hi - at);
            const size_t e = nl ? static_cast<size_t>(static_cast<const char*>(nl) - d) : hi;   // exclusive, '\n' stripped
            const size_t next = nl ? e + 1 : n;
            if (bad != UINT64_MAX && next > bad) return;
            if (res[k]) {
                ++shown;
                if (echo) {
                    out.append(d + at, e - at);
                    out.push_back('\n');
                }
            }
            at = next;
        }
    }
};

template <class F>
void run_pieces(std::vector<Piece>& pieces, F f) {
    if (pieces.size() <= 1) {
        for (Piece& pc : pieces) f(pc);
        return;
    }
    std::vector<std::thread> ts;
    for (Piece& pc : pieces) ts.emplace_back([&f, &pc] { f(pc); });
    for (auto& t : ts) t.join();
}

// Split at line boundaries into about T pieces and count each one's lines.
std::vector<Piece> split_lines(const char* d, size_t n, unsigned T) {
    std::vector<Piece> pieces;
    size_t lo = 0;
    for (unsigned k = 1; k <= T && lo < n; ++k) {
        size_t hi = k == T ? n : std::max(lo, n / T * k);
        if (hi < n) {
            const void* nl = std::memchr(d + hi, '\n', n - hi);
            hi = nl ? static_cast<size_t>(static_cast<const char*>(nl) - d) + 1 : n;
        }
        if (hi <= lo) continue;
        Piece pc;
        pc.lo = lo;
        pc.hi = hi;
        pieces.push_back(std::move(pc));
        lo = hi;
    }
    run_pieces(pieces, [&](Piece& pc) { pc.count(d, n); });
    return pieces;
}

int usage() {
    std::fprintf(stderr, "usage: rxgmatch [--count] [--device N] PATTERN [INPUT...]\n");
    return kError;
}

}  // namespace

int main(int argc, char** argv) {
    Phases ph;
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
    // The device context and tables are built on a second thread while the
    // input is read (creating a CUDA context takes 1-3 s on these boxes, most of
    // the end-to-end time; tools/cuda_init_probe.cpp).
    rxg_heap* h = nullptr;
    int made = RXG_OK;
    std::string made_err;
    std::thread maker([&] {
        made = rxg_heap_create_pattern(pattern.data(), pattern.size(), device, &h);
        if (made != RXG_OK) made_err = rxg_last_error();
    });
    // candidates: the INPUT arguments as lines of one buffer, or stdin
    Input in;
    const bool from_args = i < argc;
    bool read_ok = true;
    if (from_args) {
        for (; i < argc; ++i) {
            if (std::strchr(argv[i], '\n')) {   // an argument is one candidate; keep it a single line
                std::fprintf(stderr, "rxvm: newline inside an INPUT argument is not supported\n");
                read_ok = false;
                break;
            }
            in.own += argv[i];
            in.own += '\n';
        }
        in.data = in.own.data();
        in.size = in.own.size();
    } else {
        read_ok = in.read_stdin();
        if (!read_ok) std::fprintf(stderr, "rxvm: cannot read stdin\n");
    }
    ph.mark("input");
    // line table (std::getline semantics), in pieces on the host threads;
    // faults a mapped input in on many cores at once
    const unsigned T = in.size < (8u << 20) ? 1u : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<Piece> pieces = split_lines(in.data, in.size, T);
    ph.mark("lines");
    maker.join();
    if (made != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", made_err.c_str());
        return kError;
    }
    if (!read_ok) {
        rxg_heap_destroy(h);
        return kError;
    }
    uint64_t lines = 0;
    for (Piece& pc : pieces) {
        pc.first = lines;
        lines += pc.lines;
    }
    ph.mark("create");
    std::unique_ptr<uint8_t[]> res(new uint8_t[lines + 1]);
    uint64_t matches = 0, bad = UINT64_MAX;
    if (rxg_match_batch_host_ex(h, reinterpret_cast<const uint8_t*>(in.data), in.size, '\n', 0, &matches, res.get(),
                                &bad) != RXG_OK) {
        std::fprintf(stderr, "rxvm: %s\n", rxg_last_error());
        rxg_heap_destroy(h);
        return kError;
    }
    ph.mark("match");
    if (ph.on && std::getenv("RXGMATCH_TIMES")[0] == '2') {   // steady-state call cost, for the breakdown only
        rxg_heap* h2 = nullptr;
        rxg_heap_create_pattern(pattern.data(), pattern.size(), device, &h2);
        ph.mark("create2");
        for (int r = 0; r < 2; ++r) {
            rxg_match_batch_host_ex(h2, reinterpret_cast<const uint8_t*>(in.data), in.size, '\n', 0, &matches, res.get(),
                                    &bad);
            ph.mark(r ? "match3" : "match2");
        }
        rxg_heap_destroy(h2);
    }
    rxg_heap_destroy(h);
    ph.mark("destroy");
    // Matching lines before the first line that is not valid UTF-8 (the
    // reference throws there): line k is shown iff its successor starts at or
    // before the bad byte. Each piece formats its own lines; the pieces are
    // written in order.
    const bool echo = !from_args && !count_only;
    run_pieces(pieces, [&](Piece& pc) { pc.emit(in.data, in.size, res.get(), bad, echo); });
    uint64_t shown = 0;
    for (const Piece& pc : pieces) {
        shown += pc.shown;
        if (echo && !pc.out.empty()) std::fwrite(pc.out.data(), 1, pc.out.size(), stdout);
    }
    const bool any = shown > 0;
    if (count_only) std::printf("%llu\n", static_cast<unsigned long long>(shown));
    std::fflush(stdout);
    ph.mark("output");
    if (bad != UINT64_MAX) {
        size_t ls = static_cast<size_t>(bad);   // start of the line holding the bad byte
        while (ls > 0 && in.data[ls - 1] != '\n') --ls;
        std::fprintf(stderr, "rxvm: invalid UTF-8 at byte %llu\n", static_cast<unsigned long long>(bad - ls));
        return kError;
    }
    return any ? kMatch : kNoMatch;
}
