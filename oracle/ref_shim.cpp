// TEST INFRASTRUCTURE — C shim over the UNMODIFIED reference library
// (arxiv/paper_1108_3126, /root/reference/proj/src/*.cpp), compiled from its
// sources by oracle/Makefile into oracle/_ref/librxref.so. Used only by
// tests/ (golden generation, parity cross-checks) and by bench.py's
// reference arm / cpu_baseline. Nothing here is product code.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "rx/crosscheck.hpp"
#include "rx/heap.hpp"
#include "rx/lockstep.hpp"
#include "rx/parallel.hpp"
#include "rx/pwpi.hpp"
#include "rx/regex.hpp"
#include "rx/utf8.hpp"

namespace {

int put_str(const std::string& s, char* out, size_t cap) {
    if (out && cap) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), n);
        out[n] = '\0';
    }
    return static_cast<int>(s.size());
}

struct Prepared {
    std::vector<rx::Input> strings;
};

rx::AddrSet to_set(const int32_t* s, int n) { return rx::AddrSet(s, s + n); }

int from_set(const rx::AddrSet& s, int32_t* out) {
    int k = 0;
    for (rx::Addr a : s) out[k++] = a;
    return k;
}

}  // namespace

extern "C" {

// 0 ok; 1 ParseError (err_pos set); 2 other exception (msg set)
int ref_parse_compile(const char* pat, size_t len, void* nodes, int32_t* knodes, int32_t cap, int32_t* n_out,
                      size_t* err_pos, char* msg, size_t msgcap) {
    try {
        rx::Heap h = rx::compile(*rx::parse(std::string_view(pat, len)));
        *n_out = h.size();
        const int32_t n = std::min(cap, h.size());
        static_assert(sizeof(rx::Node) == 16, "rx::Node layout");
        if (nodes) std::memcpy(nodes, h.nodes.data(), static_cast<size_t>(n) * sizeof(rx::Node));
        if (knodes) std::memcpy(knodes, h.knodes.data(), static_cast<size_t>(n) * sizeof(int32_t));
        return 0;
    } catch (const rx::ParseError& e) {
        if (err_pos) *err_pos = e.pos;
        put_str(e.what(), msg, msgcap);
        return 1;
    } catch (const std::exception& e) {
        put_str(e.what(), msg, msgcap);
        return 2;
    }
}

int ref_print(const char* pat, size_t len, char* out, size_t cap) {
    try {
        return put_str(rx::print(rx::parse(std::string_view(pat, len))), out, cap);
    } catch (...) {
        return -1;
    }
}

int ref_dump(const char* pat, size_t len, char* out, size_t cap) {
    try {
        return put_str(rx::dump(rx::compile(*rx::parse(std::string_view(pat, len)))), out, cap);
    } catch (...) {
        return -1;
    }
}

void* ref_compile(const char* pat, size_t len) {
    try {
        return new rx::Heap(rx::compile(*rx::parse(std::string_view(pat, len))));
    } catch (...) {
        return nullptr;
    }
}

void ref_free(void* h) { delete static_cast<rx::Heap*>(h); }

int ref_accepts(void* h, const uint32_t* w, size_t n, uint64_t* enqueued) {
    rx::LockstepStats st;
    const bool ok = rx::lockstep_accepts(*static_cast<rx::Heap*>(h),
                                         rx::InputView(reinterpret_cast<const char32_t*>(w), n), &st);
    if (enqueued) *enqueued = st.enqueued;
    return ok ? 1 : 0;
}

int ref_par_accepts(void* h, const uint32_t* w, size_t n, unsigned workers, uint64_t seed, uint64_t* claims,
                    uint64_t* launches, uint32_t* max_claims) {
    rx::ParStats st;
    const bool ok = rx::par_accepts(*static_cast<rx::Heap*>(h),
                                    rx::InputView(reinterpret_cast<const char32_t*>(w), n), workers, seed, &st);
    if (claims) *claims = st.claims;
    if (launches) *launches = st.launches;
    if (max_claims) *max_claims = st.max_claims_per_node_step;
    return ok ? 1 : 0;
}

int ref_evolve(void* h, const int32_t* s, int n, int32_t* out) {
    return from_set(rx::evolve(*static_cast<rx::Heap*>(h), to_set(s, n)), out);
}

int ref_step_char(void* h, const int32_t* s, int n, uint32_t a, int32_t* out) {
    try {
        return from_set(rx::step_char(*static_cast<rx::Heap*>(h), to_set(s, n), static_cast<char32_t>(a)), out);
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int ref_eps_reaches_null(void* h, const int32_t* s, int n) {
    return rx::eps_reaches_null(*static_cast<rx::Heap*>(h), to_set(s, n)) ? 1 : 0;
}

int ref_trace(void* h, const uint32_t* w, size_t n, char* out, size_t cap) {
    return put_str(rx::lockstep_trace(*static_cast<rx::Heap*>(h), rx::InputView(reinterpret_cast<const char32_t*>(w), n)),
                   out, cap);
}

// Splits a byte buffer into strings exactly like rxvm's std::getline loop
// (delimiter >= 0) or at a fixed stride, decoding each with decode_utf8.
// Returns nullptr on invalid UTF-8.
void* ref_prepare(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride) {
    auto* p = new Prepared;
    try {
        uint64_t at = 0;
        if (delimiter < 0) {
            for (; at + stride <= len; at += stride)
                p->strings.push_back(rx::decode_utf8(std::string_view(reinterpret_cast<const char*>(text + at), stride)));
        } else {
            while (at < len) {
                const void* hit = std::memchr(text + at, delimiter, len - at);
                const uint64_t end = hit ? static_cast<uint64_t>(static_cast<const uint8_t*>(hit) - text) : len;
                p->strings.push_back(
                    rx::decode_utf8(std::string_view(reinterpret_cast<const char*>(text + at), end - at)));
                at = end + 1;
            }
        }
    } catch (...) {
        delete p;
        return nullptr;
    }
    return p;
}

uint64_t ref_prepared_count(void* p) { return static_cast<Prepared*>(p)->strings.size(); }
void ref_prepared_free(void* p) { delete static_cast<Prepared*>(p); }

// rx::lockstep_accepts over every prepared string on `threads` threads
// (static interleaved partition, the crosscheck pattern crosscheck.cpp:121).
uint64_t ref_run(void* heap, void* prep, uint8_t* results, int threads) {
    const rx::Heap& h = *static_cast<rx::Heap*>(heap);
    const auto& ss = static_cast<Prepared*>(prep)->strings;
    threads = std::max(1, threads);
    std::atomic<uint64_t> total{0};
    auto work = [&](int t) {
        uint64_t c = 0;
        for (size_t k = static_cast<size_t>(t); k < ss.size(); k += static_cast<size_t>(threads)) {
            const bool ok = rx::lockstep_accepts(h, ss[k]);
            if (results) results[k] = ok ? 1 : 0;
            c += ok;
        }
        total += c;
    };
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    return total.load();
}

// Every regex with <= max_nodes AST nodes over the given ASCII alphabet
// (crosscheck.cpp:13-34), printed canonically, '\n'-separated.
int ref_enumerate(int max_nodes, const char* alphabet, char* out, size_t cap) {
    std::vector<rx::Symbol> al;
    for (const char* c = alphabet; *c; ++c) al.push_back(static_cast<unsigned char>(*c));
    std::string s;
    for (const rx::RegexPtr& e : rx::enumerate_regexes(static_cast<size_t>(max_nodes), al)) {
        s += rx::print(e);
        s += '\n';
    }
    return put_str(s, out, cap);
}

// Seeded random regexes (crosscheck.cpp:52-67), one per line.
int ref_random_regexes(int count, int max_nodes, const char* alphabet, uint64_t seed, char* out, size_t cap) {
    std::vector<rx::Symbol> al;
    for (const char* c = alphabet; *c; ++c) al.push_back(static_cast<unsigned char>(*c));
    std::mt19937_64 rng(seed);
    std::string s;
    for (int k = 0; k < count; ++k) {
        const size_t nodes = 1 + static_cast<size_t>(rng() % static_cast<uint64_t>(max_nodes));
        s += rx::print(rx::random_regex(nodes, al, rng));
        s += '\n';
    }
    return put_str(s, out, cap);
}

// rx::decode_utf8 (utf8.cpp:16-46): -1 when it decodes, else N from its
// runtime_error "invalid UTF-8 at byte N".
int64_t ref_decode_utf8_error(const uint8_t* s, size_t n) {
    try {
        (void)rx::decode_utf8(std::string_view(reinterpret_cast<const char*>(s), n));
        return -1;
    } catch (const std::runtime_error& e) {
        const std::string m = e.what();
        const size_t at = m.rfind(' ');
        return at == std::string::npos ? -2 : static_cast<int64_t>(std::stoull(m.substr(at + 1)));
    }
}

}  // extern "C"
