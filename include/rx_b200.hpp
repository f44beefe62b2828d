// rx_b200.hpp — header-only C++ facade with the reference's matcher API
// (arxiv/paper_1108_3126, proj/include/rx) on top of the C ABI in rxg.h.
//
// A caller of the reference hot path
//     rx::Heap h = rx::compile(*rx::parse(pattern));       // regex.hpp:60, heap.hpp:43
//     bool ok   = rx::lockstep_accepts(h, w);               // lockstep.hpp:43
//     bool ok2  = rx::par_accepts(h, w, workers, seed);     // parallel.hpp:102
// switches to this header and links librxg.so; the calls keep their names,
// argument meaning and error behaviour (rx::ParseError with the scalar
// position, std::runtime_error for malformed UTF-8). Matching runs on the
// GPU; there is no CPU fallback. Batch entry points (match_lines) expose the
// `rxvm match` loop (tools/rxvm.cpp:100-112) as one device call.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "rxg.h"
#include "rxg_utf8.hpp"

namespace rx {

using Symbol = char32_t;
using Input = std::u32string;
using InputView = std::u32string_view;
using Addr = int32_t;
inline constexpr Addr null_addr = -1;

struct ParseError : std::runtime_error {
    size_t pos;
    ParseError(size_t p, const std::string& what) : std::runtime_error(what), pos(p) {}
};

// rx::decode_utf8 / encode_utf8 (utf8.hpp): the host-side conversions the
// reference's callers apply around the matcher (rxvm.cpp:85-87). Same
// acceptance rules and error text ("invalid UTF-8 at byte N").
inline std::u32string decode_utf8(std::string_view bytes) {
    std::u32string out;
    out.reserve(bytes.size());
    auto fail = [](size_t at) -> void { throw std::runtime_error("invalid UTF-8 at byte " + std::to_string(at)); };
    for (size_t i = 0; i < bytes.size();) {
        const auto lead = static_cast<unsigned char>(bytes[i]);
        if (lead < 0x80) {
            out.push_back(lead);
            ++i;
            continue;
        }
        const size_t n = (lead & 0xE0) == 0xC0 ? 2 : (lead & 0xF0) == 0xE0 ? 3 : (lead & 0xF8) == 0xF0 ? 4 : 0;
        if (n == 0 || i + n > bytes.size()) fail(i);
        char32_t cp = lead & (n == 2 ? 0x1F : n == 3 ? 0x0F : 0x07);
        for (size_t k = 1; k < n; ++k) {
            const auto b = static_cast<unsigned char>(bytes[i + k]);
            if ((b & 0xC0) != 0x80) fail(i + k);
            cp = (cp << 6) | (b & 0x3F);
        }
        const char32_t least = n == 2 ? 0x80 : n == 3 ? 0x800 : 0x10000;
        if (cp < least || cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) fail(i);
        out.push_back(cp);
        i += n;
    }
    return out;
}

inline std::string encode_utf8(char32_t cp) {
    std::string s;
    rxg::append_utf8(s, cp);
    return s;
}

inline std::string encode_utf8(std::u32string_view text) {
    std::string s;
    s.reserve(text.size());
    for (char32_t cp : text) s += encode_utf8(cp);
    return s;
}

// The facade keeps the validated pattern; compile() lays it out.
struct Regex {
    std::string text;
};
using RegexPtr = std::shared_ptr<const Regex>;

struct Node {
    enum class Kind : uint8_t { Eps, Chr, Alt, Seq, Star };
    Kind kind;
    Symbol sym = 0;
    Addr left = null_addr;
    Addr right = null_addr;
};
static_assert(sizeof(Node) == sizeof(rxg_node), "rx::Node must keep the 16-byte layout");

struct LockstepStats {
    uint64_t enqueued = 0;   // not instrumented on the GPU path (kept for signature parity)
};

struct ParStats {
    uint64_t claims = 0;
    uint64_t launches = 0;
    uint64_t macro_steps = 0;
    uint32_t max_claims_per_node_step = 0;
};

namespace detail {
[[noreturn]] inline void raise(int rc) {
    throw std::runtime_error(std::string(rxg_strerror(rc)) + ": " + rxg_last_error());
}
inline void check(int rc) {
    if (rc != RXG_OK) raise(rc);
}
// Symbols to the UTF-8 bytes the device matches (literals are expanded to
// UTF-8 byte chains, so this is exact for every scalar).
inline std::string narrow(InputView w) { return rxg::symbols_to_bytes(w); }
}  // namespace detail

// The compiled heap (heap.hpp:28-37) plus its device-resident tables. The
// device handle is created on first use on `device` and shared by copies.
class Heap {
public:
    std::vector<Node> nodes;
    std::vector<Addr> knodes;

    Addr root() const { return 0; }
    Addr size() const { return static_cast<Addr>(nodes.size()); }
    bool contains(Addr p) const { return p >= 0 && p < size(); }
    const Node& node(Addr p) const { return nodes[static_cast<size_t>(p)]; }
    Addr knode(Addr p) const { return knodes[static_cast<size_t>(p)]; }

    rxg_heap* device_handle(int device = 0) const {
        if (!dev_ || dev_id_ != device) {
            rxg_heap* h = nullptr;
            detail::check(rxg_heap_create(reinterpret_cast<const rxg_node*>(nodes.data()), knodes.data(), size(),
                                          device, &h));
            dev_ = std::shared_ptr<rxg_heap>(h, rxg_heap_destroy);
            dev_id_ = device;
        }
        return dev_.get();
    }

private:
    mutable std::shared_ptr<rxg_heap> dev_;
    mutable int dev_id_ = -1;
};

inline RegexPtr parse(std::string_view text) {
    int32_t n = 0;
    size_t pos = 0;
    const int rc = rxg_parse_compile(text.data(), text.size(), nullptr, nullptr, 0, &n, &pos);
    if (rc == RXG_EPARSE) throw ParseError(pos, rxg_last_error());
    detail::check(rc);
    return std::make_shared<const Regex>(Regex{std::string(text)});
}

inline Heap compile(const Regex& e) {
    int32_t n = 0;
    size_t pos = 0;
    detail::check(rxg_parse_compile(e.text.data(), e.text.size(), nullptr, nullptr, 0, &n, &pos));
    Heap h;
    h.nodes.resize(static_cast<size_t>(n));
    h.knodes.resize(static_cast<size_t>(n));
    detail::check(rxg_parse_compile(e.text.data(), e.text.size(), reinterpret_cast<rxg_node*>(h.nodes.data()),
                                    h.knodes.data(), n, &n, &pos));
    return h;
}

inline std::string print(const Regex& e) {
    size_t len = 0;
    detail::check(rxg_print(e.text.data(), e.text.size(), nullptr, 0, &len));
    std::string s(len + 1, '\0');
    detail::check(rxg_print(e.text.data(), e.text.size(), s.data(), s.size(), &len));
    s.resize(len);
    return s;
}

inline std::string dump(const Heap& h) {
    size_t len = 0;
    const auto* nodes = reinterpret_cast<const rxg_node*>(h.nodes.data());
    detail::check(rxg_dump(nodes, h.knodes.data(), h.size(), nullptr, 0, &len));
    std::string s(len + 1, '\0');
    detail::check(rxg_dump(nodes, h.knodes.data(), h.size(), s.data(), s.size(), &len));
    s.resize(len);
    return s;
}

inline bool check_knode(const Heap& h) {
    int32_t ok = 0;
    detail::check(rxg_check_knode(reinterpret_cast<const rxg_node*>(h.nodes.data()), h.knodes.data(), h.size(), &ok));
    return ok != 0;
}

// rx::lockstep_accepts (lockstep.hpp:43) on the GPU.
inline bool lockstep_accepts(const Heap& h, InputView w, LockstepStats* stats = nullptr) {
    (void)stats;
    const std::string b = detail::narrow(w);
    int32_t acc = 0;
    detail::check(rxg_match_one(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(),
                                RXG_ENGINE_AUTO, &acc));
    return acc != 0;
}

// rx::par_accepts (parallel.hpp:102): the paper's thread-per-node protocol on
// the GPU. `workers` / `seed` only perturbed CPU interleavings in the
// reference; results are schedule independent (Theorem 4).
inline bool par_accepts(const Heap& h, InputView w, unsigned workers, uint64_t seed, ParStats* stats = nullptr) {
    (void)workers;
    (void)seed;
    const std::string b = detail::narrow(w);
    int32_t acc = 0;
    int rc = rxg_match_one(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(), RXG_ENGINE_ROUNDS,
                           &acc);
    if (rc == RXG_EUNSUPPORTED)   // non-ASCII literals: the thread-per-node bitset form of the same scheme
        rc = rxg_match_one(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(), RXG_ENGINE_PERNODE,
                           &acc);
    detail::check(rc);
    if (stats) *stats = ParStats{};
    return acc != 0;
}

// The `rxvm match` loop as one call: per-line results for a '\n'-separated
// UTF-8 buffer (std::getline semantics). Returns the number of matching lines.
inline uint64_t match_lines(const Heap& h, std::string_view text, std::vector<uint8_t>* per_line = nullptr,
                            uint64_t* utf8_first_bad = nullptr) {
    uint64_t count = 0;
    if (per_line) {
        uint64_t lines = 0;
        for (char c : text) lines += c == '\n';
        if (!text.empty() && text.back() != '\n') ++lines;
        per_line->assign(lines + 1, 0);
    }
    // utf8_first_bad: the device UTF-8 check of every line, fused into the same pass
    // (UINT64_MAX when every line decodes; else the buffer offset decode_utf8 names)
    detail::check(rxg_match_batch_host_ex(h.device_handle(), reinterpret_cast<const uint8_t*>(text.data()),
                                          text.size(), '\n', 0, &count, per_line ? per_line->data() : nullptr,
                                          utf8_first_bad));
    if (per_line && !per_line->empty()) per_line->pop_back();
    return count;
}

}  // namespace rx
