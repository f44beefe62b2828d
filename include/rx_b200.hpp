// rx_b200.hpp — header-only C++ facade with the reference's matcher API
// (arxiv/paper_1108_3126, proj/include/rx) on top of the C ABI in rxg.h.
//
// A caller of the reference hot path
//     rx::Heap h = rx::compile(*rx::parse(pattern));       // regex.hpp:60, heap.hpp:43
//     bool ok   = rx::lockstep_accepts(h, w, &stats);      // lockstep.hpp:43
//     bool ok2  = rx::par_accepts(h, w, workers, seed);     // parallel.hpp:102
// switches to this header and links librxg.so; the calls keep their names,
// argument meaning, instrumentation and error behaviour (rx::ParseError with
// the scalar position, std::runtime_error for malformed UTF-8,
// std::invalid_argument from step_char). Covered surface:
//   regex.hpp     Regex AST, eps/chr/star/seq/alt, cmp/equal, ast_size, parse, print
//   heap.hpp      Node, Heap, compile, dump, check_knode, addr_name
//   pwpi.hpp      eps_successors, char_successor (the Fig. 3 micro steps)
//   lockstep.hpp  AddrSet, LockstepStats, evolve, evolve_ordered, eps_reaches_null,
//                 step_char, lockstep_accepts, lockstep_trace, format
//   parallel.hpp  ParState, end_of_input, par_task, ParStats, RoundOutcome,
//                 ParallelMatcher (macro_step, accepts), par_accepts, par_report
// Whole-string matching and the paper's protocol (par_task, the rounds of a
// macro step) run on the GPU; there is no CPU fallback for them. The
// one-set / one-symbol functions (evolve, step_char, eps_reaches_null) are
// host code in librxg, like the front end. Batch entry points (match_lines)
// expose the `rxvm match` loop (tools/rxvm.cpp:100-112) as one device call.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <memory>
#include <optional>
#include <set>
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
    for (char32_t cp : text) rxg::append_utf8(s, cp);
    return s;
}

namespace detail {
[[noreturn]] inline void raise(int rc) {
    throw std::runtime_error(std::string(rxg_strerror(rc)) + ": " + rxg_last_error());
}
inline void check(int rc) {
    if (rc != RXG_OK) raise(rc);
}
// Symbols to the UTF-8 bytes the device matches (literals are expanded to
// UTF-8 byte chains, so this is exact for every scalar; values that are not
// scalars become 0xFF, which no literal matches).
inline std::string narrow(InputView w) { return rxg::symbols_to_bytes(w); }
}  // namespace detail

// ── syntax (regex.hpp:22-66) ────────────────────────────────────────────

struct Regex;
using RegexPtr = std::shared_ptr<const Regex>;

// Abstract syntax: eps | a | e* | e1 e2 | e1|e2 (regex.hpp:26-32).
struct Regex {
    enum class Kind : uint8_t { Eps, Chr, Star, Seq, Alt };
    Kind kind;
    Symbol sym = 0;   // Chr
    RegexPtr left;    // Star body; Seq/Alt left
    RegexPtr right;   // Seq/Alt right
};

inline RegexPtr eps() {
    static const RegexPtr e = std::make_shared<Regex>(Regex{Regex::Kind::Eps, 0, nullptr, nullptr});
    return e;
}
inline RegexPtr chr(Symbol a) { return std::make_shared<Regex>(Regex{Regex::Kind::Chr, a, nullptr, nullptr}); }
inline RegexPtr star(RegexPtr body) {
    return std::make_shared<Regex>(Regex{Regex::Kind::Star, 0, std::move(body), nullptr});
}
inline RegexPtr seq(RegexPtr l, RegexPtr r) {
    return std::make_shared<Regex>(Regex{Regex::Kind::Seq, 0, std::move(l), std::move(r)});
}
inline RegexPtr alt(RegexPtr l, RegexPtr r) {
    return std::make_shared<Regex>(Regex{Regex::Kind::Alt, 0, std::move(l), std::move(r)});
}

// Structural three-way comparison (regex.cpp:34-49).
inline int cmp(const RegexPtr& a, const RegexPtr& b);
inline int cmp(const Regex& a, const Regex& b) {
    if (a.kind != b.kind) return a.kind < b.kind ? -1 : 1;
    switch (a.kind) {
    case Regex::Kind::Eps: return 0;
    case Regex::Kind::Chr: return a.sym == b.sym ? 0 : (a.sym < b.sym ? -1 : 1);
    case Regex::Kind::Star: return cmp(a.left, b.left);
    case Regex::Kind::Seq:
    case Regex::Kind::Alt:
        if (int c = cmp(a.left, b.left)) return c;
        return cmp(a.right, b.right);
    }
    return 0;
}
inline int cmp(const RegexPtr& a, const RegexPtr& b) { return a.get() == b.get() ? 0 : cmp(*a, *b); }
inline bool equal(const RegexPtr& a, const RegexPtr& b) { return cmp(a, b) == 0; }

// regex.cpp:51-63
inline size_t ast_size(const Regex& e) {
    switch (e.kind) {
    case Regex::Kind::Eps:
    case Regex::Kind::Chr: return 1;
    case Regex::Kind::Star: return 1 + ast_size(*e.left);
    case Regex::Kind::Seq:
    case Regex::Kind::Alt: return 1 + ast_size(*e.left) + ast_size(*e.right);
    }
    return 0;
}

namespace detail {
// The tree as the C ABI's node array (children first; shared subtrees are
// written once per use, so the array is a tree). Returns the root index.
inline int32_t flatten(const Regex& e, std::vector<rxg_ast_node>& out) {
    rxg_ast_node n{static_cast<uint8_t>(e.kind), {0, 0, 0}, static_cast<uint32_t>(e.sym), -1, -1};
    if (e.kind == Regex::Kind::Star) {
        n.left = flatten(*e.left, out);
    } else if (e.kind == Regex::Kind::Seq || e.kind == Regex::Kind::Alt) {
        n.left = flatten(*e.left, out);
        n.right = flatten(*e.right, out);
    }
    out.push_back(n);
    return static_cast<int32_t>(out.size()) - 1;
}
inline RegexPtr unflatten(const std::vector<rxg_ast_node>& a, int32_t i) {
    const rxg_ast_node& n = a[static_cast<size_t>(i)];
    switch (static_cast<Regex::Kind>(n.kind)) {
    case Regex::Kind::Eps: return eps();
    case Regex::Kind::Chr: return chr(n.sym);
    case Regex::Kind::Star: return star(unflatten(a, n.left));
    case Regex::Kind::Seq: return seq(unflatten(a, n.left), unflatten(a, n.right));
    case Regex::Kind::Alt: return alt(unflatten(a, n.left), unflatten(a, n.right));
    }
    throw std::logic_error("bad tree node");
}
}  // namespace detail

// rx::parse (regex.hpp:60): ParseError(pos) / std::runtime_error (bad UTF-8).
inline RegexPtr parse(std::string_view text) {
    int32_t n = 0, root = -1;
    size_t pos = 0;
    const int rc = rxg_parse_ast(text.data(), text.size(), nullptr, 0, &n, &root, &pos);
    if (rc == RXG_EPARSE) throw ParseError(pos, rxg_last_error());
    if (rc == RXG_EUTF8) throw std::runtime_error(rxg_last_error());
    detail::check(rc);
    std::vector<rxg_ast_node> a(static_cast<size_t>(n));
    detail::check(rxg_parse_ast(text.data(), text.size(), a.data(), n, &n, &root, &pos));
    return detail::unflatten(a, root);
}

// rx::print (regex.hpp:65): canonical form, parse(print(e)) == e.
inline std::string print(const Regex& e) {
    std::vector<rxg_ast_node> a;
    const int32_t root = detail::flatten(e, a);
    size_t len = 0;
    detail::check(rxg_print_ast(a.data(), static_cast<int32_t>(a.size()), root, nullptr, 0, &len));
    std::string s(len + 1, '\0');
    detail::check(rxg_print_ast(a.data(), static_cast<int32_t>(a.size()), root, s.data(), s.size(), &len));
    s.resize(len);
    return s;
}
inline std::string print(const RegexPtr& e) { return print(*e); }

// ── heap (heap.hpp:14-70) ───────────────────────────────────────────────

struct Node {
    enum class Kind : uint8_t { Eps, Chr, Alt, Seq, Star };
    Kind kind = Kind::Eps;
    uint8_t pad_[3] = {0, 0, 0};
    Symbol sym = 0;
    Addr left = null_addr;
    Addr right = null_addr;
};
static_assert(sizeof(Node) == sizeof(rxg_node), "rx::Node must keep the 16-byte layout");

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

    const rxg_node* c_nodes() const { return reinterpret_cast<const rxg_node*>(nodes.data()); }

    rxg_heap* device_handle(int device = 0) const {
        if (!dev_ || dev_id_ != device) {
            rxg_heap* h = nullptr;
            detail::check(rxg_heap_create(c_nodes(), knodes.data(), size(), device, &h));
            dev_ = std::shared_ptr<rxg_heap>(h, rxg_heap_destroy);
            dev_id_ = device;
        }
        return dev_.get();
    }

private:
    mutable std::shared_ptr<rxg_heap> dev_;
    mutable int dev_id_ = -1;
};

// rx::compile (heap.hpp:43): breadth-first addresses, knode laws.
inline Heap compile(const Regex& e) {
    std::vector<rxg_ast_node> a;
    const int32_t root = detail::flatten(e, a);
    const int32_t n = static_cast<int32_t>(a.size());
    Heap h;
    h.nodes.resize(a.size());
    h.knodes.resize(a.size());
    int32_t got = 0;
    detail::check(rxg_compile_ast(a.data(), n, root, reinterpret_cast<rxg_node*>(h.nodes.data()), h.knodes.data(), n,
                                  &got));
    return h;
}

inline std::string addr_name(Addr p) { return p == null_addr ? "null" : "p" + std::to_string(p); }

inline std::string dump(const Heap& h) {
    size_t len = 0;
    detail::check(rxg_dump(h.c_nodes(), h.knodes.data(), h.size(), nullptr, 0, &len));
    std::string s(len + 1, '\0');
    detail::check(rxg_dump(h.c_nodes(), h.knodes.data(), h.size(), s.data(), s.size(), &len));
    s.resize(len);
    return s;
}

inline bool check_knode(const Heap& h) {
    int32_t ok = 0;
    detail::check(rxg_check_knode(h.c_nodes(), h.knodes.data(), h.size(), &ok));
    return ok != 0;
}

// ── Fig. 3 micro steps (pwpi.hpp:27-34) ─────────────────────────────────

inline std::vector<Addr> eps_successors(const Heap& h, Addr p) {
    const Node& n = h.node(p);
    switch (n.kind) {
    case Node::Kind::Alt: return {n.left, n.right};
    case Node::Kind::Seq: return {n.left};
    case Node::Kind::Star: return {n.left, h.knode(p)};
    case Node::Kind::Eps: return {h.knode(p)};
    case Node::Kind::Chr: return {};
    }
    return {};
}

inline std::optional<Addr> char_successor(const Heap& h, Addr p, Symbol a) {
    const Node& n = h.node(p);
    if (n.kind == Node::Kind::Chr && n.sym == a) return h.knode(p);
    return std::nullopt;
}

// ── lockstep (lockstep.hpp:14-49) ───────────────────────────────────────

using AddrSet = std::set<Addr>;

struct LockstepStats {
    uint64_t enqueued = 0;   // addresses pushed onto evolve worklists
};

namespace detail {
inline std::vector<Addr> vec(const AddrSet& s) { return std::vector<Addr>(s.begin(), s.end()); }
}  // namespace detail

inline std::vector<Addr> evolve_ordered(const Heap& h, const AddrSet& s, LockstepStats* stats = nullptr) {
    const std::vector<Addr> in = detail::vec(s);
    std::vector<Addr> out(static_cast<size_t>(h.size()) + 1);
    int32_t n = 0;
    uint64_t enq = 0;
    detail::check(rxg_evolve(h.c_nodes(), h.knodes.data(), h.size(), in.data(), static_cast<int32_t>(in.size()),
                             out.data(), &n, &enq));
    if (stats) stats->enqueued += enq;
    out.resize(static_cast<size_t>(n));
    return out;
}

inline AddrSet evolve(const Heap& h, const AddrSet& s, LockstepStats* stats = nullptr) {
    const std::vector<Addr> o = evolve_ordered(h, s, stats);
    return AddrSet(o.begin(), o.end());
}

inline bool eps_reaches_null(const Heap& h, const AddrSet& s) {
    const std::vector<Addr> in = detail::vec(s);
    int32_t r = 0;
    detail::check(
        rxg_eps_reaches_null(h.c_nodes(), h.knodes.data(), h.size(), in.data(), static_cast<int32_t>(in.size()), &r));
    return r != 0;
}

inline AddrSet step_char(const Heap& h, const AddrSet& s, Symbol a) {
    const std::vector<Addr> in = detail::vec(s);
    std::vector<Addr> out(in.size() + 1);
    int32_t n = 0;
    const int rc = rxg_step_char(h.c_nodes(), h.knodes.data(), h.size(), in.data(), static_cast<int32_t>(in.size()),
                                 static_cast<uint32_t>(a), out.data(), &n);
    if (rc == RXG_EINVAL) throw std::invalid_argument(rxg_last_error());
    detail::check(rc);
    return AddrSet(out.begin(), out.begin() + n);
}

inline std::string format(const AddrSet& s) {
    std::string out = "{";
    bool first = true;
    for (Addr p : s) {
        if (!first) out += ",";
        first = false;
        out += addr_name(p);
    }
    return out + "}";
}

namespace detail {
inline bool host_walk_enqueued(const Heap& h, InputView w, LockstepStats* stats) {
    AddrSet s{h.root()};
    for (Symbol a : w) {
        s = step_char(h, evolve(h, s, stats), a);
        if (s.empty()) return false;
    }
    return s.count(null_addr) || eps_reaches_null(h, s);
}
}  // namespace detail

// rx::lockstep_accepts (lockstep.hpp:43) on the GPU. With `stats`, the run
// goes through the literal §8 protocol kernel, whose claims per macro step
// are exactly the addresses evolve enqueues; LockstepStats.enqueued is
// accumulated like the reference's. (Patterns with non-ASCII literals, which
// that byte-comparing kernel does not take, count with the host set
// functions beside the GPU answer.)
inline bool lockstep_accepts(const Heap& h, InputView w, LockstepStats* stats = nullptr) {
    const std::string b = detail::narrow(w);
    int32_t acc = 0;
    if (stats) {
        rxg_match_stats ms{};
        const int rc = rxg_match_one_stats(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(),
                                           &acc, &ms);
        if (rc == RXG_OK) {
            stats->enqueued += ms.enqueued;
            return acc != 0;
        }
        if (rc != RXG_EUNSUPPORTED) detail::raise(rc);
        LockstepStats host;
        detail::host_walk_enqueued(h, w, &host);
        stats->enqueued += host.enqueued;
    }
    detail::check(rxg_match_one(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(),
                                RXG_ENGINE_AUTO, &acc));
    return acc != 0;
}

namespace detail {
inline std::string format_seq(const std::vector<Addr>& s) {
    std::string out = "{";
    for (size_t i = 0; i < s.size(); ++i) {
        if (i) out += ",";
        out += addr_name(s[i]);
    }
    return out + "}";
}
}  // namespace detail

// `{p0} =eps=> {p2,p4} =a=> {p3}` per consumed symbol, then the
// end-of-input acceptance line (lockstep.cpp:108-122).
inline std::string lockstep_trace(const Heap& h, InputView w) {
    std::string out;
    AddrSet s{h.root()};
    for (Symbol a : w) {
        const std::vector<Addr> evolved = evolve_ordered(h, s);
        AddrSet next = step_char(h, AddrSet(evolved.begin(), evolved.end()), a);
        out += format(s) + " =eps=> " + detail::format_seq(evolved) + " =" + encode_utf8(a) + "=> " + format(next) +
               "\n";
        s = std::move(next);
        if (s.empty()) break;
    }
    const bool ok = !s.empty() && (s.count(null_addr) || eps_reaches_null(h, s));
    out += format(s) + (ok ? " accept\n" : " reject\n");
    return out;
}

// ── the paper's §8 protocol (parallel.hpp:14-106) ───────────────────────

// c[i] == t: scheduled; c[i] == -t: claimed; n[j] == t+1: scheduled for the
// next macro step; stale values are inert (parallel.hpp:14-22). The state
// lives with the caller; par_task and the rounds of a macro step run on the
// GPU over a copy of it.
struct ParState {
    explicit ParState(size_t nodes) : c(nodes), n(nodes), claim_count(nodes) {}

    std::vector<std::atomic<int64_t>> c, n;
    int64_t t = 1;
    std::atomic<bool> more_c{false};
    std::atomic<bool> any_n{false};
    std::atomic<bool> accept_pending{false};
    std::atomic<bool> accept_next{false};
    std::vector<std::atomic<uint32_t>> claim_count;

    void schedule_root(Addr root) { c[static_cast<size_t>(root)].store(t); }
    AddrSet current_schedule() const {
        AddrSet s;
        for (size_t i = 0; i < c.size(); ++i)
            if (c[i].load() == t) s.insert(static_cast<Addr>(i));
        return s;
    }
    AddrSet next_schedule() const {
        AddrSet s;
        for (size_t j = 0; j < n.size(); ++j)
            if (n[j].load() == t + 1) s.insert(static_cast<Addr>(j));
        return s;
    }
    AddrSet claimed() const {
        AddrSet s;
        for (size_t i = 0; i < c.size(); ++i)
            if (c[i].load() == -t) s.insert(static_cast<Addr>(i));
        return s;
    }
    void swap_step() {   // parallel.cpp:40-48
        c.swap(n);
        t += 1;
        accept_pending.store(accept_next.load());
        accept_next.store(false);
        more_c.store(false);
        any_n.store(false);
        for (auto& cc : claim_count) cc.store(0);
    }
};

inline constexpr Symbol end_of_input = 0xFFFFFFFF;   // not a Unicode scalar

namespace detail {
// Runs one device call of the protocol on a plain copy of `st`.
template <class F>
inline void with_par_state(ParState& st, F f) {
    const size_t N = st.c.size();
    std::vector<int64_t> c(N), n(N);
    std::vector<uint32_t> cc(N);
    for (size_t i = 0; i < N; ++i) {
        c[i] = st.c[i].load();
        n[i] = st.n[i].load();
        cc[i] = st.claim_count[i].load();
    }
    rxg_par_state ps{c.data(), n.data(), cc.data(), st.t, st.more_c.load(), st.any_n.load(), st.accept_pending.load(),
                     st.accept_next.load()};
    f(ps);
    for (size_t i = 0; i < N; ++i) {
        st.c[i].store(c[i]);
        st.n[i].store(n[i]);
        st.claim_count[i].store(cc[i]);
    }
    st.more_c.store(ps.more_c != 0);
    st.any_n.store(ps.any_n != 0);
    st.accept_pending.store(ps.accept_pending != 0);
    st.accept_next.store(ps.accept_next != 0);
}
}  // namespace detail

// par_task (parallel.cpp:50-78) on the device: claim node i (CAS t -> -t),
// then forward the schedule along its unlabeled steps, or test the symbol.
inline void par_task(const Heap& h, ParState& st, Addr i, Symbol a) {
    detail::with_par_state(st, [&](rxg_par_state& ps) {
        detail::check(rxg_par_task(h.device_handle(), &ps, i, static_cast<uint32_t>(a)));
    });
}

struct ParStats {
    uint64_t claims = 0;
    uint64_t launches = 0;               // barrier-delimited rounds
    uint64_t macro_steps = 0;
    uint32_t max_claims_per_node_step = 0;
    std::vector<size_t> schedule_sizes;  // nodes scheduled per macro step
};

struct RoundOutcome {
    AddrSet claimed;
    AddrSet next;
    bool accept_pending = false;
    bool accept_next = false;
    uint64_t launches = 0;
};

// ParallelMatcher (parallel.hpp:80-99). The rounds of a macro step run in
// one GPU launch (one thread per node, CTA barriers between rounds), so
// `workers` and `seed` — which set the CPU pool size and perturbed its
// interleavings in the reference — do not change anything observable:
// results are schedule independent (Theorem 4).
class ParallelMatcher {
public:
    explicit ParallelMatcher(unsigned workers, uint64_t seed = 0) : workers_(workers == 0 ? 1 : workers), seed_(seed) {}
    ParallelMatcher(const ParallelMatcher&) = delete;
    ParallelMatcher& operator=(const ParallelMatcher&) = delete;

    unsigned workers() const { return workers_; }

    // parallel.cpp:156-178
    RoundOutcome macro_step(const Heap& h, ParState& st, std::optional<Symbol> a, ParStats* stats = nullptr) {
        RoundOutcome out;
        if (stats) {
            ++stats->macro_steps;
            stats->schedule_sizes.push_back(st.current_schedule().size());
        }
        uint64_t launches = 0;
        detail::with_par_state(st, [&](rxg_par_state& ps) {
            detail::check(rxg_par_run_rounds(h.device_handle(), &ps, static_cast<uint32_t>(a.value_or(end_of_input)),
                                             &launches));
        });
        out.launches = launches;
        if (stats) stats->launches += launches;
        out.claimed = st.claimed();
        out.next = st.next_schedule();
        out.accept_pending = st.accept_pending.load();
        out.accept_next = st.accept_next.load();
        if (stats)
            for (const auto& cc : st.claim_count) {
                const uint32_t k = cc.load();
                stats->claims += k;
                stats->max_claims_per_node_step = std::max(stats->max_claims_per_node_step, k);
            }
        if (a) st.swap_step();
        return out;
    }

    // parallel.cpp:180-190, one device call per macro step. par_accepts runs
    // the whole string in one launch instead.
    bool accepts(const Heap& h, InputView w, ParStats* stats = nullptr) {
        ParState st(static_cast<size_t>(h.size()));
        st.schedule_root(h.root());
        for (Symbol a : w) {
            const RoundOutcome out = macro_step(h, st, a, stats);
            if (out.next.empty() && !out.accept_next) return false;
        }
        macro_step(h, st, std::nullopt, stats);
        return st.accept_pending.load();
    }

private:
    unsigned workers_;
    uint64_t seed_;
};

// rx::par_accepts (parallel.hpp:102): the whole string through the literal
// protocol in one GPU launch (k_rounds), with the reference's counters.
// Patterns with non-ASCII literals (that kernel compares bytes) run the same
// protocol one macro step per launch on symbols.
inline bool par_accepts(const Heap& h, InputView w, unsigned workers, uint64_t seed, ParStats* stats = nullptr) {
    const std::string b = detail::narrow(w);
    int32_t acc = 0;
    std::vector<uint32_t> sched(stats ? b.size() + 1 : 0);
    rxg_match_stats ms{};
    ms.schedule = stats ? sched.data() : nullptr;
    const int rc =
        rxg_match_one_stats(h.device_handle(), reinterpret_cast<const uint8_t*>(b.data()), b.size(), &acc, &ms);
    if (rc == RXG_EUNSUPPORTED) {
        ParallelMatcher m(workers, seed);
        return m.accepts(h, w, stats);
    }
    detail::check(rc);
    if (stats) {
        stats->claims += ms.claims;
        stats->launches += ms.launches;
        stats->macro_steps += ms.macro_steps;
        stats->max_claims_per_node_step = std::max(stats->max_claims_per_node_step, ms.max_claims_per_node_step);
        for (uint64_t i = 0; i < ms.schedule_len; ++i) stats->schedule_sizes.push_back(sched[i]);
    }
    return acc != 0;
}

// Text report of the instrumentation counters for one run (parallel.cpp:197-214).
inline std::string par_report(const Heap& h, InputView w, unsigned workers, uint64_t seed) {
    ParStats stats;
    const bool ok = par_accepts(h, w, workers, seed, &stats);
    std::string out;
    out += "workers\t" + std::to_string(workers) + "\n";
    out += "seed\t" + std::to_string(seed) + "\n";
    out += "macro steps\t" + std::to_string(stats.macro_steps) + "\n";
    out += "kernel launches\t" + std::to_string(stats.launches) + "\n";
    out += "claims\t" + std::to_string(stats.claims) + "\n";
    out += "max claims per node per step\t" + std::to_string(stats.max_claims_per_node_step) + "\n";
    out += "schedule sizes\t";
    for (size_t i = 0; i < stats.schedule_sizes.size(); ++i)
        out += (i ? " " : "") + std::to_string(stats.schedule_sizes[i]);
    out += "\nresult\t";
    out += ok ? "accept" : "reject";
    out += "\n";
    return out;
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
