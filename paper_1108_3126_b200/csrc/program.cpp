// Derived tables for the kernels. See program.hpp for the position form and
// its correspondence with the reference lockstep machine.
#include "program.hpp"
#include "rxg_utf8.hpp"

#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>

namespace rxg {

namespace {

inline void set_bit(uint32_t* s, int32_t b) { s[b >> 5] |= 1u << (b & 31); }

// Unlabeled successors of p in the reference's fixed order (pwpi.cpp:9-20).
// Returns the count; entries may be kNull.
inline int eps_succ(const Heap& h, Addr p, Addr out[2]) {
    const HeapNode& n = h.nodes[static_cast<size_t>(p)];
    switch (n.kind) {
    case kAlt: out[0] = n.left; out[1] = n.right; return 2;
    case kSeq: out[0] = n.left; return 1;
    case kStar: out[0] = n.left; out[1] = h.knodes[static_cast<size_t>(p)]; return 2;
    case kEps: out[0] = h.knodes[static_cast<size_t>(p)]; return 1;
    default: return 0;
    }
}

// evolve({start}) as position bits into `row`, plus whether the null address
// is eps-reachable (eps_reaches_null({start}), lockstep.cpp:42-62). The two
// reference walks visit the same eps graph and stop at Chr nodes, so one
// traversal yields both.
struct Closure {
    const Heap& h;
    const std::vector<int32_t>& addr_pos;
    std::vector<uint32_t> stamp;
    std::vector<Addr> stack;
    uint32_t epoch = 0;

    Closure(const Heap& heap, const std::vector<int32_t>& ap)
        : h(heap), addr_pos(ap), stamp(static_cast<size_t>(heap.size()), 0) {}

    bool run(Addr start, uint32_t* row) {
        if (start == kNull) return true;
        ++epoch;
        bool null_reached = false;
        stack.clear();
        stack.push_back(start);
        stamp[static_cast<size_t>(start)] = epoch;
        while (!stack.empty()) {
            const Addr p = stack.back();
            stack.pop_back();
            if (h.nodes[static_cast<size_t>(p)].kind == kChr) {
                set_bit(row, addr_pos[static_cast<size_t>(p)]);
                continue;
            }
            Addr succ[2];
            const int k = eps_succ(h, p, succ);
            for (int j = 0; j < k; ++j) {
                const Addr q = succ[j];
                if (q == kNull) {
                    null_reached = true;
                    continue;
                }
                if (stamp[static_cast<size_t>(q)] == epoch) continue;
                stamp[static_cast<size_t>(q)] = epoch;
                stack.push_back(q);
            }
        }
        return null_reached;
    }
};

std::vector<uint8_t> utf8_bytes(uint32_t cp) {
    std::string s;
    rxg::append_utf8(s, static_cast<char32_t>(cp));
    return std::vector<uint8_t>(s.begin(), s.end());
}

// Rewrites the scalar position form into the UTF-8 byte position form.
void expand_utf8(Program& p) {
    const int32_t n_old = p.n_pos;
    const size_t W_old = static_cast<size_t>(p.W);
    std::vector<int32_t> entry(static_cast<size_t>(n_old) + 1);
    std::vector<std::vector<uint8_t>> bytes(static_cast<size_t>(n_old));
    int32_t n_new = 0;
    for (int32_t q = 0; q < n_old; ++q) {
        entry[static_cast<size_t>(q)] = n_new;
        bytes[static_cast<size_t>(q)] = utf8_bytes(p.pos_sym[static_cast<size_t>(q)]);
        n_new += static_cast<int32_t>(bytes[static_cast<size_t>(q)].size());
    }
    entry[static_cast<size_t>(n_old)] = n_new;   // accept bit
    const int32_t W_new = (n_new + 1 + 31) / 32;
    auto remap = [&](const uint32_t* src, uint32_t* dst) {
        for (int32_t q = 0; q <= n_old; ++q)
            if ((src[q >> 5] >> (q & 31)) & 1u) set_bit(dst, entry[static_cast<size_t>(q)]);
    };
    std::vector<uint32_t> follow(static_cast<size_t>(n_new + 1) * static_cast<size_t>(W_new), 0u);
    std::vector<uint32_t> init(static_cast<size_t>(W_new), 0u);
    std::vector<uint32_t> sym(static_cast<size_t>(n_new));
    std::vector<Addr> addr(static_cast<size_t>(n_new));
    for (int32_t q = 0; q < n_old; ++q) {
        const auto& b = bytes[static_cast<size_t>(q)];
        const int32_t e = entry[static_cast<size_t>(q)];
        for (size_t j = 0; j < b.size(); ++j) {
            const int32_t np = e + static_cast<int32_t>(j);
            sym[static_cast<size_t>(np)] = b[j];
            addr[static_cast<size_t>(np)] = p.pos_addr[static_cast<size_t>(q)];
            uint32_t* row = &follow[static_cast<size_t>(np) * static_cast<size_t>(W_new)];
            if (j + 1 < b.size()) set_bit(row, np + 1);
            else remap(&p.follow[static_cast<size_t>(q) * W_old], row);
        }
    }
    remap(p.init.data(), init.data());
    for (Addr a = 0; a < static_cast<Addr>(p.addr_pos.size()); ++a)
        if (p.addr_pos[static_cast<size_t>(a)] >= 0) p.addr_pos[static_cast<size_t>(a)] = entry[static_cast<size_t>(p.addr_pos[static_cast<size_t>(a)])];
    p.scalar_pos = n_old;
    p.n_pos = n_new;
    p.n_bits = n_new + 1;
    p.W = W_new;
    p.follow.swap(follow);
    p.init.swap(init);
    p.pos_sym.swap(sym);
    p.pos_addr.swap(addr);
}

}  // namespace

Program build_program(const Heap& h) {
    const std::string bad = validate_heap(h);
    if (!bad.empty()) throw std::invalid_argument("bad heap: " + bad);
    Program p;
    p.heap = h;
    const int32_t N = h.size();
    p.scalar_pos = 0;
    p.addr_pos.assign(static_cast<size_t>(N), -1);

    // Positions in left-to-right leaf order (pre-order walk, left child
    // first), so a concatenation of literals gets consecutive positions and
    // its follow relation becomes a one-bit shift. Guard against cyclic
    // caller-supplied heaps with a visit stamp.
    {
        std::vector<Addr> st{0};
        std::vector<uint8_t> seen(static_cast<size_t>(N), 0);
        while (!st.empty()) {
            const Addr a = st.back();
            st.pop_back();
            if (seen[static_cast<size_t>(a)]) continue;
            seen[static_cast<size_t>(a)] = 1;
            const HeapNode& n = h.nodes[static_cast<size_t>(a)];
            if (n.kind == kChr) {
                p.addr_pos[static_cast<size_t>(a)] = static_cast<int32_t>(p.pos_addr.size());
                p.pos_addr.push_back(a);
                p.pos_sym.push_back(n.sym);
            } else if (n.kind == kAlt || n.kind == kSeq) {
                st.push_back(n.right);
                st.push_back(n.left);
            } else if (n.kind == kStar) {
                st.push_back(n.left);
            }
        }
        // Chr nodes unreachable from the root (only possible in hand-made
        // heaps) still get positions so every Chr address maps somewhere.
        for (Addr a = 0; a < N; ++a) {
            if (h.nodes[static_cast<size_t>(a)].kind == kChr && p.addr_pos[static_cast<size_t>(a)] < 0) {
                p.addr_pos[static_cast<size_t>(a)] = static_cast<int32_t>(p.pos_addr.size());
                p.pos_addr.push_back(a);
                p.pos_sym.push_back(h.nodes[static_cast<size_t>(a)].sym);
            }
        }
    }
    p.n_pos = static_cast<int32_t>(p.pos_addr.size());
    p.n_bits = p.n_pos + 1;
    p.W = (p.n_bits + 31) / 32;
    size_t W = static_cast<size_t>(p.W);
    const int32_t A = p.n_pos;

    Closure cl(h, p.addr_pos);
    p.follow.assign(static_cast<size_t>(p.n_bits) * W, 0u);
    for (int32_t q = 0; q < p.n_pos; ++q) {
        uint32_t* row = &p.follow[static_cast<size_t>(q) * W];
        const Addr k = h.knodes[static_cast<size_t>(p.pos_addr[static_cast<size_t>(q)])];
        if (cl.run(k, row)) set_bit(row, A);
    }
    p.init.assign(W, 0u);
    if (cl.run(0, p.init.data())) set_bit(p.init.data(), A);

    // Symbols are matched as UTF-8 bytes. A literal whose scalar needs k > 1
    // bytes becomes a chain of k byte positions (entry = first byte); every
    // follow set that contained the literal now contains its entry. UTF-8 is
    // prefix-free and the lead byte fixes the length, so on valid UTF-8 input
    // the k byte steps reproduce the reference's one scalar step exactly
    // (decode_utf8, utf8.cpp:16-46, then step_char).
    bool valid = true, multi = false;
    for (uint32_t s : p.pos_sym) {
        if (s > 0x10FFFF || (s >= 0xD800 && s <= 0xDFFF)) valid = false;
        if (s >= 0x80) multi = true;
    }
    p.byte_symbols = valid;
    if (valid && multi) expand_utf8(p);

    W = static_cast<size_t>(p.W);
    // Byte classes: bytes with the same matching position set share a class;
    // class 0 is the empty set (bytes no position matches).
    std::vector<std::vector<uint32_t>> masks(256, std::vector<uint32_t>(W, 0u));
    for (int32_t q = 0; q < p.n_pos; ++q) {
        const uint32_t s = p.pos_sym[static_cast<size_t>(q)];
        if (s < 256) set_bit(masks[s].data(), q);
    }
    std::unordered_map<std::string, int32_t> ids;
    p.class_mask.assign(W, 0u);   // class 0
    ids.emplace(std::string(W * 4, '\0'), 0);
    p.n_classes = 1;
    for (int b = 0; b < 256; ++b) {
        std::string key(reinterpret_cast<const char*>(masks[b].data()), W * 4);
        auto it = ids.find(key);
        if (it == ids.end()) {
            it = ids.emplace(std::move(key), p.n_classes++).first;
            p.class_mask.insert(p.class_mask.end(), masks[b].begin(), masks[b].end());
        }
        p.byte_class[b] = static_cast<uint8_t>(it->second);
    }
    return p;
}

void step_set(const Program& p, const uint32_t* E, int32_t cls, uint32_t* out) {
    const size_t W = static_cast<size_t>(p.W);
    std::memset(out, 0, W * 4);
    const uint32_t* M = &p.class_mask[static_cast<size_t>(cls) * W];
    for (size_t w = 0; w < W; ++w) {
        uint32_t fire = E[w] & M[w];
        while (fire) {
            const int b = __builtin_ctz(fire);
            fire &= fire - 1;
            const uint32_t* row = &p.follow[(w * 32 + static_cast<size_t>(b)) * W];
            for (size_t j = 0; j < W; ++j) out[j] |= row[j];
        }
    }
}

bool build_dfa(const Program& p, int32_t max_states, Dfa& d) {
    const size_t W = static_cast<size_t>(p.W);
    const int32_t A = p.n_pos;
    d = Dfa{};
    d.n_classes = p.n_classes;
    std::unordered_map<std::string, int32_t> ids;
    ids.reserve(1024);
    auto intern = [&](const uint32_t* s) -> int32_t {
        std::string key(reinterpret_cast<const char*>(s), W * 4);
        auto it = ids.find(key);
        if (it != ids.end()) return it->second;
        if (d.n_states >= max_states) return -1;
        const int32_t id = d.n_states++;
        ids.emplace(std::move(key), id);
        d.sets.insert(d.sets.end(), s, s + W);
        d.accept.push_back(static_cast<uint8_t>((s[A >> 5] >> (A & 31)) & 1u));
        return id;
    };
    std::vector<uint32_t> empty(W, 0u), nxt(W, 0u);
    d.start = intern(p.init.data());
    if (d.start < 0) return false;
    for (int32_t s = 0; s < d.n_states; ++s) {
        for (int32_t c = 0; c < p.n_classes; ++c) {
            step_set(p, &d.sets[static_cast<size_t>(s) * W], c, nxt.data());
            const int32_t t = intern(nxt.data());
            if (t < 0) return false;
            d.next.push_back(t);
        }
    }
    d.dead = intern(empty.data());   // class 0 from any state reaches it, so it exists
    return d.dead >= 0;
}

int32_t minimize_dfa(Dfa& d, uint64_t max_work) {
    const int32_t S = d.n_states, C = d.n_classes;
    if (S <= 1) return S;
    std::vector<int32_t> blk(static_cast<size_t>(S)), nb(static_cast<size_t>(S));
    for (int32_t s = 0; s < S; ++s) blk[static_cast<size_t>(s)] = d.accept[static_cast<size_t>(s)];
    int32_t nblocks = -1;
    uint64_t work = 0;
    std::vector<int32_t> sig(static_cast<size_t>(C) + 1);
    for (;;) {
        std::unordered_map<std::string, int32_t> ids;
        ids.reserve(static_cast<size_t>(S) * 2);
        for (int32_t s = 0; s < S; ++s) {
            sig[0] = blk[static_cast<size_t>(s)];
            for (int32_t c = 0; c < C; ++c)
                sig[static_cast<size_t>(c) + 1] = blk[static_cast<size_t>(d.next[static_cast<size_t>(s) * C + c])];
            std::string key(reinterpret_cast<const char*>(sig.data()), sig.size() * sizeof(int32_t));
            auto it = ids.emplace(std::move(key), static_cast<int32_t>(ids.size())).first;
            nb[static_cast<size_t>(s)] = it->second;
        }
        work += static_cast<uint64_t>(S) * static_cast<uint64_t>(C + 1);
        const int32_t k = static_cast<int32_t>(ids.size());
        blk.swap(nb);
        if (k == nblocks) break;   // stable: the partition no longer splits
        nblocks = k;
        if (work > max_work) return S;
    }
    if (nblocks == S) return S;
    Dfa m;
    m.n_states = nblocks;
    m.n_classes = C;
    const size_t W = d.sets.size() / static_cast<size_t>(S);
    std::vector<int32_t> rep(static_cast<size_t>(nblocks), -1);
    for (int32_t s = 0; s < S; ++s)
        if (rep[static_cast<size_t>(blk[static_cast<size_t>(s)])] < 0) rep[static_cast<size_t>(blk[static_cast<size_t>(s)])] = s;
    m.next.resize(static_cast<size_t>(nblocks) * C);
    m.accept.resize(static_cast<size_t>(nblocks));
    m.sets.resize(static_cast<size_t>(nblocks) * W);
    for (int32_t b = 0; b < nblocks; ++b) {
        const int32_t r = rep[static_cast<size_t>(b)];
        m.accept[static_cast<size_t>(b)] = d.accept[static_cast<size_t>(r)];
        for (int32_t c = 0; c < C; ++c)
            m.next[static_cast<size_t>(b) * C + c] = blk[static_cast<size_t>(d.next[static_cast<size_t>(r) * C + c])];
        std::copy(d.sets.begin() + static_cast<std::ptrdiff_t>(r * W), d.sets.begin() + static_cast<std::ptrdiff_t>((r + 1) * W),
                  m.sets.begin() + static_cast<std::ptrdiff_t>(b * W));
    }
    m.start = blk[static_cast<size_t>(d.start)];
    m.dead = d.dead >= 0 ? blk[static_cast<size_t>(d.dead)] : -1;
    d = std::move(m);
    return S;
}

BitsetPlan build_bitset_plan(const Program& p) {
    const size_t W = static_cast<size_t>(p.W);
    BitsetPlan plan;
    plan.shift.assign(W, 0u);
    plan.has_group.assign(W, 0u);
    plan.group.assign(static_cast<size_t>(p.n_bits), -1);
    // How many positions share each full follow row: shared rows stay whole
    // (one group serves them all); a row owned by a single position that
    // contains q+1 is split into the shift bit plus a residual.
    std::unordered_map<std::string, int32_t> row_users;
    for (int32_t q = 0; q < p.n_pos; ++q) {
        const uint32_t* row = &p.follow[static_cast<size_t>(q) * W];
        ++row_users[std::string(reinterpret_cast<const char*>(row), W * 4)];
    }
    std::unordered_map<std::string, int32_t> ids;
    std::vector<uint32_t> resid(W);
    for (int32_t q = 0; q < p.n_pos; ++q) {
        const uint32_t* row = &p.follow[static_cast<size_t>(q) * W];
        std::memcpy(resid.data(), row, W * 4);
        const int32_t nb = q + 1;
        const bool shared =
            row_users[std::string(reinterpret_cast<const char*>(row), W * 4)] > 1;
        if (!shared && ((row[nb >> 5] >> (nb & 31)) & 1u)) {
            set_bit(plan.shift.data(), q);
            resid[static_cast<size_t>(nb >> 5)] &= ~(1u << (nb & 31));
        }
        bool any = false;
        for (uint32_t x : resid) any |= x != 0;
        if (!any) continue;
        std::string key(reinterpret_cast<const char*>(resid.data()), W * 4);
        auto it = ids.find(key);
        if (it == ids.end()) {
            it = ids.emplace(std::move(key), plan.n_groups++).first;
            plan.rows.insert(plan.rows.end(), resid.begin(), resid.end());
            plan.trigger.insert(plan.trigger.end(), W, 0u);
        }
        plan.group[static_cast<size_t>(q)] = it->second;
        set_bit(&plan.trigger[static_cast<size_t>(it->second) * W], q);
        set_bit(plan.has_group.data(), q);
    }
    return plan;
}

}  // namespace rxg
