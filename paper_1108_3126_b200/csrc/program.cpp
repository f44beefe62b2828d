// Derived tables for the kernels. See program.hpp for the position form and
// its correspondence with the reference lockstep machine.
#include "program.hpp"

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

}  // namespace

Program build_program(const Heap& h) {
    const std::string bad = validate_heap(h);
    if (!bad.empty()) throw std::invalid_argument("bad heap: " + bad);
    Program p;
    p.heap = h;
    const int32_t N = h.size();
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
    const size_t W = static_cast<size_t>(p.W);
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

    // Byte classes: bytes with the same matching position set share a class;
    // class 0 is the empty set (bytes no position matches).
    p.byte_symbols = true;
    for (uint32_t s : p.pos_sym)
        if (s >= 0x80) p.byte_symbols = false;
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
