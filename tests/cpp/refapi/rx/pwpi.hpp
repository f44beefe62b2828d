// TEST INFRASTRUCTURE: <rx/pwpi.hpp> for the reference suites. The Fig. 3
// micro steps come from the facade; pwpi_accepts — the reference's memoized
// DFS decision over (address, position) states (pwpi.cpp:29-95), an engine
// this build does not ship (out of scope) — is restated here only
// as the independent checker the reference's test_lockstep.cpp compares with.
#pragma once

#include <vector>

#include "rx_b200.hpp"

namespace rx {

inline bool pwpi_accepts(const Heap& h, InputView w) {
    enum Mark : unsigned char { Unknown, InProgress, Dead, Live };
    const size_t cols = w.size() + 1;
    std::vector<unsigned char> mark(static_cast<size_t>(h.size() + 1) * cols, Unknown);
    auto reach = [&](auto&& self, Addr p, size_t pos) -> bool {
        const size_t i = static_cast<size_t>(p + 1) * cols + pos;
        if (mark[i] == Live) return true;
        if (mark[i] != Unknown) return false;   // dead, or on the current path (eps cycle)
        mark[i] = InProgress;
        bool live = false;
        if (p == null_addr) {
            live = pos == w.size();
        } else if (h.node(p).kind == Node::Kind::Chr) {
            live = pos < w.size() && h.node(p).sym == w[pos] && self(self, h.knode(p), pos + 1);
        } else {
            for (Addr q : eps_successors(h, p))
                if (self(self, q, pos)) {
                    live = true;
                    break;
                }
        }
        mark[i] = live ? Live : Dead;
        return live;
    };
    return reach(reach, h.root(), 0);
}

}  // namespace rx
