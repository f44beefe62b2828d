// TEST INFRASTRUCTURE: declarations the reference's tests/support.hpp names
// (its ProcInvariantChecker for the process-calculus suites). The process
// calculus is out of scope for this build; these types exist only
// so support.hpp compiles for the lockstep and parallel suites, which use
// nothing from it but example_heap().
#pragma once

#include <vector>

#include "rx_b200.hpp"

namespace rx {

struct SeqTerm {
    enum class Kind { Recv, Send, Sync };
    Kind kind = Kind::Send;
    Addr addr = null_addr;
    Symbol sym = 0;
    bool operator==(const SeqTerm& o) const { return kind == o.kind && addr == o.addr && sym == o.sym; }
};
struct ProcTerm {
    std::vector<SeqTerm> terms;
};
struct MicroStep {
    Addr channel = null_addr;
};
inline SeqTerm send(Addr a) { return SeqTerm{SeqTerm::Kind::Send, a, 0}; }
inline SeqTerm sync_then(Symbol a, std::vector<SeqTerm> then) {
    return SeqTerm{SeqTerm::Kind::Sync, then.empty() ? null_addr : then[0].addr, a};
}
inline int cmp(const SeqTerm& a, const SeqTerm& b) {
    if (a.kind != b.kind) return a.kind < b.kind ? -1 : 1;
    if (a.addr != b.addr) return a.addr < b.addr ? -1 : 1;
    return a.sym == b.sym ? 0 : (a.sym < b.sym ? -1 : 1);
}

}  // namespace rx
