// Derived matcher tables built from a compiled heap (the "front end step 2"
// of SURVEY.md §7): the position form of the reference lockstep machine.
//
// Reference machine (proj/src/lockstep.cpp:75-82):
//     S0 = {root};  S <- step_char(evolve(S), a) for each symbol, reject on S = {};
//     accept iff null in S or eps_reaches_null(S).
// Position form used by every kernel (SURVEY.md §8(a) "verified restatement"):
//     positions      = Chr nodes, numbered left-to-right (pre-order), plus one
//                      extra "accept" bit A = n_pos
//     F'(q)          = evolve({knode q})  ∪ {A if knode q = null or eps_reaches_null({knode q})}
//     E0             = evolve({root})     ∪ {A if eps_reaches_null({root})}
//     E_{i+1}        = ∪ { F'(q) : q in E_i, sym(q) = a_i }      (A never matches)
//     accept(w)      = A in E_|w|
// Literals are then expanded to UTF-8 byte chains (expand_utf8) so that the
// kernels step on bytes; for ASCII literals nothing changes.
// evolve distributes over union, so E_i = evolve(S_i) ∪ {A iff S_i accepts}
// at every step, and the early reject of the reference is the absorbing
// empty set here. DFA states are memoized E sets of exactly this step.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "frontend.hpp"

namespace rxg {

struct Program {
    Heap heap;
    int32_t n_pos = 0;    // |C|
    int32_t n_bits = 0;   // |C| + 1 (accept bit last)
    int32_t W = 0;        // 32-bit words per position set
    std::vector<Addr> pos_addr;     // position -> heap address
    std::vector<int32_t> addr_pos;  // heap address -> position or -1
    std::vector<uint32_t> pos_sym;  // position -> symbol
    std::vector<uint32_t> follow;   // n_bits x W ; row A is empty
    std::vector<uint32_t> init;     // W
    bool byte_symbols = true;       // every literal is a Unicode scalar: matched as its UTF-8 bytes
    int32_t scalar_pos = 0;         // Chr nodes before UTF-8 expansion (0 if every literal is ASCII)
    uint8_t byte_class[256] = {};   // byte -> class id; class 0 matches no position
    int32_t n_classes = 0;
    std::vector<uint32_t> class_mask;   // n_classes x W

    bool test(const std::vector<uint32_t>& s, int32_t bit) const {
        return (s[static_cast<size_t>(bit) >> 5] >> (bit & 31)) & 1u;
    }
};

Program build_program(const Heap& h);

// One lockstep step on host bitsets (E -> E'), used by the DFA builder and tests.
void step_set(const Program& p, const uint32_t* E, int32_t cls, uint32_t* out);

struct Dfa {
    int32_t n_states = 0;
    int32_t n_classes = 0;
    int32_t start = 0;
    int32_t dead = -1;                 // id of the empty set (always present)
    std::vector<int32_t> next;         // n_states x n_classes
    std::vector<uint8_t> accept;       // accept bit of each state set
    std::vector<uint32_t> sets;        // n_states x W  (the memoized E sets)
};

// Subset construction over byte classes. Returns false (and leaves `out`
// partially filled) if more than max_states states would be needed.
bool build_dfa(const Program& p, int32_t max_states, Dfa& out);

// Moore partition refinement: merges states with the same accept bit on
// every continuation (the kernels only need each string's accept bit, which
// the minimal automaton gives for every input). `sets` keeps one member's E
// set per merged state. Returns the state count before minimisation; leaves
// the automaton unchanged if the refinement would exceed `max_work` steps.
int32_t minimize_dfa(Dfa& d, uint64_t max_work = 400'000'000ull);

// Decomposition of F' used by the bitset kernels:
//   F'(q) = ({q+1} if shift[q]) ∪ R(q),   R(q) = rows[group[q]] (group -1 = empty)
// Identical residual rows share one group (dedup by row equality).
struct BitsetPlan {
    std::vector<uint32_t> shift;        // W : bit q set iff q+1 in F'(q)
    std::vector<int32_t> group;         // n_bits : residual row id or -1
    int32_t n_groups = 0;
    std::vector<uint32_t> rows;         // n_groups x W
    std::vector<uint32_t> trigger;      // n_groups x W : positions whose residual is that row
    std::vector<uint32_t> has_group;    // W : positions with a nonempty residual
};

BitsetPlan build_bitset_plan(const Program& p);

}  // namespace rxg
