// Shared-memory images of the memoized lockstep step for the DFA kernels.
//
// Every DFA state is an E set of the position form (program.hpp), so a row
// lookup T[s][byte] is exactly one reference macro step
// step_char(evolve(S), a) (lockstep.cpp:64-80) applied to the set s stands
// for. Rows are addressed by their byte offset inside the image, so one
// shared-memory load per input byte advances a string.
#pragma once

#include <cstdint>
#include <vector>

#include "program.hpp"

namespace rxg {

struct KTable {
    std::vector<uint8_t> img;   // rows, then class map (if cls); padded to 16 B
    bool cls = false;           // rows indexed by byte class (else by raw byte)
    int esize = 2;              // entry bytes: 2 or 4
    int ncols = 0;              // symbol columns (256 or n_classes [+1 delimiter class])
    uint32_t row_bytes = 0;     // (ncols + 1) * esize ; last column = accept flag
    uint32_t cls_off = 0;       // offset of the 256-byte class map
    uint32_t start = 0;         // offset of the start state's row
    uint32_t dead = 0;          // offset of the empty-set row
    // delimited (line) tables only
    bool delimited = false;
    uint32_t delim_col = 0;     // column of the delimiter
    uint32_t skip = 0;          // SKIP row: swallow bytes until the first delimiter
    uint32_t acc_row = 0;       // START_A row = 1 << acc_shift (entered on an accepted line end)
    uint32_t acc_shift = 0;
    uint32_t tail_delta = 0;    // main row offset + tail_delta = tail-copy row offset
    uint32_t term_acc = 0;      // absorbing rows entered at the first delimiter in tail mode
    uint32_t term_rej = 0;
    int32_t n_states = 0;
    std::vector<uint8_t> accept;   // per DFA state (for checkpoints / host tests)
    std::vector<uint32_t> state_of_row;   // row index -> dfa state (main rows), for decoding
};

// Plain table: every byte is a symbol (single strings, fixed-stride batches).
KTable make_plain_table(const Program& p, const Dfa& d, bool force_class = false);

// Line table for delimiter byte `delim` (the delimiter is
// not part of a string, like std::getline in rxvm.cpp:102).
KTable make_line_table(const Program& p, const Dfa& d, uint8_t delim, bool force_class = false);

// Host model of the kernels' table walk (used by host tests of the images).
uint32_t ktable_step(const KTable& t, uint32_t off, uint8_t byte);
uint32_t ktable_accept(const KTable& t, uint32_t off);

}  // namespace rxg
