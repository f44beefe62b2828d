/* TEST INFRASTRUCTURE — see lockstep_oracle.c. Not part of the product. */
#ifndef LOCKSTEP_ORACLE_H
#define LOCKSTEP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same 16-byte layout as rx::Node (proj/include/rx/heap.hpp:17-23). */
typedef struct oracle_node {
    uint8_t kind;
    uint8_t pad[3];
    uint32_t sym;
    int32_t left;
    int32_t right;
} oracle_node;

typedef struct oracle_heap {
    const oracle_node* nodes;
    const int32_t* knodes;
    int32_t n;
} oracle_heap;

typedef struct oracle_ws {
    int32_t n;
    uint32_t* seen;
    int32_t* queue;
    uint32_t epoch;
} oracle_ws;

void oracle_ws_init(oracle_ws* ws, int32_t n);
void oracle_ws_free(oracle_ws* ws);
int32_t oracle_evolve(const oracle_heap* h, oracle_ws* ws, const int32_t* s, int32_t ns, int32_t* out,
                      uint64_t* enqueued);
int oracle_eps_reaches_null(const oracle_heap* h, oracle_ws* ws, const int32_t* s, int32_t ns);
int32_t oracle_step_char(const oracle_heap* h, oracle_ws* ws, const int32_t* e, int32_t ne, uint32_t a,
                         int32_t* out);
int oracle_lockstep_accepts(const oracle_heap* h, oracle_ws* ws, const uint32_t* w, uint64_t len,
                            int32_t* buf_a, int32_t* buf_b, uint64_t* enqueued);
int oracle_accepts_bytes(const oracle_heap* h, const uint8_t* bytes, uint64_t len);
int32_t oracle_walk_from(const oracle_heap* h, int32_t* s_io, int32_t n_io, const uint8_t* bytes, uint64_t len);
uint64_t oracle_split(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* starts,
                      uint64_t* lens);
uint64_t oracle_match_batch(const oracle_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                            uint32_t stride, uint8_t* results, int nthreads);
int64_t oracle_decode_utf8_error(const uint8_t* s, uint64_t n);
uint64_t oracle_utf8_first_bad(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride);

#ifdef __cplusplus
}
#endif

#endif
