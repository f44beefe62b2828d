/*
 * rxg.h — C ABI of the B200 lockstep regular-expression matcher.
 *
 * This is the drop-in boundary for the reference's matcher API
 * (arxiv/paper_1108_3126, proj/include/rx). Plain pointers and sizes only; no
 * C++ or torch types. Every entry point returns an int status (RXG_OK = 0);
 * rxg_last_error() gives a thread-local detail string for the last failure.
 *
 * Reference interface each entry point replaces (file:line under proj/):
 *   rxg_parse_compile       rx::parse (include/rx/regex.hpp:60, src/regex.cpp:186-194)
 *                           + rx::compile (include/rx/heap.hpp:43, src/heap.cpp:13-72)
 *   rxg_dump / rxg_parse_dump  rx::dump / rx::parse_dump (include/rx/heap.hpp:68-69)
 *   rxg_check_knode         rx::check_knode (include/rx/heap.hpp:52, src/heap.cpp:106-128)
 *   rxg_heap_create         (new) uploads a compiled rx::Heap {nodes, knodes}
 *                           (include/rx/heap.hpp:28-37) and its derived tables to a GPU
 *   rxg_match_one           rx::lockstep_accepts(const Heap&, InputView, LockstepStats*)
 *                           (include/rx/lockstep.hpp:43, src/lockstep.cpp:75-82);
 *                           engine RXG_ENGINE_ROUNDS / PERNODE reproduce rx::par_accepts
 *                           (include/rx/parallel.hpp:102, src/parallel.cpp:192-195)
 *   rxg_match_batch*        rx::lockstep_accepts over every line of a buffer, the loop of
 *                           `rxvm match` (tools/rxvm.cpp:100-112, std::getline semantics)
 *   rxg_match_batch_multi   the same, sharded over several GPUs with one count all-reduce
 *
 * Symbols are bytes: every literal is matched as the UTF-8 encoding of its
 * scalar (a multi-byte literal is a chain of byte positions). UTF-8 is
 * prefix-free and the lead byte fixes the length, so on valid UTF-8 input
 * this is exactly the reference's match over decode_utf8 scalars. On invalid
 * UTF-8 the reference throws; here the affected strings simply do not match
 * (rxgmatch validates and exits 2 like rxvm). The literal rounds engine
 * (RXG_ENGINE_ROUNDS) compares raw bytes with literals and needs ASCII
 * literals (RXG_EUNSUPPORTED otherwise).
 */
#ifndef RXG_H
#define RXG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define RXG_OK 0
#define RXG_EINVAL 1        /* bad argument (null pointer, bad size, misaligned buffer) */
#define RXG_EPARSE 2        /* pattern syntax error; rx::ParseError (regex.hpp:50-54) */
#define RXG_EUTF8 3         /* malformed UTF-8 pattern; decode_utf8 (utf8.cpp:32-41) */
#define RXG_EUNSUPPORTED 4  /* engine cannot run this pattern / mode */
#define RXG_ECUDA 5         /* CUDA runtime error */
#define RXG_ENOMEM 6        /* allocation failed */
#define RXG_ETOOBIG 7       /* memoized step table exceeds the shared-memory budget */
#define RXG_ENCCL 8         /* NCCL unavailable or failed */
#define RXG_EHEAP 9         /* malformed heap table */
#define RXG_ENODEV 10       /* handle has no device tables (created with device < 0) */

/* node kinds, rx::Node::Kind order (heap.hpp:18) */
#define RXG_NODE_EPS 0
#define RXG_NODE_CHR 1
#define RXG_NODE_ALT 2
#define RXG_NODE_SEQ 3
#define RXG_NODE_STAR 4

/* single-string engines (rxg_match_one*) */
#define RXG_ENGINE_AUTO 0     /* memoized step (chunk-parallel) when its table fits, else PERNODE */
#define RXG_ENGINE_DFA_SEQ 1  /* one thread walks the memoized step table */
#define RXG_ENGINE_PERNODE 2  /* K1: paper §8 thread-per-node lockstep, bitset form, one warp per
                                 string; strings of 1 MiB and more as segments across SMs (warp per
                                 segment, guessed entry sets, exact repair rounds; cooperative launch) */
#define RXG_ENGINE_ROUNDS 3   /* literal §8 protocol: one thread per heap node, c/n stamps, rounds */
#define RXG_ENGINE_CHUNKED 4  /* chunk-parallel walk of the step table (all SMs) */

/* Byte layout identical to rx::Node (heap.hpp:17-23): 16 bytes. */
typedef struct rxg_node {
    uint8_t kind;
    uint8_t pad[3];
    uint32_t sym;
    int32_t left;
    int32_t right;
} rxg_node;

typedef struct rxg_heap rxg_heap;

typedef struct rxg_heap_info {
    int32_t nodes;         /* N */
    int32_t positions;     /* |C| (Chr nodes) */
    int32_t words;         /* W = ceil((|C|+1)/32) */
    int32_t classes;       /* byte classes (class 0 = matches nothing) */
    int32_t dfa_states;    /* states of the minimised memoized step (0 if over the cap) */
    int32_t byte_symbols;  /* 1 if every literal is ASCII */
    int32_t device;        /* CUDA device, or -1 for a host-only handle */
    int32_t nullable;      /* root eps-reaches null: the empty string matches */
    uint32_t line_table_bytes;   /* shared-memory image for '\n' lines (0 if none) */
    uint32_t plain_table_bytes;  /* shared-memory image for single strings / fixed stride */
    int32_t dfa_sets;      /* distinct memoized E sets before minimisation (0 if over the cap) */
    int32_t line_tma_layout;   /* TMA table built for '\n' lines so far: 0 none, 1 direct, 2 class map, 3 class rows with range-clamped columns */
    int32_t line_col_bytes;    /* its column stride (direct layout; chosen by rxg_heap_tune) */
    int32_t chunk_lookback;    /* single-string engine: bytes walked to guess a range's entry (tuned) */
} rxg_heap_info;

const char* rxg_strerror(int status);
const char* rxg_last_error(void);
const char* rxg_version(void);

/* ── front end (host only; no GPU needed) ─────────────────────────────── */

/* Parse + compile. Writes min(n, cap) nodes/knodes; *n_out = N. On
 * RXG_EPARSE / RXG_EUTF8, *err_pos is the scalar / byte offset. */
int rxg_parse_compile(const char* pattern, size_t len, rxg_node* nodes, int32_t* knodes,
                      int32_t cap, int32_t* n_out, size_t* err_pos);

/* Canonical printer (rx::print, regex.hpp:65). Writes a NUL-terminated string. */
int rxg_print(const char* pattern, size_t len, char* out, size_t cap, size_t* out_len);

/* Heap dump text (three tab-separated columns per address). */
int rxg_dump(const rxg_node* nodes, const int32_t* knodes, int32_t n, char* out, size_t cap,
             size_t* out_len);
int rxg_parse_dump(const char* text, size_t len, rxg_node* nodes, int32_t* knodes, int32_t cap,
                   int32_t* n_out);
int rxg_check_knode(const rxg_node* nodes, const int32_t* knodes, int32_t n, int32_t* ok);

/* ── compiled heap handle ─────────────────────────────────────────────── */

/* device >= 0: upload tables to that GPU. device < 0: host-only handle
 * (front end, derived tables and DFA; no kernels). */
int rxg_heap_create(const rxg_node* nodes, const int32_t* knodes, int32_t n, int device,
                    rxg_heap** out);
int rxg_heap_create_pattern(const char* pattern, size_t len, int device, rxg_heap** out);
void rxg_heap_destroy(rxg_heap* h);
int rxg_heap_info_get(const rxg_heap* h, rxg_heap_info* info);

/* Planner hint: sample the state x byte visit frequencies of typical input
 * for `delimiter`-separated lines and re-place the shared-memory table rows
 * so concurrent lanes in different states hit different banks. Changes
 * speed only, never results. rxg_match_batch_host tunes itself from the
 * head of its buffer on first use. delimiter = -1: the sample is one long
 * string (placement of the chunk-parallel single-string table). */
int rxg_heap_tune(rxg_heap* h, const uint8_t* sample, uint64_t len, int32_t delimiter);

/* Derived tables of the position form, for tests/tools.
 * pos_addr: |C| heap addresses; follow: (|C|+1)*W words; init: W words. */
int rxg_heap_tables(const rxg_heap* h, int32_t* pos_addr, uint32_t* follow, uint32_t* init);

/* Host walk of the memoized step (no GPU): E sets after each symbol.
 * sets_out: (len+1)*W words (row 0 = E_0), may be null; *accept set. */
int rxg_host_walk(const rxg_heap* h, const uint8_t* bytes, uint64_t len, uint32_t* sets_out,
                  int32_t* accept);

/* Host emulation of the batch kernels (same table image, same chunk
 * ownership / SKIP / tail rules), for CPU tests of the device logic.
 * chunk: bytes per chain (multiple of 16; 0 = default). */
int rxg_host_emulate_batch(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                           uint32_t stride, uint32_t chunk, uint64_t* count, uint8_t* results);

/* Same for the TMA-staged line kernel's layout and range partition
 * (chunk: multiple of 32). RXG_ETOOBIG if the DFA does not fit that layout. */
int rxg_host_emulate_lines_tma(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                               uint32_t chunk, uint64_t* count);
/* Host emulation of the single-string TMA table (the chunked engine's
 * layout for this heap): walks the whole string from the start state.
 * layout (nullable): 1 direct, 2 class map, 3 range-clamped class rows,
 * 4 packed per-byte transition words (DFA <= 6 states). Tests only. */
int rxg_host_emulate_chunk_tma(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t* accept,
                               int32_t* layout);

/* ── matching ─────────────────────────────────────────────────────────── */

/* One string, host buffer (synchronous). */
int rxg_match_one(rxg_heap* h, const uint8_t* bytes, uint64_t len, int engine, int32_t* accept);

/* One string, device buffer, asynchronous on `stream` (cudaStream_t or NULL).
 * d_accept is a device int32; d_bytes must be 16-byte aligned (RXG_EINVAL
 * otherwise: every engine reads 16-byte vectors). The chunk-parallel engine keeps its scratch
 * (guesses, exits, checkpoints: ~16 B per 256 input bytes) and seam counters
 * per (heap, stream), grown to the largest string seen on that stream and
 * freed with the heap; make the first call of a given size outside
 * CUDA-graph capture. */
int rxg_match_one_device(rxg_heap* h, const uint8_t* d_bytes, uint64_t len, int engine,
                         int32_t* d_accept, void* stream);

/* Per-engine options and instrumentation for rxg_match_one_ex (all optional;
 * zero-initialise). Device pointers. */
typedef struct rxg_one_opts {
    uint32_t checkpoint_every;        /* PERNODE: E set (W words) after every k symbols ... */
    uint32_t* d_checkpoints;          /* ... into (len / k) x W words (the chunk-parallel oracle check) */
    unsigned long long* d_stats;      /* ROUNDS: claims, rounds, macro steps, max claims per node per step
                                         (rx::ParStats, parallel.hpp:52-58) */
    uint32_t* d_trace;                /* ROUNDS: per symbol the next schedule as (N+1)-bit rows, bit N = null;
                                         zeroed by the caller (test_parallel.cpp:114-137) */
    uint32_t chunk;                   /* CHUNKED: bytes per range (multiple of 32 on the TMA path, 64 otherwise), 0 = auto */
    uint32_t lookback;                /* CHUNKED: bytes walked before a range to guess its entry state
                                         (0 = the heap's default: 64, or 16/32/64 after rxg_heap_tune) */
    unsigned long long* d_repairs;    /* CHUNKED: ranges re-walked by the in-order repair pass */
    uint32_t flags;                   /* RXG_ONE_ENTRY: start in entry_state instead of the start state */
    uint32_t entry_state;             /* CHUNKED: opaque table state (from a d_exit_state of the same pattern) */
    uint32_t* d_exit_state;           /* CHUNKED: the table state after the string (device, nullable). States
                                         are interchangeable between heaps of the same pattern built alike
                                         (same tuning); this is how segments of one string chain. */
    unsigned long long* d_enqueued;   /* ROUNDS: rx::LockstepStats.enqueued of the same string (lockstep.hpp:16-18):
                                         the addresses evolve enqueues = every macro step's claims but the
                                         end-of-input step's */
    uint32_t* d_schedule;             /* ROUNDS: nodes scheduled at the start of each macro step, len + 1 entries max
                                         (rx::ParStats.schedule_sizes, parallel.hpp:57) */
} rxg_one_opts;
#define RXG_ONE_ENTRY 1u
#define RXG_ONE_SINGLE_WARP 2u   /* PERNODE: walk a long string with one warp (no segments) */

int rxg_match_one_ex(rxg_heap* h, const uint8_t* d_bytes, uint64_t len, int engine, int32_t* d_accept,
                     const rxg_one_opts* opts, void* stream);

/* Batch over a device buffer, asynchronous on `stream`.
 *   delimiter in [0,255]: strings are the lines of the buffer split on that
 *     byte (the delimiter is not part of a string; a final unterminated
 *     segment is a string, a trailing delimiter does not open one);
 *   delimiter < 0: fixed stride, strings text[i*stride, (i+1)*stride).
 * d_count (device u64) receives the number of matching strings (it is
 * overwritten). d_results (device, nullable) receives one 0/1 byte per
 * string; it needs room for (#delimiters + 1) bytes in line mode. d_text
 * must be 16-byte aligned. The first call on a stream allocates a 32-byte
 * per-(heap, stream) completion slot (the kernels publish the count through
 * it, no memset per call); make that first call outside CUDA-graph capture. */
int rxg_match_batch(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter,
                    uint32_t stride, unsigned long long* d_count, uint8_t* d_results,
                    void* stream);

/* Batch engines for rxg_match_batch_ex */
#define RXG_BATCH_AUTO 0    /* memoized-step (DFA) kernels; bitset if the DFA is over the cap */
#define RXG_BATCH_DFA 1     /* K2: one lane per byte range, memoized step in shared memory */
#define RXG_BATCH_BITSET 2  /* K2b: one warp per line, bitset lockstep (line mode only) */

int rxg_match_batch_ex(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride,
                       int engine, unsigned long long* d_count, uint8_t* d_results, void* stream);

/* Same, host buffers; copies in and out inside the call (synchronous). */
int rxg_match_batch_host(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                         uint32_t stride, uint64_t* count, uint8_t* results);

/* rxg_match_batch_host plus, when utf8_first_bad is non-null, the device
 * UTF-8 check of every string (rxg_utf8_check) fused into the same pipelined
 * pass: *utf8_first_bad = offset of the first byte at which rx::decode_utf8
 * would throw on its string, or UINT64_MAX. This is the whole per-line loop
 * of `rxvm match` (tools/rxvm.cpp:100-112: getline, decode_utf8, lockstep). */
int rxg_match_batch_host_ex(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                            uint32_t stride, uint64_t* count, uint8_t* results,
                            uint64_t* utf8_first_bad);

/* Device UTF-8 decode check, exactly rx::decode_utf8 (src/utf8.cpp:16-46)
 * applied to every string of the buffer (delimiter in [0,127] or -1 with a
 * fixed stride, as rxg_match_batch; delimiter -1 and stride 0 = the whole
 * buffer is one string): *d_first_bad (device u64) receives the byte offset
 * the reference's runtime_error "invalid UTF-8 at byte N" names for the
 * first failing string (N + the string's offset), or UINT64_MAX when every
 * string decodes. Asynchronous on `stream`; any alignment. */
int rxg_utf8_check(int device, const uint8_t* d_text, uint64_t len, int32_t delimiter,
                   uint32_t stride, uint64_t* d_first_bad, void* stream);

/* Same on a host buffer (synchronous). */
int rxg_utf8_check_host(int device, const uint8_t* text, uint64_t len, int32_t delimiter,
                        uint32_t stride, uint64_t* first_bad);

/* One long string split over `ndev` GPUs (chunk-speculative
 * matching across devices): segment k starts in the state its 64-byte prefix
 * leads to from the start state (one small walk), every device runs the
 * chunk-parallel engine on its segment at once, then the host chains the
 * segments' entry and exit states in order and re-runs a segment only where
 * its guessed entry differs from the exact exit of the previous one. Exact
 * for every pattern; *accept = rx::lockstep_accepts over the whole string.
 * The same device may appear more than once. */
int rxg_match_one_multi(const int* devices, int ndev, const char* pattern, size_t plen, const uint8_t* text,
                        uint64_t len, int32_t* accept, int32_t* resegments);

/* One string through the literal §8 protocol (RXG_ENGINE_ROUNDS, host buffer,
 * synchronous) with the reference's instrumentation: rx::LockstepStats
 * (lockstep.hpp:16-18) and rx::ParStats (parallel.hpp:52-58). schedule
 * (host, nullable) receives one entry per macro step (len + 1 max);
 * *schedule_len = entries. RXG_EUNSUPPORTED for non-ASCII literals. */
typedef struct rxg_match_stats {
    uint64_t enqueued;
    uint64_t claims, launches, macro_steps;
    uint32_t max_claims_per_node_step;
    uint32_t* schedule;
    uint64_t schedule_len;
} rxg_match_stats;
int rxg_match_one_stats(rxg_heap* h, const uint8_t* bytes, uint64_t len, int32_t* accept, rxg_match_stats* stats);

/* ── the paper's protocol on caller-held state (parallel.hpp:24-103) ────
 * rx::ParState in plain arrays: c / n stamps (N x int64: c[i] == t scheduled,
 * -t claimed; n[j] == t + 1 scheduled next), claim counters (N x u32), the
 * macro-step counter t and the four flags. rxg_par_task runs one par_task
 * (parallel.cpp:50-78) on the device; rxg_par_run_rounds runs the rounds of
 * one macro step (parallel.cpp:120-154: dispatch {i : c[i] == t} fixed per
 * round, until no task schedules more work), *launches = rounds. Both copy
 * the state in and out (host arrays); symbol 0xFFFFFFFF = end of input. */
typedef struct rxg_par_state {
    int64_t* c;
    int64_t* n;
    uint32_t* claim_count;
    int64_t t;
    int32_t more_c, any_n, accept_pending, accept_next;
} rxg_par_state;
int rxg_par_task(rxg_heap* h, rxg_par_state* st, int32_t node, uint32_t symbol);
int rxg_par_run_rounds(rxg_heap* h, rxg_par_state* st, uint32_t symbol, uint64_t* launches);

/* ── syntax trees (regex.hpp:26-66) and set-level functions (lockstep.hpp:24-49), host ──
 * A tree is an array of nodes whose children precede them (kinds in
 * rx::Regex::Kind order), one root, no sharing. */
#define RXG_AST_EPS 0
#define RXG_AST_CHR 1
#define RXG_AST_STAR 2
#define RXG_AST_SEQ 3
#define RXG_AST_ALT 4
typedef struct rxg_ast_node {
    uint8_t kind;
    uint8_t pad[3];
    uint32_t sym;
    int32_t left;
    int32_t right;
} rxg_ast_node;
/* rx::parse (regex.cpp:186-194): *n_out nodes (min(n, cap) written), *root. */
int rxg_parse_ast(const char* pattern, size_t len, rxg_ast_node* nodes, int32_t cap, int32_t* n_out, int32_t* root,
                  size_t* err_pos);
/* rx::print (regex.cpp:196-200) of a tree. */
int rxg_print_ast(const rxg_ast_node* nodes, int32_t n, int32_t root, char* out, size_t cap, size_t* out_len);
/* rx::compile (heap.cpp:13-72) of a tree: the heap has exactly n nodes. */
int rxg_compile_ast(const rxg_ast_node* nodes, int32_t n, int32_t root, rxg_node* heap, int32_t* knodes,
                    int32_t cap, int32_t* n_out);
/* rx::evolve_ordered (lockstep.cpp:10-35): s = the set in std::set order
 * (ascending, -1 = null first); out (capacity n) = Chr addresses in worklist
 * discovery order; *enqueued += pushes (LockstepStats, nullable). */
int rxg_evolve(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns,
               int32_t* out, int32_t* n_out, uint64_t* enqueued);
/* rx::eps_reaches_null (lockstep.cpp:42-62). */
int rxg_eps_reaches_null(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns,
                         int32_t* result);
/* rx::step_char (lockstep.cpp:64-73): out (capacity ns) ascending; RXG_EINVAL
 * when a member is neither a Chr node nor null (the reference throws
 * std::invalid_argument). */
int rxg_step_char(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns, uint32_t a,
                  int32_t* out, int32_t* n_out);

/* ── several GPUs ────────────────────────────────────
 * Strings are independent: a batch is cut into contiguous byte-balanced
 * shards at string boundaries (rxg_shard_bounds), each GPU matches its shard,
 * and one all-reduce of the 8-byte match count is the only inter-GPU
 * traffic. The reference has no multi-device code (its data-parallel axis is
 * crosscheck's job pool over independent cases, crosscheck.cpp:119-149). */

/* One process per GPU (torchrun / MPI): a NCCL communicator over the ranks.
 * Rank 0 makes the 128-byte id, the host plumbing broadcasts it, every rank
 * calls rxg_comm_init_rank (collective: blocks until all ranks joined). */
typedef struct rxg_comm rxg_comm;
int rxg_comm_unique_id(uint8_t* id, size_t cap);
int rxg_comm_init_rank(const uint8_t* id, size_t id_len, int nranks, int rank, int device, rxg_comm** out);
void rxg_comm_destroy(rxg_comm* c);

/* rxg_match_batch on this rank's shard, then ncclAllReduce(sum) of *d_count
 * across the communicator, both enqueued on `stream`: when the stream reaches
 * the end, d_count holds the whole job's match count on every rank. */
int rxg_match_batch_allreduce(rxg_heap* h, rxg_comm* c, const uint8_t* d_text, uint64_t len,
                              int32_t delimiter, uint32_t stride, unsigned long long* d_count,
                              uint8_t* d_results, void* stream);

/* One process, several GPUs: a persistent handle. The pattern is compiled and
 * its memoized step built once, then uploaded to every device; one worker
 * thread per device drives that device's pipelined host path (copy of piece
 * k+1 overlapping the match of piece k); NCCL communicators (ncclCommInitAll)
 * are created once. A device may be listed more than once (shards then share
 * that GPU; NCCL needs distinct GPUs, so the counts are summed on the host). */
typedef struct rxg_multi rxg_multi;
int rxg_multi_create(const int* devices, int ndev, const char* pattern, size_t plen, rxg_multi** out);
void rxg_multi_destroy(rxg_multi* m);
int rxg_multi_info(const rxg_multi* m, int32_t* ndev, int32_t* uses_nccl);
/* rxg_heap_tune for every device (sampled once). */
int rxg_multi_tune(rxg_multi* m, const uint8_t* sample, uint64_t len, int32_t delimiter);
/* Shard a host buffer over the handle's devices; *count = total matches
 * (all-reduced over NCCL when the devices are distinct); results (nullable):
 * one 0/1 byte per string, in order. Synchronous; one call at a time per handle. */
int rxg_multi_match_batch(rxg_multi* m, const uint8_t* text, uint64_t len, int32_t delimiter,
                          uint32_t stride, uint64_t* count, uint8_t* results);

/* One-shot form of the above (handle created and destroyed inside the call). */
int rxg_match_batch_multi(const int* devices, int ndev, const char* pattern, size_t plen,
                          const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                          uint64_t* count, uint8_t* results);

/* Every pattern against every string — the reference's crosscheck sweep
 * shape (crosscheck.cpp:111-185) as one device call; a GPU `EngineId` for
 * run_engine (engines.cpp:40-82) can answer from this. patterns: n_patterns
 * NUL-terminated UTF-8 patterns back to back. Strings: the lines of text
 * (delimiter >= 0) or fixed-stride pieces. results: n_patterns x n_strings
 * bytes (row-major, 0/1). On a pattern error returns RXG_EPARSE/RXG_EUTF8 and
 * *bad_pattern = its index. */
int rxg_match_many(int device, const char* patterns, int32_t n_patterns, const uint8_t* text, uint64_t len,
                   int32_t delimiter, uint32_t stride, uint8_t* results, uint64_t* n_strings, int32_t* bad_pattern);

/* Shard boundaries used by rxg_match_batch_multi: offsets[0..ndev], split at
 * delimiter boundaries (line mode) or stride multiples. Host only. */
int rxg_shard_bounds(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                     int ndev, uint64_t* offsets);

/* Strings in a host buffer as the batch calls split it (delimiter 0-255:
 * delimiters plus an unterminated last string, std::getline semantics;
 * delimiter < 0: len / stride): the size of a per-string results buffer.
 * Host only, counted on a few host threads. */
int rxg_count_strings(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* n);

/* Number of kernels the last matching call on this thread launched. */
int rxg_last_launch_count(void);

/* Process-wide tuning and test switches: they select kernel variants and
 * table layouts (speed only, never results). value NULL or "" unsets. Names:
 * RXG_NO_TMA, RXG_NO_LT, RXG_NO_FIXED_TMA (generic kernels), RXG_LINE_CHUNK
 * (bytes per range), RXG_LT_SHAPE, RXG_CHUNK_SHAPE, RXG_TMA_PROMO,
 * RXG_SKIP_SHARE, RXG_COL_BYTES, RXG_NO_ROW_PAIRS, RXG_FORCE_CLASS,
 * RXG_NO_RANGE_LAYOUT, RXG_NO_PACKED, RXG_NO_BITS_TMA (the bitset engine's
 * generic kernel), RXG_CHUNK_FN ("0"/"1": force the
 * chunk engine's transfer-function mode off/on for packed tables; by default
 * it is on for automata with a byte that permutes states), RXG_COPY_THREADS
 * (host threads filling pinned staging from pageable input). The library
 * reads no environment. */
int rxg_set_option(const char* name, const char* value);

/* ── synthetic workloads of SURVEY.md §8(d) (host only) ───────────────── */
int rxg_synth_pattern(char config, char* out, size_t cap, size_t* out_len);
uint64_t rxg_synth_input_size(char config);
int rxg_synth_input(char config, uint64_t seed, uint8_t* out, uint64_t cap, uint64_t* written);

#ifdef __cplusplus
}
#endif

#endif /* RXG_H */
