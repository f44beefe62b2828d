/*
 * TEST INFRASTRUCTURE — CPU oracle for the B200 lockstep matcher.
 *
 * A plain-C restatement of the reference's sequential lockstep machine
 * (arxiv/paper_1108_3126, proj/src/lockstep.cpp) over the compiled heap
 * table {nodes, knodes} (proj/include/rx/heap.hpp:17-37). It is the checker
 * the parity tests compare the CUDA kernels against, and the "port" kind of
 * the bench's cpu_baseline. The product library never links or calls it.
 *
 * Pinned against the reference two ways (tests/test_oracle.py):
 *   - the golden vectors of proj/tests/test_lockstep.cpp:15-58 and the
 *     exhaustive small suite of test_lockstep.cpp:60-72 / acceptance
 *     criterion 3 (acceptance_main.cpp:93-105), via tests/golden/;
 *   - against oracle/_ref (the reference's own lockstep.cpp compiled from its
 *     sources by oracle/Makefile) on seeded random cases.
 *
 * Function-by-function correspondence:
 *   eps_successors     proj/src/pwpi.cpp:9-20
 *   evolve             proj/src/lockstep.cpp:10-40   (FIFO worklist + seen)
 *   eps_reaches_null   proj/src/lockstep.cpp:42-62
 *   step_char          proj/src/lockstep.cpp:64-73
 *   lockstep_accepts   proj/src/lockstep.cpp:75-82
 */
#include "lockstep_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { EPS = 0, CHR = 1, ALT = 2, SEQ = 3, STAR = 4 };

/* pwpi.cpp:9-20: unlabeled successors in fixed order; may contain null (-1). */
static int eps_successors(const oracle_heap* h, int32_t p, int32_t out[2]) {
    const oracle_node* n = &h->nodes[p];
    switch (n->kind) {
    case ALT: out[0] = n->left; out[1] = n->right; return 2;
    case SEQ: out[0] = n->left; return 1;
    case STAR: out[0] = n->left; out[1] = h->knodes[p]; return 2;
    case EPS: out[0] = h->knodes[p]; return 1;
    default: return 0;
    }
}

void oracle_ws_init(oracle_ws* ws, int32_t n) {
    ws->n = n;
    ws->seen = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
    ws->queue = (int32_t*)malloc((size_t)(n + 1) * sizeof(int32_t));
    ws->epoch = 0;
}

void oracle_ws_free(oracle_ws* ws) {
    free(ws->seen);
    free(ws->queue);
    ws->seen = NULL;
    ws->queue = NULL;
}

static uint32_t next_epoch(oracle_ws* ws) {
    if (++ws->epoch == 0) {
        memset(ws->seen, 0, (size_t)ws->n * sizeof(uint32_t));
        ws->epoch = 1;
    }
    return ws->epoch;
}

/* lockstep.cpp:10-35: the character nodes eps-reachable from s, FIFO order,
 * each address enqueued at most once; null members ignored. `out` receives
 * the Chr addresses in discovery order; returns their count. *enqueued (if
 * non-null) is incremented like LockstepStats::enqueued. */
int32_t oracle_evolve(const oracle_heap* h, oracle_ws* ws, const int32_t* s, int32_t ns, int32_t* out,
                      uint64_t* enqueued) {
    const uint32_t ep = next_epoch(ws);
    int32_t head = 0, tail = 0, nout = 0;
    for (int32_t i = 0; i < ns; ++i) {
        const int32_t p = s[i];
        if (p < 0 || ws->seen[p] == ep) continue;
        ws->seen[p] = ep;
        ws->queue[tail++] = p;
        if (enqueued) ++*enqueued;
    }
    while (head < tail) {
        const int32_t p = ws->queue[head++];
        if (h->nodes[p].kind == CHR) {
            out[nout++] = p;
            continue;
        }
        int32_t succ[2];
        const int k = eps_successors(h, p, succ);
        for (int j = 0; j < k; ++j) {
            const int32_t q = succ[j];
            if (q < 0 || ws->seen[q] == ep) continue;
            ws->seen[q] = ep;
            ws->queue[tail++] = q;
            if (enqueued) ++*enqueued;
        }
    }
    return nout;
}

/* lockstep.cpp:42-62 */
int oracle_eps_reaches_null(const oracle_heap* h, oracle_ws* ws, const int32_t* s, int32_t ns) {
    for (int32_t i = 0; i < ns; ++i)
        if (s[i] < 0) return 1;
    const uint32_t ep = next_epoch(ws);
    int32_t head = 0, tail = 0;
    for (int32_t i = 0; i < ns; ++i) {
        if (ws->seen[s[i]] == ep) continue;
        ws->seen[s[i]] = ep;
        ws->queue[tail++] = s[i];
    }
    while (head < tail) {
        const int32_t p = ws->queue[head++];
        int32_t succ[2];
        const int k = eps_successors(h, p, succ);
        for (int j = 0; j < k; ++j) {
            const int32_t q = succ[j];
            if (q < 0) return 1;
            if (ws->seen[q] == ep) continue;
            ws->seen[q] = ep;
            ws->queue[tail++] = q;
        }
    }
    return 0;
}

/* lockstep.cpp:64-73: knode of every Chr member labeled a (null skipped);
 * set semantics: duplicates removed. Returns the count, or -1 when a member
 * is neither null nor a Chr node (the reference throws invalid_argument). */
int32_t oracle_step_char(const oracle_heap* h, oracle_ws* ws, const int32_t* e, int32_t ne, uint32_t a,
                         int32_t* out) {
    const uint32_t ep = next_epoch(ws);
    int32_t nout = 0;
    int have_null = 0;
    for (int32_t i = 0; i < ne; ++i) {
        const int32_t p = e[i];
        if (p < 0) continue;
        if (h->nodes[p].kind != CHR) return -1;
        if (h->nodes[p].sym != a) continue;
        const int32_t q = h->knodes[p];
        if (q < 0) {
            if (!have_null) out[nout++] = -1;
            have_null = 1;
        } else if (ws->seen[q] != ep) {
            ws->seen[q] = ep;
            out[nout++] = q;
        }
    }
    return nout;
}

/* lockstep.cpp:75-82. Sets are kept as address lists; S holds at most n+1
 * entries (every address plus null). */
int oracle_lockstep_accepts(const oracle_heap* h, oracle_ws* ws, const uint32_t* w, uint64_t len,
                            int32_t* buf_a, int32_t* buf_b, uint64_t* enqueued) {
    int32_t* s = buf_a;
    int32_t* e = buf_b;
    int32_t ns = 1;
    s[0] = 0;
    for (uint64_t i = 0; i < len; ++i) {
        const int32_t ne = oracle_evolve(h, ws, s, ns, e, enqueued);
        ns = oracle_step_char(h, ws, e, ne, w[i], s);
        if (ns <= 0) return 0;
    }
    return oracle_eps_reaches_null(h, ws, s, ns);
}

/* lockstep.cpp:77-80 from an arbitrary start set: S <- step_char(evolve(S), a)
 * for each byte (bytes are the symbols here: ASCII inputs only), stopping early on the empty set. s_io holds the start set on
 * entry (n_io entries, null allowed) and the final set on exit; capacity n+1.
 * Used to verify a long single-string run chunk by chunk from checkpoints
 * (SURVEY.md §8(c) parity plan item 2). */
int32_t oracle_walk_from(const oracle_heap* h, int32_t* s_io, int32_t n_io, const uint8_t* bytes, uint64_t len) {
    oracle_ws ws;
    oracle_ws_init(&ws, h->n);
    int32_t* e = (int32_t*)malloc((size_t)(h->n + 1) * sizeof(int32_t));
    int32_t* t = (int32_t*)malloc((size_t)(h->n + 1) * sizeof(int32_t));
    int32_t ns = n_io;
    memcpy(t, s_io, (size_t)ns * sizeof(int32_t));
    for (uint64_t i = 0; i < len && ns > 0; ++i) {
        const int32_t ne = oracle_evolve(h, &ws, t, ns, e, NULL);
        ns = oracle_step_char(h, &ws, e, ne, bytes[i], t);
        if (ns < 0) ns = 0;
    }
    memcpy(s_io, t, (size_t)ns * sizeof(int32_t));
    free(e);
    free(t);
    oracle_ws_free(&ws);
    return ns;
}

/* rx::decode_utf8 (proj/src/utf8.cpp:16-46): bytes -> Unicode scalars.
 * Returns the number of scalars, or -1 where the reference throws
 * std::runtime_error (malformed, truncated, overlong, surrogate, > U+10FFFF). */
static int64_t decode_utf8(const uint8_t* s, uint64_t n, uint32_t* out) {
    static const uint32_t min_for_len[5] = {0, 0, 0x80, 0x800, 0x10000};
    uint64_t i = 0, k = 0;
    while (i < n) {
        const uint32_t b0 = s[i];
        if (b0 < 0x80) {
            out[k++] = b0;
            ++i;
            continue;
        }
        uint32_t len, cp;
        if ((b0 & 0xE0) == 0xC0) { len = 2; cp = b0 & 0x1F; }
        else if ((b0 & 0xF0) == 0xE0) { len = 3; cp = b0 & 0x0F; }
        else if ((b0 & 0xF8) == 0xF0) { len = 4; cp = b0 & 0x07; }
        else return -1;
        if (i + len > n) return -1;
        for (uint32_t j = 1; j < len; ++j) {
            const uint32_t b = s[i + j];
            if ((b & 0xC0) != 0x80) return -1;
            cp = (cp << 6) | (b & 0x3F);
        }
        if (cp < min_for_len[len] || cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return -1;
        out[k++] = cp;
        i += len;
    }
    return (int64_t)k;
}

/* One string as the `rxvm match` loop sees it (rxvm.cpp:85-87): decode_utf8,
 * then lockstep_accepts. A string decode_utf8 rejects (the reference throws)
 * counts as no match, the product's documented behaviour (include/rxg.h). */
static int accepts_utf8(const oracle_heap* h, oracle_ws* ws, const uint8_t* bytes, uint64_t len, uint32_t* w,
                        int32_t* a, int32_t* b) {
    const int64_t ns = decode_utf8(bytes, len, w);
    if (ns < 0) return 0;
    return oracle_lockstep_accepts(h, ws, w, (uint64_t)ns, a, b, NULL);
}

int oracle_accepts_bytes(const oracle_heap* h, const uint8_t* bytes, uint64_t len) {
    oracle_ws ws;
    oracle_ws_init(&ws, h->n);
    int32_t* a = (int32_t*)malloc((size_t)(h->n + 1) * sizeof(int32_t));
    int32_t* b = (int32_t*)malloc((size_t)(h->n + 1) * sizeof(int32_t));
    uint32_t* w = (uint32_t*)malloc((len ? len : 1) * sizeof(uint32_t));
    const int r = accepts_utf8(h, &ws, bytes, len, w, a, b);
    free(w);
    free(a);
    free(b);
    oracle_ws_free(&ws);
    return r;
}

/* ── batch driver (std::getline semantics of rxvm.cpp:100-112) ──────── */

typedef struct {
    const oracle_heap* h;
    const uint8_t* text;
    const uint64_t* starts;
    const uint64_t* lens;
    uint64_t nstr;
    uint8_t* results;
    int tid, nthreads;
    uint64_t count;
} job_t;

static void* run_job(void* arg) {
    job_t* j = (job_t*)arg;
    oracle_ws ws;
    oracle_ws_init(&ws, j->h->n);
    int32_t* a = (int32_t*)malloc((size_t)(j->h->n + 1) * sizeof(int32_t));
    int32_t* b = (int32_t*)malloc((size_t)(j->h->n + 1) * sizeof(int32_t));
    uint64_t cap = 1024;
    uint32_t* w = (uint32_t*)malloc(cap * sizeof(uint32_t));
    /* static interleaved partition, crosscheck.cpp:121 */
    for (uint64_t k = (uint64_t)j->tid; k < j->nstr; k += (uint64_t)j->nthreads) {
        const uint64_t len = j->lens[k];
        if (len > cap) {
            cap = len * 2;
            w = (uint32_t*)realloc(w, cap * sizeof(uint32_t));
        }
        const int r = accepts_utf8(j->h, &ws, j->text + j->starts[k], len, w, a, b);
        if (j->results) j->results[k] = (uint8_t)r;
        j->count += (uint64_t)r;
    }
    free(w);
    free(a);
    free(b);
    oracle_ws_free(&ws);
    return NULL;
}

uint64_t oracle_split(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* starts,
                      uint64_t* lens) {
    uint64_t n = 0;
    if (delimiter < 0) {
        for (uint64_t at = 0; at + stride <= len; at += stride) {
            if (starts) {
                starts[n] = at;
                lens[n] = stride;
            }
            ++n;
        }
        return n;
    }
    uint64_t at = 0;
    while (at < len) {
        const uint8_t* hit = (const uint8_t*)memchr(text + at, delimiter, len - at);
        const uint64_t end = hit ? (uint64_t)(hit - text) : len;
        if (starts) {
            starts[n] = at;
            lens[n] = end - at;
        }
        ++n;
        at = end + 1;
    }
    return n;
}

uint64_t oracle_match_batch(const oracle_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                            uint32_t stride, uint8_t* results, int nthreads) {
    const uint64_t n = oracle_split(text, len, delimiter, stride, NULL, NULL);
    uint64_t* starts = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* lens = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    oracle_split(text, len, delimiter, stride, starts, lens);
    if (nthreads < 1) nthreads = 1;
    job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (job_t){h, text, starts, lens, n, results, t, nthreads, 0};
        if (nthreads > 1) pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    if (nthreads == 1) run_job(&jobs[0]);
    uint64_t count = 0;
    for (int t = 0; t < nthreads; ++t) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        count += jobs[t].count;
    }
    free(jobs);
    free(th);
    free(starts);
    free(lens);
    return count;
}

/* rx::decode_utf8 (proj/src/utf8.cpp:16-46) restated: the index of the byte
 * named by its "invalid UTF-8 at byte N" error, or -1 when it decodes.
 * Checks in the reference's order: lead class, truncation, continuation
 * bytes, then overlong / surrogate / > U+10FFFF. */
int64_t oracle_decode_utf8_error(const uint8_t* s, uint64_t n) {
    static const uint32_t min_for_len[5] = {0, 0, 0x80, 0x800, 0x10000};
    uint64_t i = 0;
    while (i < n) {
        const uint32_t b0 = s[i];
        if (b0 < 0x80) {
            ++i;
            continue;
        }
        uint32_t len, cp;
        if ((b0 & 0xE0) == 0xC0) { len = 2; cp = b0 & 0x1F; }
        else if ((b0 & 0xF0) == 0xE0) { len = 3; cp = b0 & 0x0F; }
        else if ((b0 & 0xF8) == 0xF0) { len = 4; cp = b0 & 0x07; }
        else return (int64_t)i;
        if (i + len > n) return (int64_t)i;
        for (uint32_t k = 1; k < len; ++k) {
            const uint32_t b = s[i + k];
            if ((b & 0xC0) != 0x80) return (int64_t)(i + k);
            cp = (cp << 6) | (b & 0x3F);
        }
        if (cp < min_for_len[len]) return (int64_t)i;
        if (cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return (int64_t)i;
        i += len;
    }
    return -1;
}

/* decode_utf8 over every string of a buffer (the `rxvm match` getline loop,
 * rxvm.cpp:100-112): global offset of the first failing byte, or UINT64_MAX.
 * delimiter < 0 with stride 0: the whole buffer is one string. */
uint64_t oracle_utf8_first_bad(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride) {
    if (delimiter < 0 && stride == 0) {
        const int64_t e = oracle_decode_utf8_error(text, len);
        return e < 0 ? UINT64_MAX : (uint64_t)e;
    }
    const uint64_t n = oracle_split(text, len, delimiter, stride, NULL, NULL);
    uint64_t* starts = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* lens = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    oracle_split(text, len, delimiter, stride, starts, lens);
    uint64_t bad = UINT64_MAX;
    for (uint64_t k = 0; k < n && bad == UINT64_MAX; ++k) {
        const int64_t e = oracle_decode_utf8_error(text + starts[k], lens[k]);
        if (e >= 0) bad = starts[k] + (uint64_t)e;
    }
    free(starts);
    free(lens);
    return bad;
}
