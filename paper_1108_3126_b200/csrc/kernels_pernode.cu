// Single-string engines that follow the paper's §8 "thread per node" scheme.
//
// k_rounds  — the literal protocol of proj/src/parallel.cpp:50-190 inside one
//             CTA: one thread per heap node, counter vectors c/n with ±t
//             stamps in shared memory, CAS claim t -> -t (claim once), the
//             null continuation carried in accept_pending / accept_next,
//             repeated barrier-delimited rounds ("kernel launches" in the
//             paper) until no task schedules more work, then the c/n swap.
//             Used for parity of the paper's protocol and its instrumentation
//             (claims per node per step, rounds per step).
//
// k_pernode — K1: the same thread-per-node lockstep over the precomputed
//             closures of the position form (program.hpp). One warp; every
//             lane owns the ballot words of 32 Chr nodes (its slice of the
//             active set E). Per symbol:
//               fire = E & M[class(a)]                     (nodes that match a)
//               E'   = shift(fire & SH) | OR{ R[g] : g hit } (successors)
//             where shift is the one-bit successor of consecutive literals
//             (carry across lanes by shuffle) and R[g] are the deduplicated
//             residual follow rows; a group is "hit" when any firing node
//             triggers it (warp vote), so every distinct row is applied once
//             per step — the dedup-by-pointer-equality of the paper.
#include <cstdint>

#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>

#include "launch.hpp"
#include "pernode.hpp"

namespace rxg {

namespace cg = cooperative_groups;

namespace {

// ── k_rounds ──────────────────────────────────────────────────────────────

struct RoundsArgs {
    const uint8_t* text;
    uint64_t len;
    const uint8_t* kind;      // N
    const uint32_t* sym;      // N
    const int32_t* left;      // N
    const int32_t* right;     // N
    const int32_t* knode;     // N
    int32_t n;
    int32_t* accept;
    unsigned long long* stats;   // [claims, rounds, macro_steps, max_claims_per_node_step] or null
    uint32_t* trace;             // per symbol: next-schedule bitset ((N+1+31)/32 words, bit N = null), or null
    uint32_t trace_words;
    unsigned long long* enqueued;   // rx::LockstepStats.enqueued of the same run, or null (see below)
    uint32_t* schedule;             // per macro step: nodes scheduled at its start (ParStats.schedule_sizes), or null
};

enum : uint8_t { kEps = 0, kChr = 1, kAlt = 2, kSeq = 3, kStar = 4 };
constexpr uint32_t kEndOfInput = 0xFFFFFFFFu;   // parallel.hpp:43

__global__ void __launch_bounds__(1024) k_rounds(const __grid_constant__ RoundsArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int32_t N = a.n;
    int32_t* c = reinterpret_cast<int32_t*>(sm);
    int32_t* n = c + N;
    uint32_t* claims = reinterpret_cast<uint32_t*>(n + N);
    __shared__ int more, accept_pending, accept_next, any_n;
    __shared__ unsigned long long s_claims, s_rounds, s_steps, s_step_claims, s_eoi_claims;
    __shared__ uint32_t s_maxc, s_sched;
    for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
        c[i] = 0;
        n[i] = 0;
        claims[i] = 0;
    }
    if (threadIdx.x == 0) {
        accept_pending = accept_next = any_n = 0;
        s_claims = s_rounds = s_steps = s_step_claims = s_eoi_claims = 0;
        s_maxc = s_sched = 0;
    }
    __syncthreads();
    int32_t t = 1;
    if (threadIdx.x == 0) c[0] = t;   // schedule_root (parallel.cpp:14-17)
    int32_t* cur = c;
    int32_t* nxt = n;
    const bool instrument = a.stats || a.enqueued || a.schedule;
    for (uint64_t pos = 0; pos <= a.len; ++pos) {
        const uint32_t sym = pos < a.len ? static_cast<uint32_t>(a.text[pos]) : kEndOfInput;
        if (a.schedule) {   // |current_schedule()| at the macro step's start (parallel.cpp:160-161)
            uint32_t k = 0;
            for (int32_t i = threadIdx.x; i < N; i += blockDim.x) k += cur[i] == t;
            atomicAdd(&s_sched, k);
            __syncthreads();
            if (threadIdx.x == 0) {
                a.schedule[pos] = s_sched;
                s_sched = 0;
            }
        }
        // run_rounds (parallel.cpp:120-154)
        for (;;) {
            __syncthreads();
            if (threadIdx.x == 0) {
                more = 0;
                ++s_rounds;
            }
            __syncthreads();
            // dispatch list fixed at the round start, like run_rounds' scan
            // (parallel.cpp:125-127): nodes scheduled during this round wait
            // for the next one, so a stale read below can never re-arm a node
            // that is claimed in the same round.
            uint32_t mine = 0;
            for (int32_t i = threadIdx.x, b = 0; i < N; i += blockDim.x, ++b)
                if (cur[i] == t) mine |= 1u << b;
            __syncthreads();
            for (int32_t i = threadIdx.x, b = 0; i < N; i += blockDim.x, ++b) {
                if (!((mine >> b) & 1u)) continue;
                // par_task (parallel.cpp:50-78): claim t -> -t, exactly one winner
                if (atomicCAS(&cur[i], t, -t) != t) continue;
                claims[i] += 1;
                const uint8_t k = a.kind[i];
                if (k == kChr) {
                    if (sym != kEndOfInput && a.sym[i] == sym) {
                        const int32_t j = a.knode[i];
                        if (j < 0) accept_next = 1;
                        else nxt[j] = t + 1;
                        any_n = 1;
                    }
                    continue;
                }
                int32_t succ[2];
                int ns = 0;
                if (k == kAlt) { succ[0] = a.left[i]; succ[1] = a.right[i]; ns = 2; }
                else if (k == kSeq) { succ[0] = a.left[i]; ns = 1; }
                else if (k == kStar) { succ[0] = a.left[i]; succ[1] = a.knode[i]; ns = 2; }
                else { succ[0] = a.knode[i]; ns = 1; }
                for (int e = 0; e < ns; ++e) {
                    const int32_t q = succ[e];
                    if (q < 0) {
                        accept_pending = 1;
                        continue;
                    }
                    const int32_t v = cur[q];
                    if (v == t || v == -t) continue;   // already scheduled or simulated
                    cur[q] = t;                          // racing stores write the same value
                    more = 1;
                }
            }
            __syncthreads();
            if (!more) break;
        }
        // macro boundary: instrumentation + optional trace of the next schedule
        if (instrument) {
            uint32_t local = 0, mx = 0;
            for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
                local += claims[i];
                mx = max(mx, claims[i]);
                claims[i] = 0;
            }
            atomicAdd(&s_claims, static_cast<unsigned long long>(local));
            atomicAdd(&s_step_claims, static_cast<unsigned long long>(local));
            atomicMax(&s_maxc, mx);
            __syncthreads();
            if (threadIdx.x == 0) {
                ++s_steps;
                // the claims of one macro step are exactly the addresses
                // rx::evolve enqueues for the same set (both walk the eps
                // graph from S once, stopping at Chr nodes), so
                // LockstepStats.enqueued = every step's claims but the
                // end-of-input step's, which lockstep_accepts never runs
                if (pos == a.len) s_eoi_claims = s_step_claims;
                s_step_claims = 0;
            }
        }
        if (a.trace && pos < a.len) {
            uint32_t* row = a.trace + pos * a.trace_words;
            for (int32_t i = threadIdx.x; i < N; i += blockDim.x)
                if (nxt[i] == t + 1) atomicOr(&row[i >> 5], 1u << (i & 31));
            if (threadIdx.x == 0 && accept_next) atomicOr(&row[N >> 5], 1u << (N & 31));
        }
        __syncthreads();
        if (pos == a.len) break;
        // early reject (parallel.cpp:186): nothing scheduled and no null continuation
        const bool dead = !any_n && !accept_next;
        __syncthreads();
        if (dead) {
            if (threadIdx.x == 0) accept_pending = 0;
            break;
        }
        // swap_step (parallel.cpp:40-48)
        int32_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        ++t;
        __syncthreads();
        if (threadIdx.x == 0) {
            accept_pending = accept_next;
            accept_next = 0;
            any_n = 0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *a.accept = accept_pending;
        if (a.stats) {
            a.stats[0] = s_claims;
            a.stats[1] = s_rounds;
            a.stats[2] = s_steps;
            a.stats[3] = s_maxc;
        }
        if (a.enqueued) *a.enqueued = s_claims - s_eoi_claims;
    }
}

// ── k_par: one par_task or one run_rounds on caller-held state ──────────
//
// The reference's ParState (parallel.hpp:24-41) lives with the caller
// (int64 c/n stamps, claim counters, flags); this kernel applies either one
// par_task (parallel.cpp:50-78) to node `single`, or run_rounds
// (parallel.cpp:120-154): rounds over the dispatch list {i : c[i] == t},
// fixed at each round's start, until no task schedules more work. One CTA,
// one thread per node (strided), CAS claims on the global int64 stamps.
struct ParArgs {
    const uint8_t* kind;
    const uint32_t* sym;
    const int32_t* left;
    const int32_t* right;
    const int32_t* knode;
    int32_t n;
    long long* c;
    long long* nx;
    uint32_t* claims;
    int* flags;                  // more_c, any_n, accept_pending, accept_next
    long long t;
    uint32_t symbol;             // kEndOfInput: every Chr test fails
    int32_t single;              // >= 0: one par_task on this node; < 0: run_rounds
    unsigned long long* launches;
};

__device__ void par_task_dev(const ParArgs& a, int32_t i) {
    const long long t = a.t;
    if (atomicCAS(reinterpret_cast<unsigned long long*>(&a.c[i]), static_cast<unsigned long long>(t),
                  static_cast<unsigned long long>(-t)) != static_cast<unsigned long long>(t))
        return;
    atomicAdd(&a.claims[i], 1u);
    const uint8_t k = a.kind[i];
    if (k == kChr) {
        if (a.symbol != kEndOfInput && a.sym[i] == a.symbol) {
            const int32_t j = a.knode[i];
            if (j < 0) atomicExch(&a.flags[3], 1);
            else atomicExch(reinterpret_cast<unsigned long long*>(&a.nx[j]), static_cast<unsigned long long>(t + 1));
            atomicExch(&a.flags[1], 1);
        }
        return;
    }
    int32_t succ[2];
    int ns = 0;
    if (k == kAlt) { succ[0] = a.left[i]; succ[1] = a.right[i]; ns = 2; }
    else if (k == kSeq) { succ[0] = a.left[i]; ns = 1; }
    else if (k == kStar) { succ[0] = a.left[i]; succ[1] = a.knode[i]; ns = 2; }
    else { succ[0] = a.knode[i]; ns = 1; }
    for (int e = 0; e < ns; ++e) {
        const int32_t q = succ[e];
        if (q < 0) {
            atomicExch(&a.flags[2], 1);
            continue;
        }
        const long long v = *reinterpret_cast<volatile long long*>(&a.c[q]);
        if (v == t || v == -t) continue;   // already scheduled or simulated
        *reinterpret_cast<volatile long long*>(&a.c[q]) = t;   // racing stores write the same value
        atomicExch(&a.flags[0], 1);
    }
}

__global__ void __launch_bounds__(1024) k_par(const __grid_constant__ ParArgs a) {
    if (a.single >= 0) {
        if (threadIdx.x == 0) par_task_dev(a, a.single);
        return;
    }
    __shared__ unsigned long long launch;
    if (threadIdx.x == 0) launch = 0;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            a.flags[0] = 0;   // more_c
            ++launch;
        }
        uint32_t mine = 0;   // the dispatch list, fixed at the round start
        for (int32_t i = threadIdx.x, b = 0; i < a.n; i += blockDim.x, ++b)
            if (*reinterpret_cast<volatile long long*>(&a.c[i]) == a.t) mine |= 1u << b;
        __syncthreads();
        for (int32_t i = threadIdx.x, b = 0; i < a.n; i += blockDim.x, ++b)
            if ((mine >> b) & 1u) par_task_dev(a, i);
        __threadfence_block();
        __syncthreads();
        if (!*reinterpret_cast<volatile int*>(&a.flags[0])) break;
    }
    if (threadIdx.x == 0) *a.launches = launch;
}

// ── k_pernode (K1) ───────────────────────────────────────────────────────

constexpr int kMaxSlots = 8;        // words per lane: W <= 256 (8191 positions)
constexpr int kDenseGroups = 32;    // up to this many residual rows: vote per row, rows in smem
constexpr uint32_t kBitsetChunk = 4096;   // delimiter-scan chunk of the K2b line index

struct PernodeArgs {
    const uint8_t* text;
    uint64_t len;
    const uint8_t* cls;        // 256 byte classes
    const uint32_t* cmask;     // n_classes x W
    const uint32_t* shift;     // W
    const uint32_t* has_group; // W
    const int32_t* group;      // n_bits
    const uint32_t* rows;      // n_groups x W
    const uint32_t* trig;      // n_groups x W : positions whose residual is row g
    const uint32_t* init;      // W
    int32_t W, n_bits, n_groups, n_classes;
    int32_t byte_masks;        // 1: smem holds M per raw byte (256 x W), else per class
    uint32_t every;            // checkpoint period (0 = none)
    uint32_t* checkpoints;     // (len / every) x W words: E after every `every` symbols
    int32_t* accept;
    // segments (cooperative launch, one warp per segment; n_segs == 1: the one-warp walk)
    uint64_t seg;              // bytes per segment (multiple of 16)
    int32_t n_segs;
    uint32_t lookback;         // bytes walked from E0 before a segment to guess its entry set
    uint32_t* entry;           // n_segs x W: the entry set each segment last walked from
    uint32_t* exits;           // 2 x n_segs x W: exit sets (double-buffered across repair rounds)
    unsigned int* changed;     // 3 rotating round counters (zero when idle)
};

// One lockstep step of the warp-wide bitset. DENSE: <= 32 residual rows,
// each tested by a warp vote; otherwise hit rows are marked in a shared
// bitmap (claimed once per step) and OR-ed afterwards.
template <int SLOTS, bool DENSE, int GREG>
__device__ __forceinline__ void pernode_step(const PernodeArgs& a, const uint32_t (&Mw)[SLOTS], const uint32_t* TR,
                                             const uint32_t* RR, uint32_t* hit, int hw, int lane,
                                             uint32_t (&E)[SLOTS], const uint32_t (&SH)[SLOTS],
                                             const uint32_t (&HG)[SLOTS], const uint32_t (&TRr)[GREG ? GREG : 1][SLOTS],
                                             const uint32_t (&RRr)[GREG ? GREG : 1][SLOTS]) {
    const int W = a.W;
    uint32_t fire[SLOTS], nx[SLOTS];
    bool any_group = false;
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        fire[k] = E[k] & Mw[k];
        any_group |= (fire[k] & HG[k]) != 0u;
    }
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        // one-bit successor of consecutive literals; carry from word w-1
        const uint32_t sh = fire[k] & SH[k];
        uint32_t carry = __shfl_up_sync(0xFFFFFFFFu, sh >> 31, 1);
        const uint32_t wrap = __shfl_sync(0xFFFFFFFFu, k > 0 ? (fire[k - 1] & SH[k - 1]) >> 31 : 0u, 31);
        if (lane == 0) carry = wrap;
        nx[k] = (sh << 1) | carry;
    }
    if constexpr (GREG > 0) {
        // few residual rows: triggers and rows live in registers, one vote each
#pragma unroll
        for (int g = 0; g < GREG; ++g) {
            bool t = false;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) t |= (fire[k] & TRr[g][k]) != 0u;
            const bool h = __any_sync(0xFFFFFFFFu, t);
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) nx[k] |= h ? RRr[g][k] : 0u;
        }
    } else if (__any_sync(0xFFFFFFFFu, any_group)) {
        if constexpr (DENSE) {
            for (int g = 0; g < a.n_groups; ++g) {
                bool t = false;
#pragma unroll
                for (int k = 0; k < SLOTS; ++k) {
                    const int w = lane + 32 * k;
                    if (w < W) t |= (fire[k] & TR[g * W + w]) != 0u;
                }
                if (__any_sync(0xFFFFFFFFu, t)) {
#pragma unroll
                    for (int k = 0; k < SLOTS; ++k) {
                        const int w = lane + 32 * k;
                        if (w < W) nx[k] |= RR[g * W + w];
                    }
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                uint32_t f = fire[k] & HG[k];
                while (f) {
                    const int b = __ffs(f) - 1;
                    f &= f - 1;
                    const int g = __ldg(a.group + (lane + 32 * k) * 32 + b);
                    atomicOr(&hit[g >> 5], 1u << (g & 31));
                }
            }
            __syncwarp();
            for (int hwi = 0; hwi < hw; ++hwi) {
                uint32_t m = hit[hwi];
                while (m) {
                    const int g = hwi * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    const uint32_t* R = a.rows + static_cast<size_t>(g) * W;
#pragma unroll
                    for (int k = 0; k < SLOTS; ++k) {
                        const int w = lane + 32 * k;
                        if (w < W) nx[k] |= __ldg(R + w);
                    }
                }
            }
            __syncwarp();
            for (int i = lane; i < hw; i += 32) hit[i] = 0;
            __syncwarp();
        }
    }
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) E[k] = nx[k];
}

template <int SLOTS, bool DENSE, int GREG>
__global__ void __launch_bounds__(32) k_pernode(const __grid_constant__ PernodeArgs a) {
    // K1 over one long string, the paper's scheme per warp. With several
    // segments (north_star (2) first bullet, scaled across SMs): warp s walks
    // [s*seg, (s+1)*seg) from a guessed entry set (E0 walked over the
    // `lookback` bytes before the segment), the exit sets are published, and
    // repair rounds re-walk every segment whose entry differs from its
    // predecessor's current exit until no entry changes. Sets are compared
    // word for word, so the result is exactly the one-warp walk's.
    extern __shared__ __align__(16) uint32_t smp[];
    const int W = a.W;
    const int lane = threadIdx.x;
    // shared layout: masks (256 x W by byte, or n_classes x W by class), then
    // the dense rows + triggers, or the sparse hit bitmap; then the class map
    uint32_t* masks = smp;
    const int mrows = a.byte_masks ? 256 : a.n_classes;
    uint32_t* TR = masks + mrows * W;
    uint32_t* RR = TR + (DENSE ? a.n_groups * W : 0);
    uint32_t* hit = RR + (DENSE ? a.n_groups * W : 0);
    const int hw = DENSE ? 0 : (a.n_groups + 31) / 32;
    uint8_t* cls = reinterpret_cast<uint8_t*>(hit + hw);
    for (int i = lane; i < 256; i += 32) cls[i] = a.cls[i];
    __syncwarp();
    for (int i = lane; i < mrows * W; i += 32)
        masks[i] = a.byte_masks ? a.cmask[cls[i / W] * W + i % W] : a.cmask[i];
    if (DENSE)
        for (int i = lane; i < a.n_groups * W; i += 32) {
            TR[i] = a.trig[i];
            RR[i] = a.rows[i];
        }
    for (int i = lane; i < hw; i += 32) hit[i] = 0;
    uint32_t E[SLOTS], SH[SLOTS], HG[SLOTS];
    uint32_t TRr[GREG ? GREG : 1][SLOTS], RRr[GREG ? GREG : 1][SLOTS];
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        const int w = lane + 32 * k;
        E[k] = w < W ? a.init[w] : 0u;
        SH[k] = w < W ? a.shift[w] : 0u;
        HG[k] = w < W ? a.has_group[w] : 0u;
#pragma unroll
        for (int g = 0; g < (GREG ? GREG : 1); ++g) {
            TRr[g][k] = (GREG && g < a.n_groups && w < W) ? a.trig[g * W + w] : 0u;
            RRr[g][k] = (GREG && g < a.n_groups && w < W) ? a.rows[g * W + w] : 0u;
        }
    }
    __syncwarp();
    uint64_t pos = 0;
    bool live = true;
    auto rowp = [&](uint32_t b) { return a.byte_masks ? masks + b * W : masks + cls[b] * W; };
    auto one = [&](const uint32_t (&Mw)[SLOTS]) {
        pernode_step<SLOTS, DENSE, GREG>(a, Mw, TR, RR, hit, hw, lane, E, SH, HG, TRr, RRr);
        ++pos;
        if (a.every && pos % a.every == 0) {
            uint32_t* out = a.checkpoints + (pos / a.every - 1) * W;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k)
                if (lane + 32 * k < W) out[lane + 32 * k] = E[k];
        }
    };
    auto single = [&](uint32_t b) {
        const uint32_t* M = rowp(b);
        uint32_t Mw[SLOTS];
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) Mw[k] = lane + 32 * k < W ? M[lane + 32 * k] : 0u;
        one(Mw);
    };
    auto walk = [&](uint64_t lo, uint64_t hi) {
    pos = lo;
    live = true;
    // 16 input bytes per uniform load (every lane reads the same vector)
    const uint64_t head = (16 - (reinterpret_cast<uintptr_t>(a.text + lo) & 15)) & 15;
    for (uint64_t i = 0; i < head && pos < hi; ++i) single(a.text[pos]);
    while (live && pos + 16 <= hi) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        // the 16 mask rows depend only on the input: load them all before the
        // dependent chain of 16 steps starts
        uint32_t Mw[16][SLOTS];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t* M = rowp((wv[i >> 2] >> (8 * (i & 3))) & 0xFFu);
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) Mw[i][k] = lane + 32 * k < W ? M[lane + 32 * k] : 0u;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) one(Mw[i]);
        if ((pos & 63) == 0) {   // the empty set is absorbing: stop early
            bool any = false;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) any |= E[k] != 0u;
            live = __any_sync(0xFFFFFFFFu, any);
        }
    }
    while (live && pos < hi) single(a.text[pos]);
    };
    const int A = a.n_bits - 1;   // accept bit
    if (a.n_segs > 1) {
        const int s = static_cast<int>(blockIdx.x);
        const uint64_t lo = static_cast<uint64_t>(s) * a.seg, hi = min(lo + a.seg, a.len);
        auto put = [&](uint32_t* dst) {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k)
                if (lane + 32 * k < W) dst[lane + 32 * k] = E[k];
        };
        auto get = [&](const uint32_t* src) {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) E[k] = lane + 32 * k < W ? __ldcg(src + lane + 32 * k) : 0u;
        };
        if (s > 0) walk(lo >= a.lookback ? lo - a.lookback : 0, lo);   // the guess (from E0)
        const size_t sw = static_cast<size_t>(W);
        put(a.entry + s * sw);
        walk(lo, hi);
        put(a.exits + s * sw);
        cg::grid_group grid = cg::this_grid();
        __threadfence();
        grid.sync();
        // Round r counts its re-walked segments in changed[r % 3]; every block
        // reads that counter after the round's grid sync. Block 0 zeroes the
        // next round's counter during round r: its last use (round r - 2) was
        // read by every block before they passed round r - 1's sync. (With
        // two counters the reset raced with slow readers of the current one:
        // a block could see 0 and leave while the others waited at the next
        // sync.)
        for (int r = 0;; ++r) {
            const uint32_t* prev = a.exits + static_cast<size_t>(r & 1) * a.n_segs * sw;
            uint32_t* next = a.exits + static_cast<size_t>((r + 1) & 1) * a.n_segs * sw;
            if (s == 0 && lane == 0) a.changed[(r + 1) % 3] = 0;
            bool diff = false;
            if (s > 0)
                for (int w = lane; w < W; w += 32) diff |= __ldcg(prev + (s - 1) * sw + w) != __ldcg(a.entry + s * sw + w);
            if (__any_sync(0xFFFFFFFFu, diff)) {   // re-walk from the predecessor's current exit
                get(prev + (s - 1) * sw);
                put(a.entry + s * sw);
                walk(lo, hi);
                put(next + s * sw);
                if (lane == 0) atomicAdd(&a.changed[r % 3], 1u);
            } else {
                for (int w = lane; w < W; w += 32) next[s * sw + w] = __ldcg(prev + s * sw + w);
            }
            __threadfence();
            grid.sync();
            if (*reinterpret_cast<volatile unsigned int*>(&a.changed[r % 3]) == 0) {
                if (s == a.n_segs - 1) {
                    get(next + s * sw);
                    uint32_t acc = 0;
#pragma unroll
                    for (int k = 0; k < SLOTS; ++k)
                        if (lane + 32 * k == (A >> 5)) acc = (E[k] >> (A & 31)) & 1u;
                    acc = __reduce_or_sync(0xFFFFFFFFu, acc);
                    if (lane == 0) {
                        *a.accept = static_cast<int32_t>(acc);
                        a.changed[(r + 2) % 3] = 0;   // the previous round's (all blocks read it before this sync)
                    }
                }
                return;
            }
        }
    }
    walk(0, a.len);
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < SLOTS; ++k)
        if (lane + 32 * k == (A >> 5)) acc = (E[k] >> (A & 31)) & 1u;
    acc = __reduce_or_sync(0xFFFFFFFFu, acc);
    if (lane == 0) *a.accept = static_cast<int32_t>(acc);
}

template <int SLOTS, bool DENSE, int GREG>
cudaError_t run_pernode(const PernodeArgs& a, uint32_t smem, cudaStream_t st) {
    auto* k = k_pernode<SLOTS, DENSE, GREG>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (a.n_segs <= 1) {
        k<<<1, 32, smem, st>>>(a);
        return cudaGetLastError();
    }
    PernodeArgs b = a;
    void* args[] = {&b};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(a.n_segs), dim3(32), args, smem, st);
}

// Resident one-warp blocks per SM of the segmented K1 kernel (segments are capped by it).
template <int SLOTS, bool DENSE, int GREG>
int pernode_per_sm(uint32_t smem) {
    auto* k = k_pernode<SLOTS, DENSE, GREG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 32, smem);
    return n;
}

template <bool D, int G>
struct Tag {
    static constexpr bool dense = D;
    static constexpr int greg = G;
};

template <int SLOTS>
cudaError_t run_pernode2(PernodeArgs a, uint32_t smem, bool dense, cudaStream_t st, uint64_t seg_want,
                         const PernodeSegScratch* ss) {
    auto launch = [&](auto tag) {
        using T = decltype(tag);
        if (ss && seg_want) {   // segments across SMs: as many as are co-resident (cooperative launch)
            const int per = pernode_per_sm<SLOTS, T::dense, T::greg>(smem);
            int dev = 0;
            cudaGetDevice(&dev);
            const uint64_t cap = static_cast<uint64_t>(per > 0 ? per : 1) * device_sm_count(dev);
            uint64_t n = (a.len + seg_want - 1) / seg_want;
            if (n > cap) n = cap;
            if (n > ss->max_segs) n = ss->max_segs;
            if (n > 1) {
                a.seg = ((a.len + n - 1) / n + 15) / 16 * 16;
                a.n_segs = static_cast<int32_t>((a.len + a.seg - 1) / a.seg);
                a.entry = ss->entry;
                a.exits = ss->exits;
                a.changed = ss->changed;
            }
        }
        return run_pernode<SLOTS, T::dense, T::greg>(a, smem, st);
    };
    if (a.n_groups <= 1) return launch(Tag<true, 1>{});
    if (a.n_groups <= 2) return launch(Tag<true, 2>{});
    return dense ? launch(Tag<true, 0>{}) : launch(Tag<false, 0>{});
}

// ── K2b: warp-per-line bitset lockstep for batches ───────────────────────
//
// The bitset variant of the batch path (no memoized DFA: works for patterns
// whose DFA would explode). Every warp walks whole lines with the K1 step,
// its lanes holding the ballot words of the active set; tables are shared by
// the CTA's warps. Line boundaries come from a delimiter-position pass.

struct BitsetLinesArgs {
    PernodeArgs p;                       // tables (p.text / p.len unused)
    const uint8_t* text;
    uint64_t len;
    const unsigned long long* dpos;      // positions of the delimiters, ascending
    const unsigned long long* ndelim;    // device: number of delimiters
    unsigned long long* count;
    uint8_t* results;
};

template <int SLOTS, bool DENSE, int GREG>
__global__ void __launch_bounds__(256) k_lines_bitset(const __grid_constant__ BitsetLinesArgs b) {
    extern __shared__ __align__(16) uint32_t smp[];
    const PernodeArgs& a = b.p;
    const int W = a.W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t* masks = smp;
    const int mrows = a.byte_masks ? 256 : a.n_classes;
    uint32_t* TR = masks + mrows * W;
    uint32_t* RR = TR + (DENSE ? a.n_groups * W : 0);
    const int hw = DENSE ? 0 : (a.n_groups + 31) / 32;
    uint32_t* hit_all = RR + (DENSE ? a.n_groups * W : 0);
    uint8_t* cls = reinterpret_cast<uint8_t*>(hit_all + hw * nw);
    uint32_t* hit = hit_all + hw * warp;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cls[i] = a.cls[i];
    __syncthreads();
    for (int i = threadIdx.x; i < mrows * W; i += blockDim.x)
        masks[i] = a.byte_masks ? a.cmask[cls[i / W] * W + i % W] : a.cmask[i];
    if (DENSE)
        for (int i = threadIdx.x; i < a.n_groups * W; i += blockDim.x) {
            TR[i] = a.trig[i];
            RR[i] = a.rows[i];
        }
    for (int i = threadIdx.x; i < hw * nw; i += blockDim.x) hit_all[i] = 0;
    uint32_t SH[SLOTS], HG[SLOTS], I0[SLOTS];
    uint32_t TRr[GREG ? GREG : 1][SLOTS], RRr[GREG ? GREG : 1][SLOTS];
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        const int w = lane + 32 * k;
        I0[k] = w < W ? a.init[w] : 0u;
        SH[k] = w < W ? a.shift[w] : 0u;
        HG[k] = w < W ? a.has_group[w] : 0u;
#pragma unroll
        for (int g = 0; g < (GREG ? GREG : 1); ++g) {
            TRr[g][k] = (GREG && g < a.n_groups && w < W) ? a.trig[g * W + w] : 0u;
            RRr[g][k] = (GREG && g < a.n_groups && w < W) ? a.rows[g * W + w] : 0u;
        }
    }
    __syncthreads();
    const unsigned long long nd = *b.ndelim;
    // a final segment after the last delimiter is a line (std::getline)
    const unsigned long long nlines = nd + ((b.len > 0 && (nd == 0 || b.dpos[nd - 1] != b.len - 1)) ? 1ull : 0ull);
    const int A = a.n_bits - 1;
    uint32_t cnt = 0;
    auto rowp = [&](uint32_t byte) { return a.byte_masks ? masks + byte * W : masks + cls[byte] * W; };
    for (unsigned long long line = static_cast<unsigned long long>(blockIdx.x) * nw + warp; line < nlines;
         line += static_cast<unsigned long long>(gridDim.x) * nw) {
        const uint64_t lo = line == 0 ? 0 : b.dpos[line - 1] + 1;
        const uint64_t hi = line < nd ? b.dpos[line] : b.len;
        uint32_t E[SLOTS];
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) E[k] = I0[k];
        uint64_t pos = lo;
        bool live = true;
        while (live && pos + 16 <= hi) {
            uint32_t by[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) by[i] = __ldg(b.text + pos + i);
            uint32_t Mw[16][SLOTS];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t* M = rowp(by[i]);
#pragma unroll
                for (int k = 0; k < SLOTS; ++k) Mw[i][k] = lane + 32 * k < W ? M[lane + 32 * k] : 0u;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) pernode_step<SLOTS, DENSE, GREG>(a, Mw[i], TR, RR, hit, hw, lane, E, SH, HG, TRr, RRr);
            pos += 16;
            bool any = false;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) any |= E[k] != 0u;
            live = __any_sync(0xFFFFFFFFu, any);
        }
        for (; live && pos < hi; ++pos) {
            const uint32_t* M = rowp(__ldg(b.text + pos));
            uint32_t Mw[SLOTS];
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) Mw[k] = lane + 32 * k < W ? M[lane + 32 * k] : 0u;
            pernode_step<SLOTS, DENSE, GREG>(a, Mw, TR, RR, hit, hw, lane, E, SH, HG, TRr, RRr);
        }
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < SLOTS; ++k)
            if (lane + 32 * k == (A >> 5)) acc = (E[k] >> (A & 31)) & 1u;
        acc = __reduce_or_sync(0xFFFFFFFFu, acc);
        if (lane == 0) {
            if (b.results) b.results[line] = static_cast<uint8_t>(acc);
            cnt += acc;
        }
    }
    if (lane == 0 && cnt) atomicAdd(b.count, static_cast<unsigned long long>(cnt));
}

template <int SLOTS, bool DENSE, int GREG>
cudaError_t run_lines_bitset(const BitsetLinesArgs& b, uint32_t smem, int device, cudaStream_t st) {
    auto kern = k_lines_bitset<SLOTS, DENSE, GREG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    kern<<<per_sm * sms, 256, smem, st>>>(b);
    return cudaGetLastError();
}

template <int SLOTS>
cudaError_t run_lines_bitset2(const BitsetLinesArgs& b, uint32_t smem, bool dense, int device, cudaStream_t st) {
    if (b.p.n_groups <= 1) return run_lines_bitset<SLOTS, true, 1>(b, smem, device, st);
    if (b.p.n_groups <= 2) return run_lines_bitset<SLOTS, true, 2>(b, smem, device, st);
    return dense ? run_lines_bitset<SLOTS, true, 0>(b, smem, device, st)
                 : run_lines_bitset<SLOTS, false, 0>(b, smem, device, st);
}

// Delimiter positions: per chunk count -> scan (host side, cub) -> positions.
__global__ void __launch_bounds__(256) k_delim_pos(const uint8_t* __restrict__ text, uint64_t len, uint32_t chunk,
                                                   uint64_t nchunks, uint32_t delim,
                                                   const unsigned long long* __restrict__ base,
                                                   unsigned long long* __restrict__ dpos) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint64_t c0 = c * chunk, c1 = min(c0 + chunk, len);
    unsigned long long k = base[c];
    for (uint64_t p = c0; p < c1; ++p)
        if (text[p] == delim) dpos[k++] = p;
}

__global__ void __launch_bounds__(256) k_delim_count(const uint8_t* __restrict__ text, uint64_t len, uint32_t chunk,
                                                     uint64_t nchunks, uint32_t delim,
                                                     unsigned long long* __restrict__ out) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c > nchunks) return;
    if (c == nchunks) {   // trailing zero so the exclusive scan yields the total at [nchunks]
        out[c] = 0;
        return;
    }
    const uint64_t c0 = c * chunk, c1 = min(c0 + chunk, len);
    unsigned long long n = 0;
    for (uint64_t p = c0; p < c1; ++p) n += text[p] == delim;
    out[c] = n;
}

}  // namespace

cudaError_t launch_par(const RoundsTables& t, long long* c, long long* n, uint32_t* claims, int* flags, long long tt,
                       uint32_t symbol, int32_t single, unsigned long long* launches, cudaStream_t st) {
    ParArgs a{};
    a.kind = t.kind;
    a.sym = t.sym;
    a.left = t.left;
    a.right = t.right;
    a.knode = t.knode;
    a.n = t.n;
    a.c = c;
    a.nx = n;
    a.claims = claims;
    a.flags = flags;
    a.t = tt;
    a.symbol = symbol;
    a.single = single;
    a.launches = launches;
    k_par<<<1, 1024, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rounds(const RoundsTables& t, const uint8_t* text, uint64_t len, int32_t* accept,
                          unsigned long long* stats, uint32_t* trace, cudaStream_t st,
                          unsigned long long* enqueued, uint32_t* schedule) {
    RoundsArgs a{};
    a.text = text;
    a.len = len;
    a.kind = t.kind;
    a.sym = t.sym;
    a.left = t.left;
    a.right = t.right;
    a.knode = t.knode;
    a.n = t.n;
    a.accept = accept;
    a.stats = stats;
    a.trace = trace;
    a.trace_words = static_cast<uint32_t>((t.n + 1 + 31) / 32);
    a.enqueued = enqueued;
    a.schedule = schedule;
    const uint32_t smem = static_cast<uint32_t>(t.n) * 12u;
    cudaError_t e = cudaFuncSetAttribute(k_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k_rounds<<<1, 1024, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pernode(const PernodeTables& t, const uint8_t* text, uint64_t len, uint32_t every,
                           uint32_t* checkpoints, int32_t* accept, cudaStream_t st, const PernodeSegScratch* ss) {
    PernodeArgs a{};
    a.text = text;
    a.len = len;
    a.cls = t.cls;
    a.cmask = t.cmask;
    a.shift = t.shift;
    a.has_group = t.has_group;
    a.group = t.group;
    a.rows = t.rows;
    a.trig = t.trig;
    a.init = t.init;
    a.W = t.W;
    a.n_bits = t.n_bits;
    a.n_groups = t.n_groups;
    a.n_classes = t.n_classes;
    a.every = every;
    a.checkpoints = checkpoints;
    a.accept = accept;
    a.n_segs = 1;
    a.lookback = kPernodeLookback;
    // segments only without checkpoints and for long strings
    const uint64_t seg_want = (ss && !every && len >= kPernodeSegMin) ? kPernodeSegMin / 4 : 0;
    const bool dense = t.n_groups <= kDenseGroups;
    // segments: class-indexed masks keep a warp's shared memory small (more warps per SM)
    a.byte_masks = !seg_want && 256u * static_cast<uint32_t>(t.W) * 4u <= 128u * 1024u;
    const uint32_t mrows = a.byte_masks ? 256u : static_cast<uint32_t>(t.n_classes);
    const uint32_t group_words = dense ? 2u * static_cast<uint32_t>(t.n_groups * t.W)
                                       : static_cast<uint32_t>((t.n_groups + 31) / 32);
    const uint32_t smem = (mrows * static_cast<uint32_t>(t.W) + group_words) * 4u + 256u;
    const int slots = (t.W + 31) / 32;
    if (slots <= 1) return run_pernode2<1>(a, smem, dense, st, seg_want, ss);
    if (slots <= 2) return run_pernode2<2>(a, smem, dense, st, seg_want, ss);
    if (slots <= 3) return run_pernode2<3>(a, smem, dense, st, seg_want, ss);
    if (slots <= 4) return run_pernode2<4>(a, smem, dense, st, seg_want, ss);
    if (slots <= kMaxSlots) return run_pernode2<kMaxSlots>(a, smem, dense, st, seg_want, ss);
    return cudaErrorInvalidValue;
}

size_t lines_bitset_scratch_bytes(uint64_t len) {
    const uint64_t nchunks = (len + kBitsetChunk - 1) / kBitsetChunk;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<int64_t>(nchunks + 1));
    // counts, base, positions (at most one per byte), cub temp
    return (2 * (nchunks + 1) + len + 1) * sizeof(unsigned long long) + temp + 256;
}

cudaError_t launch_lines_bitset(const PernodeTables& t, const uint8_t* text, uint64_t len, uint8_t delim,
                                unsigned long long* count, uint8_t* results, void* scratch, size_t scratch_bytes,
                                int device, cudaStream_t st) {
    if (len == 0) return cudaSuccess;
    const uint64_t nchunks = (len + kBitsetChunk - 1) / kBitsetChunk;
    unsigned long long* counts = static_cast<unsigned long long*>(scratch);
    unsigned long long* base = counts + nchunks + 1;
    unsigned long long* dpos = base + nchunks + 1;
    void* temp = dpos + len + 1;
    size_t temp_bytes = scratch_bytes - (2 * (nchunks + 1) + len + 1) * sizeof(unsigned long long);
    const unsigned g = static_cast<unsigned>((nchunks + 1 + 255) / 256);
    k_delim_count<<<g, 256, 0, st>>>(text, len, kBitsetChunk, nchunks, delim, counts);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, base, static_cast<int64_t>(nchunks + 1), st);
    if (e != cudaSuccess) return e;
    k_delim_pos<<<g, 256, 0, st>>>(text, len, kBitsetChunk, nchunks, delim, base, dpos);
    BitsetLinesArgs b{};
    PernodeArgs& a = b.p;
    a.cls = t.cls;
    a.cmask = t.cmask;
    a.shift = t.shift;
    a.has_group = t.has_group;
    a.group = t.group;
    a.rows = t.rows;
    a.trig = t.trig;
    a.init = t.init;
    a.W = t.W;
    a.n_bits = t.n_bits;
    a.n_groups = t.n_groups;
    a.n_classes = t.n_classes;
    const bool dense = t.n_groups <= kDenseGroups;
    a.byte_masks = 256u * static_cast<uint32_t>(t.W) * 4u <= 96u * 1024u;
    b.text = text;
    b.len = len;
    b.dpos = dpos;
    b.ndelim = base + nchunks;
    b.count = count;
    b.results = results;
    const uint32_t mrows = a.byte_masks ? 256u : static_cast<uint32_t>(t.n_classes);
    const uint32_t group_words = dense ? 2u * static_cast<uint32_t>(t.n_groups * t.W)
                                       : 8u * static_cast<uint32_t>((t.n_groups + 31) / 32);
    const uint32_t smem = (mrows * static_cast<uint32_t>(t.W) + group_words) * 4u + 256u;
    const int slots = (t.W + 31) / 32;
    if (slots <= 1) return run_lines_bitset2<1>(b, smem, dense, device, st);
    if (slots <= 2) return run_lines_bitset2<2>(b, smem, dense, device, st);
    if (slots <= 3) return run_lines_bitset2<3>(b, smem, dense, device, st);
    if (slots <= 4) return run_lines_bitset2<4>(b, smem, dense, device, st);
    if (slots <= kMaxSlots) return run_lines_bitset2<kMaxSlots>(b, smem, dense, device, st);
    return cudaErrorInvalidValue;
}

}  // namespace rxg
