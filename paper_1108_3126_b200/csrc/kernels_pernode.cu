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

#include "pernode.hpp"

namespace rxg {

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
    __shared__ unsigned long long s_claims, s_rounds, s_steps;
    __shared__ uint32_t s_maxc;
    for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
        c[i] = 0;
        n[i] = 0;
        claims[i] = 0;
    }
    if (threadIdx.x == 0) {
        accept_pending = accept_next = any_n = 0;
        s_claims = s_rounds = s_steps = 0;
        s_maxc = 0;
    }
    __syncthreads();
    int32_t t = 1;
    if (threadIdx.x == 0) c[0] = t;   // schedule_root (parallel.cpp:14-17)
    int32_t* cur = c;
    int32_t* nxt = n;
    for (uint64_t pos = 0; pos <= a.len; ++pos) {
        const uint32_t sym = pos < a.len ? static_cast<uint32_t>(a.text[pos]) : kEndOfInput;
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
        if (a.stats) {
            uint32_t local = 0, mx = 0;
            for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
                local += claims[i];
                mx = max(mx, claims[i]);
                claims[i] = 0;
            }
            atomicAdd(&s_claims, static_cast<unsigned long long>(local));
            atomicMax(&s_maxc, mx);
            if (threadIdx.x == 0) ++s_steps;
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
    }
}

// ── k_pernode (K1) ───────────────────────────────────────────────────────

constexpr int kMaxSlots = 8;   // words per lane: W <= 256 (8191 positions)

struct PernodeArgs {
    const uint8_t* text;
    uint64_t len;
    const uint8_t* cls;        // 256 byte classes
    const uint32_t* cmask;     // n_classes x W
    const uint32_t* shift;     // W
    const uint32_t* has_group; // W
    const int32_t* group;      // n_bits
    const uint32_t* rows;      // n_groups x W
    const uint32_t* init;      // W
    int32_t W, n_bits, n_groups, n_classes;
    uint32_t every;            // checkpoint period (0 = none)
    uint32_t* checkpoints;     // (len / every) x W words: E after every `every` symbols
    int32_t* accept;
};

template <int SLOTS>
__global__ void __launch_bounds__(32) k_pernode(const __grid_constant__ PernodeArgs a) {
    extern __shared__ __align__(16) uint32_t smp[];
    const int W = a.W;
    uint32_t* cm = smp;                                   // class masks
    uint32_t* hit = cm + a.n_classes * W;                 // hit-group bitmap
    const int hw = (a.n_groups + 31) / 32;
    uint8_t* cls = reinterpret_cast<uint8_t*>(hit + hw);
    const int lane = threadIdx.x;
    for (int i = lane; i < a.n_classes * W; i += 32) cm[i] = a.cmask[i];
    for (int i = lane; i < 256; i += 32) cls[i] = a.cls[i];
    for (int i = lane; i < hw; i += 32) hit[i] = 0;
    uint32_t E[SLOTS], SH[SLOTS], HG[SLOTS];
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        const int w = lane + 32 * k;
        E[k] = w < W ? a.init[w] : 0u;
        SH[k] = w < W ? a.shift[w] : 0u;
        HG[k] = w < W ? a.has_group[w] : 0u;
    }
    __syncwarp();
    uint64_t pos = 0;
    for (; pos < a.len; ++pos) {
        const uint32_t c = cls[a.text[pos]];
        const uint32_t* M = cm + c * W;
        uint32_t fire[SLOTS], nx[SLOTS];
        bool any_group = false;
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) {
            const int w = lane + 32 * k;
            fire[k] = w < W ? (E[k] & M[w]) : 0u;
            // one-bit successor of consecutive literals; carry from word w-1
            const uint32_t sh = fire[k] & SH[k];
            uint32_t carry = __shfl_up_sync(0xFFFFFFFFu, sh >> 31, 1);
            const uint32_t wrap = __shfl_sync(0xFFFFFFFFu, k > 0 ? (fire[k - 1] & SH[k - 1]) >> 31 : 0u, 31);
            if (lane == 0) carry = wrap;
            nx[k] = (sh << 1) | carry;
            any_group |= (fire[k] & HG[k]) != 0u;
        }
        // residual rows: mark each hit group once, then OR its row (dedup by row identity)
        if (__any_sync(0xFFFFFFFFu, any_group)) {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                uint32_t f = fire[k] & HG[k];
                while (f) {
                    const int b = __ffs(f) - 1;
                    f &= f - 1;
                    const int g = a.group[(lane + 32 * k) * 32 + b];
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
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) E[k] = nx[k];
        if (a.every && (pos + 1) % a.every == 0) {
            uint32_t* out = a.checkpoints + ((pos + 1) / a.every - 1) * W;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k)
                if (lane + 32 * k < W) out[lane + 32 * k] = E[k];
        }
        if ((pos & 63) == 63) {   // the empty set is absorbing: stop early
            bool live = false;
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) live |= E[k] != 0u;
            if (!__any_sync(0xFFFFFFFFu, live)) {
                ++pos;
                break;
            }
        }
    }
    const int A = a.n_bits - 1;   // accept bit
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < SLOTS; ++k)
        if (lane + 32 * k == (A >> 5)) acc = (E[k] >> (A & 31)) & 1u;
    acc = __reduce_or_sync(0xFFFFFFFFu, acc);
    if (lane == 0) *a.accept = static_cast<int32_t>(acc);
}

template <int SLOTS>
cudaError_t run_pernode(const PernodeArgs& a, uint32_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_pernode<SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k_pernode<SLOTS><<<1, 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rounds(const RoundsTables& t, const uint8_t* text, uint64_t len, int32_t* accept,
                          unsigned long long* stats, uint32_t* trace, cudaStream_t st) {
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
    const uint32_t smem = static_cast<uint32_t>(t.n) * 12u;
    cudaError_t e = cudaFuncSetAttribute(k_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k_rounds<<<1, 1024, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pernode(const PernodeTables& t, const uint8_t* text, uint64_t len, uint32_t every,
                           uint32_t* checkpoints, int32_t* accept, cudaStream_t st) {
    PernodeArgs a{};
    a.text = text;
    a.len = len;
    a.cls = t.cls;
    a.cmask = t.cmask;
    a.shift = t.shift;
    a.has_group = t.has_group;
    a.group = t.group;
    a.rows = t.rows;
    a.init = t.init;
    a.W = t.W;
    a.n_bits = t.n_bits;
    a.n_groups = t.n_groups;
    a.n_classes = t.n_classes;
    a.every = every;
    a.checkpoints = checkpoints;
    a.accept = accept;
    const uint32_t smem = static_cast<uint32_t>(t.n_classes * t.W + (t.n_groups + 31) / 32) * 4u + 256u;
    const int slots = (t.W + 31) / 32;
    if (slots <= 1) return run_pernode<1>(a, smem, st);
    if (slots <= 2) return run_pernode<2>(a, smem, st);
    if (slots <= 4) return run_pernode<4>(a, smem, st);
    if (slots <= kMaxSlots) return run_pernode<kMaxSlots>(a, smem, st);
    return cudaErrorInvalidValue;
}

}  // namespace rxg
