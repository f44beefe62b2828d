// Chunk-parallel walk of one long string on the TMA-staged data path
// (RXG_ENGINE_CHUNKED; the algorithm of kernels_chunked.cu, the data path of
// kernels_lines_tma.cu).
//
// The string is viewed as [rows][chunk]; lane-owned rows ("ranges") stream
// through a 3-stage shared-memory ring of 32-byte column slices (2-D TMA,
// SWIZZLE_32B). Each range first guesses its entry state by walking the
// `lookback` bytes before it from the start state (direct loads), then walks
// its own bytes from the ring, recording the state every kMidT bytes and at
// its end. Each warp checks the range boundaries inside its tile from
// registers; the last CTA to finish checks the seams between tiles, then one
// of its warps runs the in-order repair pass, re-walking only ranges whose
// guess was wrong and stopping as soon as the re-walk meets the recorded
// trajectory. One launch.
// Exact for every pattern.
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "options.hpp"
#include "chunked.hpp"
#include "tma_common.cuh"

namespace cg = cooperative_groups;

namespace rxg {

namespace tma {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

CUresult make_map(CUtensorMap* map, const uint8_t* text, uint64_t rows, uint32_t chunk, uint32_t slice,
                  uint32_t box_rows) {
    auto enc = encode_fn();
    if (!enc) return CUDA_ERROR_NOT_SUPPORTED;
    const cuuint64_t dims[2] = {chunk, rows};
    const cuuint64_t strides[1] = {chunk};
    const cuuint32_t box[2] = {slice, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = slice == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : slice == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : slice == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    // 128-byte slices: promote to 256 B so a row's next slice is already in L2
    CUtensorMapL2promotion promo = slice >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    if (const char* e = rxg::option("RXG_TMA_PROMO")) {   // tuning override
        const int v = std::atoi(e);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(text), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace tma

namespace {

// Ring shape: warps per CTA, ranges per lane, bytes per range per stage, ring depth.
template <int W, int K, int SL, int ST>
struct Shape {
    static constexpr int warps = W, chains = K, rows = 32 * K, stages = ST;
    static constexpr uint32_t slice = SL, stage_bytes = static_cast<uint32_t>(rows * SL);
};
using ShapeA = Shape<24, 2, 32, 3>;   // table layouts with a dependent load per byte (latency bound)
using ShapeP = Shape<16, 1, 128, 3>;  // packed layout: 128-byte row slices, 256 B L2 promotion
                                      // ((e) 1 GiB: 194 us vs 253 us for the row layout on ShapeA)

// Calls f(shape tag) with the ring shape of table t (RXG_CHUNK_SHAPE: A/B override).
// chunk: the caller's range width (0 = auto); a packed table with a chunk that is
// not a multiple of 128 runs on the 32-byte ring.
template <class F>
auto with_shape(const LtTable& t, uint32_t chunk, F f) {
    const char* fe = rxg::option("RXG_CHUNK_SHAPE");
    const int force = fe ? std::atoi(fe) : 0;
    if (force == 5 && chunk % 128 == 0) return f(Shape<12, 2, 128, 2>{});
    if (force == 1 || (t.packed && chunk % ShapeP::slice)) return f(ShapeA{});
    return t.packed ? f(ShapeP{}) : f(ShapeA{});
}

constexpr int kMaxSlots = 128;
constexpr uint32_t kMidT = 256;   // trajectory checkpoint period (bytes)
constexpr int kRepairRounds = 64; // parallel repair rounds before the in-order pass

struct Args {
    const uint8_t* text;
    uint64_t len;
    uint64_t rows;      // full ranges in the tensor map; range `rows` (if any) is the remainder
    uint64_t nranges;
    uint64_t tiles;
    uint32_t chunk;
    uint32_t lookback;
    const uint4* img;
    uint32_t img_words;
    uint32_t bar_addr;
    uint32_t stage_addr[kMaxSlots];
    uint32_t start, row_bytes, cmap_addr, acc_off;
    uint32_t range_x, range_k;   // range-clamped class columns (L == 2)
    uint32_t* g;
    uint32_t* e;
    uint32_t* mid;      // nranges x ceil(chunk / kMidT)
    unsigned int* ticket;          // CTAs finished (non-cooperative launch; zero when idle)
    unsigned long long* bad_inv;   // ~(first range whose entry guess is wrong); 0 = none (zero-initialised)
    unsigned long long* round_inv; // the same per repair round, two slots alternating (zero when idle)
    int32_t* accept;
    unsigned long long* repairs;
    uint32_t acc_mask;     // packed layout: accept bit of each state
    unsigned int* seam;    // cooperative launch: tiles + 1 arrival counters (zero when idle; see seam_arrive)
    uint32_t entry;        // table state the string starts in (the start state unless chained)
    uint32_t* exit_state;  // nullable: table state after the string
    uint32_t fn_states;    // packed layout: > 0 = transfer-function mode with this many states (LtTable::fn_states)
};

// Packed layout (L == 3): the table word of byte b holds next*5 at bit
// 5*state for every state, one copy per lane (lane l reads bank l only);
// the state chain is one funnel shift per byte: s' = w >> (s & 31). Bits of
// s above the low five are don't-care (shf.wrap masks the amount), canon()
// clears them where states are stored or compared.
__device__ __forceinline__ uint32_t shr_wrap(uint32_t w, uint32_t s) {
    uint32_t r;
    asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(w), "r"(s));
    return r;
}

__device__ __forceinline__ uint32_t lane_base() { return kLtSmemBase + ((threadIdx.x & 31u) << 2); }

template <int L>
__device__ __forceinline__ uint32_t canon(uint32_t s) {
    return L == 3 ? (s & 31u) : s;
}

template <int L>
__device__ __forceinline__ uint32_t stepb(const Args& a, uint32_t s, uint32_t b) {
    if constexpr (L == 3) return shr_wrap(tma::lds32(lane_base() + (b << 7)), s);
    else if constexpr (L == 2) return tma::lds16(s * a.row_bytes + kLtSmemBase + 1024 + 2u * min(b ^ a.range_x, a.range_k));
    else return tma::step<L != 0>(s, b, a.row_bytes, a.cmap_addr);
}

// Step on byte k of a 4-byte word (lb = lane_base(), hoisted by the caller).
template <int L>
__device__ __forceinline__ uint32_t stepw(const Args& a, uint32_t s, uint32_t word, int k, uint32_t lb) {
    if constexpr (L == 3) return shr_wrap(tma::lds32(__dp4a(word, 128u << (8 * k), lb)), s);
    else return stepb<L>(a, s, __byte_perm(word, 0, 0x4440 + k));
}

// Walk [lo, hi) with direct loads.
template <int L>
__device__ uint32_t walk(const Args& a, uint32_t s, uint64_t lo, uint64_t hi) {
    const uint32_t lb = lane_base();
    uint64_t p = lo;
    for (; p < hi && (p & 15); ++p) s = stepb<L>(a, s, a.text[p]);
    for (; p + 64 <= hi; p += 64) {   // four independent loads in flight, then 64 steps
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const uint4*>(a.text + p) + u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k) s = stepw<L>(a, s, tma::word_of(v[u], w), k, lb);
    }
    for (; p + 16 <= hi; p += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + p));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) s = stepw<L>(a, s, tma::word_of(v, w), k, lb);
    }
    for (; p < hi; ++p) s = stepb<L>(a, s, a.text[p]);
    return canon<L>(s);
}

// Packed layout: the transfer function of [lo, hi) — the exit state from
// every state at once (six chains on one table word per byte), as six 5-bit
// fields (field i = the encoded exit state from state 5i).
__device__ uint32_t walk_fn(const Args& a, uint64_t lo, uint64_t hi) {
    const uint32_t lb = lane_base();
    uint32_t s[6] = {0u, 5u, 10u, 15u, 20u, 25u};
    auto one = [&](uint32_t w) {
#pragma unroll
        for (int i = 0; i < 6; ++i) s[i] = shr_wrap(w, s[i]);
    };
    uint64_t p = lo;
    for (; p < hi && (p & 15); ++p) one(tma::lds32(lb + (static_cast<uint32_t>(a.text[p]) << 7)));
    // 128 bytes per round trip, software pipelined (the next 128 bytes are
    // requested before these are walked: a lone thread's dependent 16-byte
    // loads would expose the DRAM latency every 16 bytes)
    constexpr int U = 8;
    uint4 nv[U];
    if (p + 16 * U <= hi) {
#pragma unroll
        for (int u = 0; u < U; ++u) nv[u] = __ldcs(reinterpret_cast<const uint4*>(a.text + p) + u);
    }
    for (; p + 16 * U <= hi; p += 16 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nv[u];
        if (p + 32 * U <= hi) {
#pragma unroll
            for (int u = 0; u < U; ++u) nv[u] = __ldcs(reinterpret_cast<const uint4*>(a.text + p + 16 * U) + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t t[16];   // the table words depend on the input only: load all 16 first
#pragma unroll
            for (int i = 0; i < 16; ++i) t[i] = tma::lds32(__dp4a(tma::word_of(v[u], i >> 2), 128u << (8 * (i & 3)), lb));
#pragma unroll
            for (int i = 0; i < 16; ++i) one(t[i]);
        }
    }
    for (; p + 16 <= hi; p += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + p));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) one(tma::lds32(__dp4a(tma::word_of(v, w), 128u << (8 * k), lb)));
    }
    for (; p < hi; ++p) one(tma::lds32(lb + (static_cast<uint32_t>(a.text[p]) << 7)));
    uint32_t f = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) f |= (s[i] & 31u) << (5 * i);
    return f;
}

// g after f (f's ranges come first): field i = g's field at f's field i.
__device__ __forceinline__ uint32_t fn_then(uint32_t f, uint32_t g) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) r |= (shr_wrap(g, (f >> (5 * i)) & 31u) & 31u) << (5 * i);
    return r;
}
constexpr uint32_t kFnIdentity = 0u | (5u << 5) | (10u << 10) | (15u << 15) | (20u << 20) | (25u << 25);

template <int L>
__device__ uint32_t entry_guess(const Args& a, uint64_t r) {
    const uint64_t c0 = r * a.chunk;
    return r == 0 ? a.entry : walk<L>(a, a.start, c0 > a.lookback ? c0 - a.lookback : 0, c0);
}

// Entry guesses of a lane's ranges (rows row0 + 32 j + lane): with the
// default 64-byte lookback every chain's four 16-byte loads are issued
// together and the chains walk interleaved, instead of one dependent walk
// after the other.
template <int L, int CH, int U>
__device__ void entry_guesses_u(const Args& a, uint64_t row0, uint32_t lane, uint32_t (&s)[CH],
                                const bool (&valid)[CH]) {
    constexpr uint64_t LB = 16 * U;
    const uint32_t lb = lane_base();
    uint4 v[CH][U];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
        const uint64_t c0 = valid[j] ? (row0 + j * 32 + lane) * a.chunk : LB;
#pragma unroll
        for (int u = 0; u < U; ++u) v[j][u] = __ldg(reinterpret_cast<const uint4*>(a.text + c0 - LB) + u);
        s[j] = a.start;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    s[j] = stepw<L>(a, s[j], tma::word_of(v[j][u], w), k, lb);
#pragma unroll
    for (int j = 0; j < CH; ++j) s[j] = valid[j] ? canon<L>(s[j]) : a.start;
}

template <int L, int CH>
__device__ void entry_guesses(const Args& a, uint64_t row0, uint32_t lane, uint32_t (&s)[CH], const bool (&valid)[CH]) {
    const uint32_t lb = a.lookback;
    bool fast = lb == 16 || lb == 32 || lb == 64;
#pragma unroll
    for (int j = 0; j < CH; ++j) fast &= !valid[j] || (row0 + j * 32 + lane) * a.chunk >= lb;
    if (!fast) {
#pragma unroll
        for (int j = 0; j < CH; ++j) s[j] = valid[j] ? entry_guess<L>(a, row0 + j * 32 + lane) : a.start;
        return;
    }
    if (lb == 16) entry_guesses_u<L, CH, 1>(a, row0, lane, s, valid);
    else if (lb == 32) entry_guesses_u<L, CH, 2>(a, row0, lane, s, valid);
    else entry_guesses_u<L, CH, 4>(a, row0, lane, s, valid);
}

// In-order repair from the first wrong guess (one warp, the table already in
// shared memory), then the answer. Run by warp 0 of the last CTA.
template <int L>
__device__ void repair_and_answer(const Args& a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t per = (a.chunk + kMidT - 1) / kMidT;
    unsigned long long repairs = 0;
    const unsigned long long fb = ~*reinterpret_cast<volatile unsigned long long*>(a.bad_inv);
    uint32_t exact = a.nranges == 0 ? a.entry : (fb == ~0ull ? a.e[a.nranges - 1] : a.e[fb - 1]);
    for (uint64_t base = fb == ~0ull ? a.nranges : fb; base < a.nranges; base += 32) {
        uint64_t j = base;
        while (j < a.nranges && j < base + 32) {
            const uint64_t jj = j + lane;
            const bool ok = jj >= a.nranges || jj >= base + 32 || (jj == j ? a.g[jj] == exact : a.g[jj] == a.e[jj - 1]);
            const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok);
            if (!bad) {
                const uint64_t lastr = min(base + 32, a.nranges) - 1;
                exact = a.e[lastr];
                j = lastr + 1;
                break;
            }
            const uint64_t r = j + (__ffs(bad) - 1);
            const uint32_t entry = r == j ? exact : a.e[r - 1];
            uint32_t s = entry;
            if (lane == 0) {
                const uint64_t c0 = r * a.chunk, c1 = min(c0 + a.chunk, a.len);
                uint32_t* mid = a.mid + r * per;
                uint32_t k = 0;
                for (uint64_t p = c0; p < c1; p += kMidT, ++k) {
                    s = walk<L>(a, s, p, min(p + kMidT, c1));
                    if (s == mid[k]) {   // trajectories coincide from here on
                        s = a.e[r];
                        break;
                    }
                    mid[k] = s;
                }
                a.g[r] = entry;
                a.e[r] = s;
                ++repairs;
            }
            __syncwarp();
            exact = __shfl_sync(0xFFFFFFFFu, s, 0);
            j = r + 1;
        }
    }
    if (lane == 0) {
        if constexpr (L == 3) {
            *a.accept = static_cast<int32_t>((a.acc_mask >> (exact / 5u)) & 1u);
        } else {
            const uint32_t acc_addr = L != 0 ? kLtSmemBase + 1024 + exact * a.row_bytes + a.acc_off : exact + a.acc_off;
            *a.accept = static_cast<int32_t>(tma::lds16(acc_addr));
        }
        if (a.repairs) *a.repairs = repairs;
        if (a.exit_state) *a.exit_state = exact;
        // idle slot for the next launch on this stream (CountSlot, launch.hpp)
        atomicExch(a.bad_inv, 0ull);
    }
}

// Seam j (first row of a tile, or the remainder range) is checked by the
// second of its two neighbours to finish: each arrives on the seam's counter
// after publishing its g / e values, and the one that reads 1 compares
// g[j] with e[j - 1]. (Cooperative launch; the grid sync that follows makes
// the verdict visible, and the counters are zeroed again after it.)
__device__ __forceinline__ void seam_arrive(const Args& a, uint64_t t, uint64_t j) {
    __threadfence();
    if (atomicAdd(a.seam + t, 1u) != 1u) return;
    __threadfence();
    if (*reinterpret_cast<volatile const uint32_t*>(a.g + j) != *reinterpret_cast<volatile const uint32_t*>(a.e + j - 1))
        atomicMax(a.bad_inv, ~static_cast<unsigned long long>(j));
}

// Transfer-function mode (packed tables, LtTable::fn_states): every lane
// walks its ranges from all S states at once on the TMA ring (S funnel shifts
// per byte instead of one, no entry guess) and stores each range's function
// in g[range]; fn_finish composes them in range order.
template <class C, int S>
__device__ void fn_tiles(const Args& a, const CUtensorMap* map, uint32_t warp, uint32_t lane, uint32_t bar0,
                         uint32_t tbar) {
    uint32_t phase = 0;
    const uint32_t ncol = a.chunk / C::slice;
    const uint32_t* stage = a.stage_addr + warp * C::stages;
    const uint32_t lb = lane_base();
    for (uint64_t tile = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x; tile < a.tiles;
         tile += static_cast<uint64_t>(gridDim.x) * C::warps) {
        const uint64_t row0 = tile * C::rows;
        if (lane == 0) {
            const uint32_t pro = ncol < C::stages ? ncol : C::stages;
            for (uint32_t st = 0; st < pro; ++st)
                tma::issue<C::stage_bytes>(map, stage[st], bar0 + st * 8, static_cast<int32_t>(st * C::slice),
                                           static_cast<int32_t>(row0));
        }
        tma::mbar_wait(tbar, 0);
        uint32_t f[C::chains][S];
#pragma unroll
        for (int j = 0; j < C::chains; ++j)
#pragma unroll
            for (int i = 0; i < S; ++i) f[j][i] = 5u * i;
        for (uint32_t col = 0; col < ncol; ++col) {
            const uint32_t st = col % C::stages;
            tma::mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
            phase ^= 1u << st;
#pragma unroll
            for (int g = 0; g < static_cast<int>(C::slice / 16); ++g) {
                uint4 v[C::chains];
#pragma unroll
                for (int j = 0; j < C::chains; ++j) {
                    const uint32_t r = j * 32 + lane;
                    v[j] = tma::lds128(stage[st] + r * C::slice + (tma::granule<C::slice>(r, g) << 4));
                }
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < C::chains; ++j) {
                            const uint32_t t = tma::lds32(__dp4a(tma::word_of(v[j], w), 128u << (8 * k), lb));
#pragma unroll
                            for (int i = 0; i < S; ++i) f[j][i] = shr_wrap(t, f[j][i]);
                        }
            }
            __syncwarp();
            if (lane == 0 && col + C::stages < ncol) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma::issue<C::stage_bytes>(map, stage[st], bar0 + st * 8, static_cast<int32_t>((col + C::stages) * C::slice),
                                           static_cast<int32_t>(row0));
            }
        }
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            const uint64_t row = row0 + j * 32 + lane;
            if (row >= a.rows) continue;
            uint32_t fn = kFnIdentity;   // states >= S keep identity fields (never reached)
#pragma unroll
            for (int i = 0; i < S; ++i) fn = (fn & ~(31u << (5 * i))) | ((f[j][i] & 31u) << (5 * i));
            a.g[row] = fn;
        }
    }
}

template <class C, bool COOP>
__device__ void fn_mode(const Args& a, const CUtensorMap* map, uint8_t* sm, uint32_t warp, uint32_t lane, uint32_t bar0,
                        uint32_t tbar) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.nranges > a.rows) {   // the remainder range, direct loads
        tma::mbar_wait(tbar, 0);
        a.g[a.rows] = walk_fn(a, a.rows * a.chunk, a.len);
    }
    switch (a.fn_states) {
    case 1: fn_tiles<C, 1>(a, map, warp, lane, bar0, tbar); break;
    case 2: fn_tiles<C, 2>(a, map, warp, lane, bar0, tbar); break;
    case 3: fn_tiles<C, 3>(a, map, warp, lane, bar0, tbar); break;
    case 4: fn_tiles<C, 4>(a, map, warp, lane, bar0, tbar); break;
    case 5: fn_tiles<C, 5>(a, map, warp, lane, bar0, tbar); break;
    default: fn_tiles<C, 6>(a, map, warp, lane, bar0, tbar); break;
    }
    tma::mbar_wait(tbar, 0);   // no CTA leaves with its table copy in flight
    auto answer = [&](uint32_t x) {
        *a.accept = static_cast<int32_t>((a.acc_mask >> (x / 5u)) & 1u);
        if (a.repairs) *a.repairs = 0;
        if (a.exit_state) *a.exit_state = x;
    };
    if constexpr (!COOP) {
        // small inputs: the last CTA to finish composes the functions in order
        uint32_t* last = reinterpret_cast<uint32_t*>(sm + (a.bar_addr + C::warps * C::stages * 8 - kLtSmemBase));
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!*last || threadIdx.x != 0) return;
        __threadfence();
        uint32_t x = a.entry;
        for (uint64_t j = 0; j < a.nranges; ++j) x = shr_wrap(*reinterpret_cast<volatile uint32_t*>(a.g + j), x) & 31u;
        answer(x);
        *a.ticket = 0;
        return;
    } else {
        cg::grid_group grid = cg::this_grid();
        grid.sync();
        // threads own contiguous runs; warp, block, grid reductions keep the order;
        // block composites go to mid[] (g holds the range functions still being read)
        const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        const uint64_t per_t = (a.nranges + nthreads - 1) / nthreads;
        uint32_t f = kFnIdentity;
        for (uint64_t j = gtid * per_t; j < min((gtid + 1) * per_t, a.nranges); ++j) f = fn_then(f, a.g[j]);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t g = __shfl_down_sync(0xFFFFFFFFu, f, off);
            if (lane + off < 32) f = fn_then(f, g);
        }
        uint32_t* wf = reinterpret_cast<uint32_t*>(sm + (a.bar_addr + C::warps * C::stages * 8 + 16 - kLtSmemBase));
        if (lane == 0) wf[warp] = f;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t b = kFnIdentity;
            for (uint32_t w = 0; w < C::warps; ++w) b = fn_then(b, wf[w]);
            a.mid[blockIdx.x] = b;
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            uint32_t x = a.entry;
            for (uint32_t b = 0; b < gridDim.x; ++b) x = shr_wrap(a.mid[b], x) & 31u;
            answer(x);
        }
    }
}

template <class C, int L, bool COOP>
__global__ void __launch_bounds__(C::warps * 32, 1) k_chunk_tma(const __grid_constant__ Args a,
                                                           const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t sm[];
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kLtSmemBase) __trap();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * C::stages * 8;
    const uint32_t tbar = a.bar_addr + C::warps * C::stages * 8 + 8;   // after the ring barriers and the `last` flag
    if (threadIdx.x == 0) {   // the table image by one bulk copy
        tma::mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma::bulk_load(kLtSmemBase, a.img, a.img_words * 16u, tbar);
    }
    if (lane == 0) {
        for (int st = 0; st < C::stages; ++st) tma::mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the table copy is waited for where it is first used: after each warp has
    // issued its first ring stages, so the two transfers overlap
    const uint32_t per = (a.chunk + kMidT - 1) / kMidT;   // checkpoints per range (the last may be partial)
    // the remainder range (past the last full row) walks with direct loads
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.nranges > a.rows) {
        tma::mbar_wait(tbar, 0);
        const uint64_t r = a.rows, c0 = r * a.chunk;
        uint32_t s = entry_guess<L>(a, r);
        a.g[r] = s;
        uint32_t k = 0;
        for (uint64_t p = c0; p < a.len; p += kMidT, ++k) {
            s = walk<L>(a, s, p, min(p + kMidT, a.len));
            a.mid[r * per + k] = s;
        }
        a.e[r] = s;
        if (COOP && a.rows > 0) seam_arrive(a, a.tiles, a.rows);
    }
    uint32_t phase = 0;
    const uint32_t ncol = a.chunk / C::slice;
    const uint32_t* stage = a.stage_addr + warp * C::stages;
    const uint32_t lb = lane_base();
    // tiles interleave the CTAs (tile = warp * grid + cta): small inputs spread over every SM
    for (uint64_t tile = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x; tile < a.tiles;
         tile += static_cast<uint64_t>(gridDim.x) * C::warps) {
        const uint64_t row0 = tile * C::rows;
        if (lane == 0) {
            const uint32_t pro = ncol < C::stages ? ncol : C::stages;
            for (uint32_t st = 0; st < pro; ++st)
                tma::issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>(st * C::slice),
                                        static_cast<int32_t>(row0));
        }
        tma::mbar_wait(tbar, 0);
        uint32_t s[C::chains], guess[C::chains];
        bool valid[C::chains];
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            valid[j] = row0 + j * 32 + lane < a.rows;
        }
        entry_guesses<L, C::chains>(a, row0, lane, s, valid);
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            guess[j] = s[j];
            if (valid[j]) a.g[row0 + j * 32 + lane] = s[j];
        }
        for (uint32_t col = 0; col < ncol; ++col) {
            const uint32_t st = col % C::stages;
            tma::mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
            phase ^= 1u << st;
#pragma unroll
            for (int g = 0; g < static_cast<int>(C::slice / 16); ++g) {
                uint4 v[C::chains];
#pragma unroll
                for (int j = 0; j < C::chains; ++j) {
                    const uint32_t r = j * 32 + lane;
                    v[j] = tma::lds128(stage[st] + r * C::slice + (tma::granule<C::slice>(r, g) << 4));
                }
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < C::chains; ++j) s[j] = stepw<L>(a, s[j], tma::word_of(v[j], w), k, lb);
            }
            __syncwarp();
            if (lane == 0 && col + C::stages < ncol) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma::issue<C::stage_bytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>((col + C::stages) * C::slice),
                                        static_cast<int32_t>(row0));
            }
            if (((col + 1) * C::slice) % kMidT == 0 || col + 1 == ncol) {
#pragma unroll
                for (int j = 0; j < C::chains; ++j)
                    if (valid[j]) a.mid[(row0 + j * 32 + lane) * per + ((col + 1) * C::slice - 1) / kMidT] = canon<L>(s[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < C::chains; ++j) {
            s[j] = canon<L>(s[j]);
            if (valid[j]) a.e[row0 + j * 32 + lane] = s[j];
        }
        // boundaries inside the tile, from registers: row j*32+lane follows
        // j*32+lane-1 (lane - 1, or lane 31 of the previous chain)
        uint32_t bad = ~0u;
#pragma unroll
        for (int j = C::chains - 1; j >= 0; --j) {
            const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, s[j], 1);
            const uint32_t wrap = j > 0 ? __shfl_sync(0xFFFFFFFFu, s[j > 0 ? j - 1 : 0], 31) : 0u;
            const bool has_pred = lane > 0 || j > 0;
            if (valid[j] && has_pred && guess[j] != (lane > 0 ? up : wrap)) bad = j * 32 + lane;
        }
        bad = __reduce_min_sync(0xFFFFFFFFu, bad);
        if (lane == 0 && bad != ~0u) atomicMax(a.bad_inv, ~(row0 + bad));
        if constexpr (COOP) {   // the seams with the neighbouring tiles (this warp's g / e are written)
            __syncwarp();
            if (lane == 0) {
                if (tile > 0) seam_arrive(a, tile, row0);
                if (tile + 1 < a.tiles) seam_arrive(a, tile + 1, row0 + C::rows);
                else if (a.nranges > a.rows) seam_arrive(a, a.tiles, a.rows);
            }
        }
    }
    tma::mbar_wait(tbar, 0);   // warps without a tile (the repair below reads the table)
    if constexpr (!COOP) {
        // small inputs: the last CTA to finish checks the seams between tiles
        // and one of its warps repairs in order (no grid-wide sync)
        uint32_t* last = reinterpret_cast<uint32_t*>(sm + (a.bar_addr + C::warps * C::stages * 8 - kLtSmemBase));
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            *last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (!*last) return;
        __threadfence();
        unsigned long long bad = ~0ull;
        for (uint64_t t = 1 + threadIdx.x; t <= a.tiles; t += blockDim.x) {
            const uint64_t j = t < a.tiles ? t * C::rows : a.rows;
            if (j >= a.nranges || (t == a.tiles && a.nranges == a.rows)) continue;
            if (a.g[j] != a.e[j - 1]) {
                bad = j;
                break;
            }
        }
        if (bad != ~0ull) atomicMax(a.bad_inv, ~bad);
        __syncthreads();
        if (threadIdx.x < 32) {
            __threadfence();
            repair_and_answer<L>(a);
            if (threadIdx.x == 0) *a.ticket = 0;
        }
        return;
    }
    // Large inputs, whole grid (cooperative launch): the seams between tiles,
    // then parallel repair rounds, then, if a chain of wrong guesses is still
    // unresolved, the in-order repair by one warp.
    cg::grid_group grid = cg::this_grid();
    grid.sync();
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (uint64_t t = gtid; t <= a.tiles; t += nthreads) a.seam[t] = 0;   // idle again (seams checked in-stream)
    unsigned long long fb = ~*reinterpret_cast<volatile unsigned long long*>(a.bad_inv);
    if constexpr (L == 3) {
        // Packed tables (<= 6 states): no repair rounds. Every range from the
        // first wrong guess on computes its transfer function (its exit from
        // every state), the functions are composed in range order (threads own
        // contiguous runs; warp, block and grid reductions keep the order), and
        // the composite applied to the exact exit before fb is the answer:
        // exact for non-synchronising automata ((aaa)*) in one extra pass.
        if (fb != ~0ull) {
            const uint64_t nfn = a.nranges - fb;
            const uint64_t per_t = (nfn + nthreads - 1) / nthreads;
            uint32_t f = kFnIdentity;
            for (uint64_t j = fb + gtid * per_t; j < fb + min((gtid + 1) * per_t, nfn); ++j)
                f = fn_then(f, walk_fn(a, j * a.chunk, min((j + 1) * a.chunk, a.len)));
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {   // lanes in order: lane i then lanes above it
                const uint32_t g = __shfl_down_sync(0xFFFFFFFFu, f, off);
                if (lane + off < 32) f = fn_then(f, g);
            }
            uint32_t* wf = reinterpret_cast<uint32_t*>(sm + (a.bar_addr + C::warps * C::stages * 8 + 16 - kLtSmemBase));
            if (lane == 0) wf[warp] = f;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t b = kFnIdentity;
                for (uint32_t w = 0; w < C::warps; ++w) b = fn_then(b, wf[w]);
                a.g[blockIdx.x] = b;   // (the guesses are not needed any more)
            }
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                uint32_t x = fb == 0 ? a.entry : a.e[fb - 1];
                for (uint32_t b = 0; b < gridDim.x; ++b) x = shr_wrap(a.g[b], x) & 31u;
                *a.accept = static_cast<int32_t>((a.acc_mask >> (x / 5u)) & 1u);
                if (a.repairs) *a.repairs = nfn;
                if (a.exit_state) *a.exit_state = x;
                atomicExch(a.bad_inv, 0ull);
            }
            return;
        }
        if (blockIdx.x == 0 && threadIdx.x < 32) repair_and_answer<L>(a);   // every guess right: the answer
        return;
    }
    // Round: every range j >= fb whose guess differs from its predecessor's
    // exit re-walks from that exit (stopping where it meets its recorded
    // trajectory). Ranges below the first mismatch are exact and final, so
    // each round moves the frontier at least one range; chains of sticky
    // states (a keyword seen once keeps the automaton accepting) resolve in
    // as many rounds as the longest run of ranges without the keyword.
    for (int round = 0; round < kRepairRounds && fb != ~0ull; ++round) {
        const uint32_t per = (a.chunk + kMidT - 1) / kMidT;
        for (uint64_t j = fb + gtid; j < a.nranges; j += nthreads) {
            if (j == 0) continue;
            const uint32_t entry = *reinterpret_cast<volatile uint32_t*>(a.e + j - 1);
            if (a.g[j] == entry) continue;
            const uint64_t c0 = j * a.chunk, c1 = min(c0 + a.chunk, a.len);
            uint32_t st = entry;
            uint32_t* mid = a.mid + j * per;
            uint32_t k = 0;
            for (uint64_t p = c0; p < c1; p += kMidT, ++k) {
                st = walk<L>(a, st, p, min(p + kMidT, c1));
                if (st == mid[k]) {   // trajectories coincide from here on
                    st = a.e[j];
                    break;
                }
                mid[k] = st;
            }
            a.g[j] = entry;
            *reinterpret_cast<volatile uint32_t*>(a.e + j) = st;
        }
        unsigned long long* slot = a.round_inv + (round & 1);
        if (gtid == 0) *slot = 0;
        grid.sync();
        {
            unsigned long long bad = ~0ull;
            for (uint64_t j = fb + gtid; j < a.nranges; j += nthreads)
                if (j > 0 && a.g[j] != a.e[j - 1]) {
                    bad = j;
                    break;
                }
            if (bad != ~0ull) atomicMax(slot, ~bad);
        }
        grid.sync();
        fb = ~*reinterpret_cast<volatile unsigned long long*>(slot);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {   // what is left in order, and the answer
        if (threadIdx.x == 0) *a.bad_inv = ~fb;
        __syncwarp();
        repair_and_answer<L>(a);
        if (threadIdx.x == 0) {
            a.round_inv[0] = 0;
            a.round_inv[1] = 0;
        }
    }
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Transfer-function mode as its own kernel (packed tables with
// LtTable::fn_states): the guessing kernel above keeps its registers.
template <class C, bool COOP>
__global__ void __launch_bounds__(C::warps * 32, 1) k_chunk_fn(const __grid_constant__ Args a,
                                                          const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t sm[];
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kLtSmemBase) __trap();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * C::stages * 8;
    const uint32_t tbar = a.bar_addr + C::warps * C::stages * 8 + 8;
    if (threadIdx.x == 0) {
        tma::mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma::bulk_load(kLtSmemBase, a.img, a.img_words * 16u, tbar);
    }
    if (lane == 0) {
        for (int st = 0; st < C::stages; ++st) tma::mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    fn_mode<C, COOP>(a, &map, sm, warp, lane, bar0, tbar);
}

template <class C, int L>
cudaError_t run(const LtTable& t, Args& a, int device, cudaStream_t st) {
    // stage ring after the table image, mbarriers after the ring
    uint32_t p = align_up(t.smem_table_end, 1024);
    for (int k = 0; k < C::warps * C::stages; ++k, p += C::stage_bytes) a.stage_addr[k] = p;
    a.bar_addr = align_up(p, 8);
    const uint32_t smem = a.bar_addr + C::warps * C::stages * 8 + 16 + 4 * C::warps - kLtSmemBase;   // ring barriers, `last`, table barrier, per-warp functions
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (a.rows > 0 && tma::make_map(&map, a.text, a.rows, a.chunk, C::slice, C::rows) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    // grid-wide repair rounds pay off above a few MB; below, the launch and two
    // grid syncs cost more than the in-order repair can
    const bool coop = a.len >= (4ull << 20) && a.seam;
    auto* kern = coop ? k_chunk_tma<C, L, true> : k_chunk_tma<C, L, false>;
    if constexpr (L == 3) {
        if (a.fn_states) kern = coop ? k_chunk_fn<C, true> : k_chunk_fn<C, false>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t want = a.tiles;   // at most one tile per CTA needed to reach every SM
    const int grid = static_cast<int>(want == 0 ? 1 : (want < static_cast<uint64_t>(sms) ? want : sms));
    // cooperative (>= 4 MiB): every CTA is resident (one per SM), the repair rounds sync the grid
    // (programmatic dependent launch measured no gain here: a cooperative grid
    // holding every SM's shared memory cannot overlap the previous one)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = coop ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a, map);
}

}  // namespace

template <class C>
uint32_t auto_chunk(uint64_t len, int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t ranges = static_cast<uint64_t>(sms) * C::warps * C::rows;
    uint64_t c = (len + ranges - 1) / ranges;
    c = (c + C::slice - 1) / C::slice * C::slice;   // slice multiple: keeps the grid at one CTA per SM
    if (c < 2 * C::slice) c = 2 * C::slice;         // small inputs: short ranges (the lookback is 64 B)
    return static_cast<uint32_t>(c);
}

uint32_t chunked_tma_auto_chunk(const LtTable& t, uint64_t len, int device) {
    return with_shape(t, 0, [&](auto c) { return auto_chunk<decltype(c)>(len, device); });
}

size_t chunked_tma_scratch_bytes(uint64_t len, uint32_t chunk) {
    const uint64_t n = (len + chunk - 1) / chunk;
    return 16 + (2 * n + n * ((chunk + kMidT - 1) / kMidT)) * sizeof(uint32_t) + 64;
}

cudaError_t launch_chunked_tma(const LtTable& t, const void* d_img, const uint8_t* text, uint64_t len, uint32_t chunk,
                               uint32_t lookback, void* scratch, int32_t* accept, unsigned long long* repairs,
                               CountSlot cs, int device, cudaStream_t st, uint32_t entry, uint32_t* exit_state) {
    const uint32_t slice = with_shape(t, chunk, [](auto c) { return decltype(c)::slice; });
    if (chunk == 0 || chunk % slice) return cudaErrorInvalidValue;
    Args a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    a.lookback = lookback;
    a.rows = len / chunk;
    a.nranges = (len + chunk - 1) / chunk;
    a.img = static_cast<const uint4*>(d_img);
    a.img_words = t.lo_bytes / 16;
    a.start = t.start;
    a.entry = entry == kStartState ? t.start : entry;
    a.exit_state = exit_state;
    a.row_bytes = t.row_bytes;
    a.cmap_addr = t.cmap_addr;
    a.acc_off = t.acc_off;
    a.bad_inv = cs.p + 1;
    a.seam = cs.seam;
    a.round_inv = cs.p + 2;
    a.ticket = reinterpret_cast<unsigned int*>(cs.p + 3) + 1;   // the high half of the second round slot
                                                               // (rounds run only cooperatively)
    uint32_t* sc = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + 16);
    a.g = sc;
    a.e = sc + a.nranges;
    a.mid = sc + 2 * a.nranges;
    a.accept = accept;
    a.repairs = repairs;
    // (len == 0: one CTA, no ranges; the repair pass answers from the start state)
    a.range_x = t.range_x;
    a.range_k = t.range_k;
    a.acc_mask = t.acc_mask;
    a.fn_states = t.packed ? t.fn_states : 0u;
    if (t.packed)
        return with_shape(t, chunk, [&](auto c) {
            using C = decltype(c);
            a.tiles = (a.rows + C::rows - 1) / C::rows;
            return run<C, 3>(t, a, device, st);
        });
    return with_shape(t, chunk, [&](auto c) {
        using C = decltype(c);
        a.tiles = (a.rows + C::rows - 1) / C::rows;
        return t.cls ? (t.range_k ? run<C, 2>(t, a, device, st) : run<C, 1>(t, a, device, st)) : run<C, 0>(t, a, device, st);
    });
}

}  // namespace rxg
