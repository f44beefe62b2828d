// K2 (lines), TMA-staged variant for memoized step tables that fit the
// raw-byte u16 layout (DFA <= ~56 states, e.g. config (c)).
//
// Data path per warp: the warp owns 64 consecutive equal byte ranges
// ("rows" of a 2-D view [rows][chunk] of the input) — two per lane. A TMA
// tensor map streams 16-byte column slices of those 64 rows into a 4-stage
// shared-memory ring (rows 16 B apart, so the per-lane 16-byte reads of 8
// consecutive rows fill one 128-byte wavefront). One elected lane arms the
// stage mbarrier and issues the copy; all lanes wait on its phase.
//
// Step per input byte (the memoized lockstep macro step, see tables.hpp):
//     b = PRMT(word, k)            extract byte
//     s = LDS.U16 [s + 4b]         s and the entries are absolute shared addresses
//     n += hi32(s * 2^17)          START_A (the accepted-line-end row) is the only
//                                  row at >= 0x8000 the main loop can enter
// Columns are 4 B apart, so the bytes of one row map to banks (row + b) mod 32
// (' ' and 'a' no longer collide); rows are 1060 B apart (265 words = 9 mod
// 32), so lanes in different states reading the same byte land in
// different banks.
//
// Line ownership (every line matched exactly once) is the rule of
// kernels_batch.cu: a range owns the lines starting in it, enters in SKIP
// unless the previous byte is the delimiter, and finishes its last line
// through the tail copy of the table with direct global loads.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "launch.hpp"
#include "lines_tma.hpp"

namespace rxg {

namespace {

struct Args {
    const uint8_t* text;
    uint64_t len;
    uint64_t rows;         // full ranges covered by the tensor map
    uint64_t tiles;        // ceil(rows / kRowsPerWarp)
    uint32_t chunk;        // range width (multiple of kSlice)
    uint32_t rem_piece;    // remainder [rows*chunk, len) split in pieces (direct loads)
    uint32_t rem_pieces;
    const uint4* img_lo;
    uint32_t lo_addr, lo_words;
    const uint4* img_hi;
    uint32_t hi_addr, hi_words;
    uint32_t bar_addr;
    uint32_t stage_addr[kLtWarps * kLtStages];
    uint32_t start, skip, void_row, tail_delta, term_acc;
    uint32_t delim;
    unsigned long long* count;
};

__device__ __forceinline__ uint32_t tab(uint32_t addr) {
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t step(uint32_t s, uint32_t word, int k) {
    return tab(s + __byte_perm(word, 0, 0x4440 + k) * kLtColBytes);
}

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LTMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LTMA_WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_issue(const CUtensorMap* map, uint32_t dst, uint32_t bar, int32_t x, int32_t y) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "n"(kLtStageBytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// Finish the line straddling a range end with direct loads (tail copy rows).
__device__ uint32_t finish_line(const Args& a, uint32_t s, uint64_t pos) {
    while (pos < a.len) {
        if (pos + 16 <= a.len) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k) s = step(s, word_of(v, w), k);
            pos += 16;
        } else {
            for (; pos < a.len; ++pos) s = tab(s + static_cast<uint32_t>(a.text[pos]) * kLtColBytes);
        }
        if (s >= a.term_acc) return s;
    }
    return tab(s + a.delim * kLtColBytes);
}

// A range processed entirely with direct loads (the remainder pieces).
__device__ void range_direct(const Args& a, uint64_t c0, uint64_t c1, uint32_t& cnt) {
    uint32_t s = (c0 == 0 || a.text[c0 - 1] == a.delim) ? a.start : a.skip;
    uint32_t last = 0;
    uint64_t pos = c0;
    for (; pos + 16 <= c1; pos += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                s = step(s, word_of(v, w), k);
                cnt += __umulhi(s, 1u << 17);
            }
        last = v.w >> 24;
    }
    for (; pos < c1; ++pos) {
        last = a.text[pos];
        s = tab(s + last * kLtColBytes);
        cnt += __umulhi(s, 1u << 17);
    }
    if (s != a.skip && last != a.delim) cnt += finish_line(a, s + a.tail_delta, c1) == a.term_acc;
}

__global__ void __launch_bounds__(kLtWarps * 32) k_lines_tma(const __grid_constant__ Args a,
                                                             const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(128) uint8_t sm[];
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    if (base != kLtSmemBase) __trap();   // the table's absolute addresses assume this window
    {
        uint4* lo = reinterpret_cast<uint4*>(sm + (a.lo_addr - base));
        for (uint32_t i = threadIdx.x; i < a.lo_words; i += blockDim.x) lo[i] = a.img_lo[i];
        uint4* hi = reinterpret_cast<uint4*>(sm + (a.hi_addr - base));
        for (uint32_t i = threadIdx.x; i < a.hi_words; i += blockDim.x) hi[i] = a.img_hi[i];
    }
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * kLtStages * 8;
    if (lane == 0) {
        for (int st = 0; st < kLtStages; ++st) mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    __syncthreads();

    uint32_t cnt = 0;
    if (blockIdx.x == 0 && warp == 0) {
        const uint64_t r0 = a.rows * a.chunk;
        for (uint32_t p = lane; p < a.rem_pieces; p += 32) {
            const uint64_t c0 = r0 + static_cast<uint64_t>(p) * a.rem_piece;
            range_direct(a, c0, min(c0 + a.rem_piece, a.len), cnt);
        }
    }

    uint32_t phase = 0;   // bit st = parity of stage st's next completion
    const uint32_t ncol = a.chunk / kLtSlice;
    const uint32_t* stage = a.stage_addr + warp * kLtStages;
    for (uint64_t tile = static_cast<uint64_t>(blockIdx.x) * kLtWarps + warp; tile < a.tiles;
         tile += static_cast<uint64_t>(gridDim.x) * kLtWarps) {
        const uint64_t row0 = tile * kLtRowsPerWarp;
        if (lane == 0) {
            const uint32_t pro = ncol < kLtStages ? ncol : kLtStages;
            for (uint32_t st = 0; st < pro; ++st)
                tma_issue(&map, stage[st], bar0 + st * 8, static_cast<int32_t>(st * kLtSlice), static_cast<int32_t>(row0));
        }
        uint32_t s[kLtChains];
        bool valid[kLtChains];
#pragma unroll
        for (int j = 0; j < kLtChains; ++j) {
            const uint64_t row = row0 + j * 32 + lane;
            valid[j] = row < a.rows;
            s[j] = a.void_row;
            if (valid[j]) {
                const uint64_t c0 = row * a.chunk;
                s[j] = (c0 == 0 || a.text[c0 - 1] == a.delim) ? a.start : a.skip;
            }
        }
        uint32_t last[kLtChains] = {};
        for (uint32_t col = 0; col < ncol; ++col) {
            const uint32_t st = col % kLtStages;
            mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
            phase ^= 1u << st;
#pragma unroll
            for (int g = 0; g < kLtSlice / 16; ++g) {
                uint4 v[kLtChains];
#pragma unroll
                for (int j = 0; j < kLtChains; ++j) {
                    const uint32_t r = j * 32 + lane;
                    v[j] = lds128(stage[st] + r * kLtSlice + g * 16u);
                }
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int j = 0; j < kLtChains; ++j) {
                            s[j] = step(s[j], word_of(v[j], w), k);
                            cnt += __umulhi(s[j], 1u << 17);
                        }
#pragma unroll
                for (int j = 0; j < kLtChains; ++j) last[j] = v[j].w >> 24;
            }
            __syncwarp();
            if (lane == 0 && col + kLtStages < ncol) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_issue(&map, stage[st], bar0 + st * 8, static_cast<int32_t>((col + kLtStages) * kLtSlice),
                          static_cast<int32_t>(row0));
            }
        }
#pragma unroll
        for (int j = 0; j < kLtChains; ++j) {
            if (valid[j] && s[j] != a.skip && last[j] != a.delim) {
                const uint64_t row = row0 + j * 32 + lane;
                cnt += finish_line(a, s[j] + a.tail_delta, (row + 1) * a.chunk) == a.term_acc;
            }
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (lane == 0 && cnt) atomicAdd(a.count, static_cast<unsigned long long>(cnt));
}

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

}  // namespace

cudaError_t launch_lines_tma(const LtTable& t, const uint8_t* text, uint64_t len, uint8_t delim, uint32_t chunk,
                             unsigned long long* count, cudaStream_t st) {
    if (len == 0) return cudaSuccess;
    if (chunk % kLtSlice) return cudaErrorInvalidValue;
    Args a{};
    a.text = text;
    a.len = len;
    a.chunk = chunk;
    a.rows = len / chunk;
    a.tiles = (a.rows + kLtRowsPerWarp - 1) / kLtRowsPerWarp;
    const uint64_t rem = len - a.rows * chunk;
    a.rem_piece = static_cast<uint32_t>(((rem + 31) / 32 + 15) & ~uint64_t(15));
    if (a.rem_piece < 16) a.rem_piece = 16;
    a.rem_pieces = rem ? static_cast<uint32_t>((rem + a.rem_piece - 1) / a.rem_piece) : 0;
    a.img_lo = static_cast<const uint4*>(t.d_lo);
    a.lo_addr = t.lo_addr;
    a.lo_words = t.lo_bytes / 16;
    a.img_hi = static_cast<const uint4*>(t.d_hi);
    a.hi_addr = t.hi_addr;
    a.hi_words = t.hi_bytes / 16;
    a.bar_addr = t.bar_addr;
    for (int i = 0; i < kLtWarps * kLtStages; ++i) a.stage_addr[i] = t.stage_addr[i];
    a.start = t.start;
    a.skip = t.skip;
    a.void_row = t.void_row;
    a.tail_delta = t.tail_delta;
    a.term_acc = t.term_acc;
    a.delim = delim;
    a.count = count;

    CUtensorMap map;
    if (a.rows > 0) {
        auto enc = encode_fn();
        if (!enc) return cudaErrorNotSupported;
        const cuuint64_t dims[2] = {chunk, a.rows};
        const cuuint64_t strides[1] = {chunk};
        const cuuint32_t box[2] = {kLtSlice, kLtRowsPerWarp};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(text), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    } else {
        std::memset(&map, 0, sizeof(map));
    }
    const uint32_t smem = t.smem_bytes;
    cudaError_t e = cudaFuncSetAttribute(k_lines_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lines_tma, kLtWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = static_cast<uint64_t>(per_sm) * device_sm_count(dev);
    const uint64_t want = (a.tiles + kLtWarps - 1) / kLtWarps;
    const int grid = static_cast<int>(want == 0 ? 1 : (want < cap ? want : cap));
    k_lines_tma<<<grid, kLtWarps * 32, smem, st>>>(a, map);
    return cudaGetLastError();
}

uint32_t lines_tma_auto_chunk(const LtTable& t, uint64_t len) {
    int per_sm = 0;
    cudaFuncSetAttribute(k_lines_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem_bytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lines_tma, kLtWarps * 32, t.smem_bytes);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t rows = static_cast<uint64_t>(per_sm) * device_sm_count(dev) * kLtWarps * kLtRowsPerWarp;
    uint64_t c = (len + rows - 1) / rows;
    c = (c + kLtSlice - 1) / kLtSlice * kLtSlice;
    if (c < 4 * kLtSlice) c = 4 * kLtSlice;
    if (c > (1u << 20)) c = 1u << 20;
    return static_cast<uint32_t>(c);
}

}  // namespace rxg
