// Device helpers shared by the TMA-staged kernels (kernels_lines_tma.cu,
// kernels_chunk_tma.cu): shared-memory loads by absolute address, mbarrier
// wait, 2-D tensor copies, swizzle addressing, and the memoized step on the
// two LtTable layouts.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "lines_tma.hpp"

namespace rxg {
namespace tma {

__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
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
        "TMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TMA_WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

template <uint32_t BYTES>
__device__ __forceinline__ void issue(const CUtensorMap* map, uint32_t dst, uint32_t bar, int32_t x, int32_t y) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "n"(BYTES) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// One bulk (non-tensor) copy global -> shared of `bytes` (multiple of 16,
// both addresses 16-byte aligned) completing on mbarrier `bar`; called by one
// thread after the barrier is initialised.
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}

// End of a counting kernel, called by every thread with its warp's count in
// `warp_cnt` (valid in lane 0). The CTA's warps sum through `sums` (one u32
// per warp, shared window address); thread 0 adds (1 << 40) | sum to slot[0]
// in one atomic, so the CTA ticket and the count travel together; the CTA that
// sees gridDim.x - 1 earlier tickets publishes the total and re-zeroes the
// slot (CountSlot, launch.hpp). One L2 round trip per CTA, no fences.
__device__ __forceinline__ void publish_count(unsigned long long* slot, unsigned long long* count, bool accumulate,
                                              uint32_t warp_cnt, uint32_t sums) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sums + 4 * warp), "r"(warp_cnt) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long c = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) c += lds32(sums + 4 * w);
        constexpr unsigned long long kTicket = 1ull << 40;
        const unsigned long long old = atomicAdd(slot, kTicket | c);
        if ((old >> 40) == gridDim.x - 1) {
            const unsigned long long total = (old & (kTicket - 1)) + c;
            if (accumulate) atomicAdd(count, total);
            else *count = total;
            atomicExch(slot, 0ull);
        }
    }
}

// Physical 16-byte granule of logical granule g in row r of a stage (TMA
// swizzle none / 32B / 64B / 128B by slice width).
template <int SL>
__device__ __forceinline__ uint32_t granule(uint32_t r, uint32_t g) {
    if constexpr (SL == 16) return 0;
    else if constexpr (SL == 32) return g ^ ((r >> 2) & 1u);
    else if constexpr (SL == 64) return g ^ ((r >> 1) & 3u);
    else return g ^ (r & 7u);
}

// One memoized step on byte b. Direct layout: s is an absolute row address,
// columns 4 bytes apart. Class layout: s is a row index; the class map holds
// the absolute address of each byte's column in row 0.
template <bool CLS>
__device__ __forceinline__ uint32_t step(uint32_t s, uint32_t b, uint32_t row_bytes, uint32_t cmap_addr) {
    if constexpr (CLS) return lds16(s * row_bytes + lds32(cmap_addr + b * 4u));
    else return lds16(s + b * kLtColBytes);
}

// Same step on byte k of a word: one IDP.4A extracts the byte, scales it and
// adds the base (the row for the direct layout, the class map otherwise).
template <bool CLS>
__device__ __forceinline__ uint32_t step_w(uint32_t s, uint32_t word, int k, uint32_t row_bytes, uint32_t cmap_addr) {
    if constexpr (CLS) return lds16(s * row_bytes + lds32(__dp4a(word, 4u << (8 * k), cmap_addr)));
    else return lds16(__dp4a(word, kLtColBytes << (8 * k), s));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

// 2-D view [rows][chunk] of `text` with a (slice x box_rows) box.
CUresult make_map(CUtensorMap* map, const uint8_t* text, uint64_t rows, uint32_t chunk, uint32_t slice,
                  uint32_t box_rows);

}  // namespace tma
}  // namespace rxg
