// Single long string kernels (configs (a), (e)).
//
//   k_seq      one thread walks the memoized step table (latency baseline)
//
// Further engines (thread-per-node K1, the literal §8 rounds protocol, and
// the chunk-parallel walk) live in kernels_pernode.cu / kernels_chunked.cu.
#include "launch.hpp"
#include "single.hpp"

namespace rxg {

namespace {

__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

template <typename E, bool CLS>
__device__ __forceinline__ uint32_t step(const uint8_t* sm, uint32_t cls_off, uint32_t s, uint32_t b) {
    const uint32_t col = CLS ? static_cast<uint32_t>(sm[cls_off + b]) : b;
    return *reinterpret_cast<const E*>(sm + s + col * static_cast<uint32_t>(sizeof(E)));
}

struct SeqArgs {
    const uint8_t* text;
    uint64_t len;
    const uint4* img;
    uint32_t img_words;
    uint32_t cls_off, start, dead, acc_col;
    int32_t* accept;
};

template <typename E, bool CLS>
__global__ void __launch_bounds__(256) k_seq(const __grid_constant__ SeqArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    for (uint32_t i = threadIdx.x; i < a.img_words; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = a.img[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t s = a.start;
    uint64_t pos = 0;
    const uint64_t head = (16 - (reinterpret_cast<uintptr_t>(a.text) & 15)) & 15;
    for (; pos < head && pos < a.len; ++pos) s = step<E, CLS>(sm, a.cls_off, s, a.text[pos]);
    for (; pos + 16 <= a.len && s != a.dead; pos += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + pos));
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) s = step<E, CLS>(sm, a.cls_off, s, (word_of(v, w) >> (8 * k)) & 0xFFu);
    }
    if (s != a.dead)
        for (; pos < a.len; ++pos) s = step<E, CLS>(sm, a.cls_off, s, a.text[pos]);
    *a.accept = static_cast<int32_t>(*reinterpret_cast<const E*>(sm + s + a.acc_col));
}

template <typename E, bool CLS>
cudaError_t run_seq(const DevTable& t, const SeqArgs& a, cudaStream_t st) {
    auto kern = k_seq<E, CLS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.img_bytes));
    if (e != cudaSuccess) return e;
    kern<<<1, 256, t.img_bytes, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_seq(const DevTable& t, const uint8_t* text, uint64_t len, int32_t* accept, cudaStream_t st) {
    SeqArgs a{};
    a.text = text;
    a.len = len;
    a.img = static_cast<const uint4*>(t.img);
    a.img_words = t.img_bytes / 16;
    a.cls_off = t.cls_off;
    a.start = t.start;
    a.dead = t.dead;
    a.acc_col = t.ncols * static_cast<uint32_t>(t.esize);
    a.accept = accept;
    if (t.esize == 2) return t.cls ? run_seq<uint16_t, true>(t, a, st) : run_seq<uint16_t, false>(t, a, st);
    return t.cls ? run_seq<uint32_t, true>(t, a, st) : run_seq<uint32_t, false>(t, a, st);
}

}  // namespace rxg
