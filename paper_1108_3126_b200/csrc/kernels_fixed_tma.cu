// K2 for fixed-stride batches on the TMA data path (config (b): 1M strings
// of 32 bytes). Each lane walks whole strings (three per lane: 96 strings per
// warp tile); the tiles of a warp stream through a 2-stage shared-memory ring
// that runs across tiles, so the next tile is in flight while the current one
// is walked (the LDG variant, k_fixed_abs, waits for each pass's loads).
//   stride 32 ("packed"): the buffer is viewed as [n/4][128 B], a tile is 24
//     such rows (one 128-byte TMA request per row, SWIZZLE_128B so the
//     16-byte reads of 8 lanes hit 8 distinct bank groups);
//   stride 32k: the buffer is [n][stride], a tile is 96 rows, streamed in
//     32-byte column slices (SWIZZLE_32B).
// Table: the raw-byte u16 image with absolute entries (step = LDS.U16
// [s + 2b], one IDP.4A forms the address).
#include <cstring>

#include "launch.hpp"
#include "tma_common.cuh"

namespace rxg {

namespace {

constexpr int kFW = 24, kFC = 3, kFRows = 32 * kFC, kFSt = 2;   // (tools/ab_fixed.py: 16x3x3 15.4 us, 24x3x2 14.4, 16x4x2 15.3, 32x2x2 15.4, 16x2x4 16.4, 24x2x3 15.4 on (b), L2 flushed)
constexpr uint32_t kFSlice = 32, kFStageBytes = kFRows * kFSlice;
constexpr uint32_t kFBase = 0x400;   // the table image's absolute entries assume this window

struct FArgs {
    uint64_t n;          // strings (covered by the tensor map)
    uint64_t tiles;      // ceil(n / 96)
    uint32_t ncol;       // stride / 32 (1 when packed)
    const uint4* img;
    uint32_t img_words;
    uint32_t start, acc_col;
    uint32_t bar_addr;
    uint32_t stage_addr[kFW * kFSt];
    unsigned long long* count;
    unsigned long long* slot;   // CountSlot (launch.hpp)
    int accumulate;
    uint8_t* results;
};

template <bool RES, bool PACK>
__global__ void __launch_bounds__(kFW * 32, 1) k_fixed_tma(const __grid_constant__ FArgs a,
                                                         const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t sm[];
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kFBase) __trap();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = a.bar_addr + warp * kFSt * 8;
    // this warp's tiles: first, first + step, ...; items = (tile, column slice) in order
    const uint64_t first = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x;
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * kFW;
    const uint64_t my_tiles = first < a.tiles ? (a.tiles - first + step - 1) / step : 0;
    const uint64_t items = my_tiles * a.ncol;
    const uint32_t* stage = a.stage_addr + warp * kFSt;
    auto issue = [&](uint64_t q) {
        const uint64_t tile = first + (q / a.ncol) * step;
        const uint32_t col = static_cast<uint32_t>(q % a.ncol);
        const uint32_t st = static_cast<uint32_t>(q % kFSt);
        if (PACK)
            tma::issue<kFStageBytes>(&map, stage[st], bar0 + st * 8, 0, static_cast<int32_t>(tile * (kFRows / 4)));
        else
            tma::issue<kFStageBytes>(&map, stage[st], bar0 + st * 8, static_cast<int32_t>(col * kFSlice),
                                     static_cast<int32_t>(tile * kFRows));
    };
    // the table image (one bulk copy) and the ring's first tiles are all in flight at once
    const uint32_t tbar = a.bar_addr + kFW * kFSt * 8;
    if (threadIdx.x == 0) {
        tma::mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma::bulk_load(kFBase, a.img, a.img_words * 16u, tbar);
    }
    if (lane == 0) {
        for (int st = 0; st < kFSt; ++st) tma::mbar_init(bar0 + st * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint64_t q = 0; q < items && q < kFSt; ++q) issue(q);
    }
    __syncthreads();   // barrier initialisation visible to every thread
    tma::mbar_wait(tbar, 0);

    uint32_t cnt = 0, phase = 0;
    uint32_t s[kFC];
    for (uint64_t q = 0; q < items; ++q) {
        const uint32_t st = static_cast<uint32_t>(q % kFSt);
        const uint32_t col = static_cast<uint32_t>(q % a.ncol);
        if (col == 0) {
#pragma unroll
            for (int j = 0; j < kFC; ++j) s[j] = a.start;
        }
        tma::mbar_wait(bar0 + st * 8, (phase >> st) & 1u);
        phase ^= 1u << st;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            uint4 v[kFC];
#pragma unroll
            for (int j = 0; j < kFC; ++j) {
                const uint32_t r = j * 32 + lane;
                if (PACK) {   // string r = 128-byte row r/4, granule 2*(r%4)+g, 128-byte swizzle
                    const uint32_t row = r >> 2;
                    v[j] = tma::lds128(stage[st] + row * 128 + (tma::granule<128>(row, ((r & 3) << 1) | g) << 4));
                } else {
                    v[j] = tma::lds128(stage[st] + r * kFSlice + (tma::granule<kFSlice>(r, g) << 4));
                }
            }
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int j = 0; j < kFC; ++j) s[j] = tma::lds16(__dp4a(tma::word_of(v[j], w), 2u << (8 * k), s[j]));
        }
        __syncwarp();
        if (lane == 0 && q + kFSt < items) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(q + kFSt);
        }
        if (col + 1 == a.ncol) {   // the tile's strings are complete
            const uint64_t row0 = (first + (q / a.ncol) * step) * kFRows;
#pragma unroll
            for (int j = 0; j < kFC; ++j) {
                const uint64_t row = row0 + j * 32 + lane;
                if (row < a.n) {
                    const uint32_t ok = tma::lds16(s[j] + a.acc_col);
                    cnt += ok;
                    if (RES) a.results[row] = static_cast<uint8_t>(ok);
                }
            }
        }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    tma::publish_count(a.slot, a.count, a.accumulate != 0, cnt, a.bar_addr + kFW * kFSt * 8 + 8);
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

template <bool RES, bool PACK>
cudaError_t run(FArgs& a, const uint8_t* text, uint32_t stride, uint32_t img_bytes, int device, cudaStream_t st) {
    uint32_t p = align_up(kFBase + img_bytes, 1024);
    for (int k = 0; k < kFW * kFSt; ++k, p += kFStageBytes) a.stage_addr[k] = p;
    a.bar_addr = align_up(p, 8);
    const uint32_t smem = a.bar_addr + kFW * kFSt * 8 + 8 + 4 * kFW - kFBase;   // ring barriers, table barrier, warp sums
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (PACK) {
        auto enc = tma::encode_fn();
        if (!enc) return cudaErrorNotSupported;
        const cuuint64_t dims[2] = {128, a.n / 4};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {128, kFRows / 4};
        const cuuint32_t estr[2] = {1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(text), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    } else if (tma::make_map(&map, text, a.n, stride, kFSlice, kFRows) != CUDA_SUCCESS) {
        return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(k_fixed_tma<RES, PACK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const uint64_t sms = static_cast<uint64_t>(device_sm_count(device));
    const int grid = static_cast<int>(a.tiles < sms ? a.tiles : sms);
    k_fixed_tma<RES, PACK><<<grid, kFW * 32, smem, st>>>(a, map);
    return cudaGetLastError();
}

}  // namespace

bool fixed_tma_fits(uint32_t img_bytes, uint32_t stride, int smem_limit) {
    const uint32_t need = align_up(kFBase + img_bytes, 1024) + kFW * kFSt * kFStageBytes + kFW * kFSt * 8 + 8 + 4 * kFW - kFBase;
    return stride % kFSlice == 0 && static_cast<int>(need) <= smem_limit;
}

cudaError_t launch_fixed_tma(const DevTable& t_abs, const uint8_t* text, uint64_t n, uint32_t stride,
                             unsigned long long* count, uint8_t* results, CountSlot cs, int device, cudaStream_t st,
                             uint64_t* n_done) {
    if (n_done) *n_done = 0;
    if (t_abs.cls || t_abs.esize != 2 || stride % kFSlice) return cudaErrorInvalidValue;
    const bool pack = stride == 32;
    FArgs a{};
    a.n = pack ? n / 4 * 4 : n;   // packed: the last n % 4 strings are left to the caller
    if (a.n == 0) return cs.accumulate ? cudaSuccess : cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    a.tiles = (a.n + kFRows - 1) / kFRows;
    a.ncol = pack ? 1 : stride / kFSlice;
    a.img = static_cast<const uint4*>(t_abs.img);
    a.img_words = t_abs.img_bytes / 16;
    a.start = t_abs.start + kFBase;
    a.acc_col = t_abs.ncols * 2u;
    a.count = count;
    a.slot = cs.p;
    a.accumulate = cs.accumulate ? 1 : 0;
    a.results = results;
    if (n_done) *n_done = a.n;
    if (pack)
        return results ? run<true, true>(a, text, stride, t_abs.img_bytes, device, st)
                       : run<false, true>(a, text, stride, t_abs.img_bytes, device, st);
    return results ? run<true, false>(a, text, stride, t_abs.img_bytes, device, st)
                   : run<false, false>(a, text, stride, t_abs.img_bytes, device, st);
}

}  // namespace rxg
