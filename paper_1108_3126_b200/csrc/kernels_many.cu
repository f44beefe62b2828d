// Multi-heap batch: every pattern of a set against every string of a set —
// the shape of the reference's crosscheck sweep (crosscheck.cpp:111-185,
// acceptance criterion 3: all regexes <= 8 nodes x all strings <= 6). One
// CTA per pattern loads that pattern's memoized step table (class map,
// accept flags, class-indexed rows of u16 state indices) into shared memory;
// its threads walk all strings (one string per thread, strings re-read from
// L1/L2 by every CTA) and write one result byte per (pattern, string).
#include <cstdint>

#include "many.hpp"

namespace rxg {

namespace {

struct ManyArgs {
    const uint8_t* tables;          // packed per-pattern images
    const uint64_t* table_off;      // n_patterns + 1 byte offsets (16-aligned)
    const uint32_t* meta;           // per pattern: n_states, n_cols, start, accept_off, rows_off
    const uint8_t* text;
    const uint64_t* str_off;        // n_strings + 1 (string i = [off[i], off[i+1] - sep))
    uint32_t sep;                   // 1 for delimited strings, 0 for fixed stride
    uint64_t n_patterns, n_strings;
    uint8_t* results;               // n_patterns x n_strings
};

__global__ void __launch_bounds__(256) k_many(const __grid_constant__ ManyArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    for (uint64_t p = blockIdx.x; p < a.n_patterns; p += gridDim.x) {
        const uint64_t lo = a.table_off[p], hi = a.table_off[p + 1];
        const uint4* src = reinterpret_cast<const uint4*>(a.tables + lo);
        for (uint32_t i = threadIdx.x; i < (hi - lo) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = src[i];
        __syncthreads();
        const uint32_t* m = a.meta + p * 5;
        const uint32_t ncols = m[1], start = m[2];
        const uint8_t* cmap = sm;                 // 256 byte classes
        const uint8_t* acc = sm + m[3];           // accept flag per state
        const uint16_t* rows = reinterpret_cast<const uint16_t*>(sm + m[4]);
        for (uint64_t s = threadIdx.x; s < a.n_strings; s += blockDim.x) {
            const uint64_t b = a.str_off[s], e = a.str_off[s + 1] - a.sep;
            uint32_t st = start;
            for (uint64_t i = b; i < e; ++i) st = rows[st * ncols + cmap[__ldg(a.text + i)]];
            a.results[p * a.n_strings + s] = acc[st];
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_many(const ManyDev& d, uint64_t n_patterns, uint64_t n_strings, uint32_t sep, uint8_t* results,
                        uint32_t max_table_bytes, int device, cudaStream_t st) {
    if (n_patterns == 0 || n_strings == 0) return cudaSuccess;
    ManyArgs a{};
    a.tables = d.tables;
    a.table_off = d.table_off;
    a.meta = d.meta;
    a.text = d.text;
    a.str_off = d.str_off;
    a.sep = sep;
    a.n_patterns = n_patterns;
    a.n_strings = n_strings;
    a.results = results;
    cudaError_t e = cudaFuncSetAttribute(k_many, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(max_table_bytes));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_many, 256, max_table_bytes);
    if (per_sm < 1) per_sm = 1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t cap = static_cast<uint64_t>(per_sm) * static_cast<uint64_t>(sms);
    const int grid = static_cast<int>(n_patterns < cap ? n_patterns : cap);
    k_many<<<grid, 256, max_table_bytes, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rxg
