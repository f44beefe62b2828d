// Measures the SM integer-pipe peak that SURVEY.md §8(d)'s roofline needs
// (t_roof = max(B / BW_HBM, B·W / INT32_peak)): 32-bit logic/add throughput in
// lane-ops per second over all SMs, for three instruction mixes a bitset
// lockstep step is made of (LOP3 = AND/OR/XOR merges, IADD3, and LOP3 + IMAD,
// which issue to different pipes). Measurement infrastructure, not product:
// bench.py loads it next to librxg.so.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace {

constexpr int kChains = 8;
constexpr int kUnroll = 16;

template <int MODE>
__global__ void __launch_bounds__(256) k_int(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u + blockIdx.x;
    const uint32_t y = seed ^ blockIdx.x, z = ~y + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if (MODE == 0) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                } else if (MODE == 1) {
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(u & 1 ? y : z));
                } else {
                    if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y | 1), "r"(z));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                }
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) r ^= x[c];
    if (r == 0x7F3A91C5u) out[0] = r;   // keeps the chains live
}

}  // namespace

extern "C" {

// tops[3] = tera lane-instructions/s for LOP3, IADD3, LOP3+IMAD (best of `reps`
// launches; SASS checked with cuobjdump: the loops hold only those instructions).
int int32_peak(int device, int reps, double* tops) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, 16) != cudaSuccess) return 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    const double ops = double(blocks) * threads * iters * kUnroll * kChains;
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e30f;
        for (int r = 0; r < reps + 1; ++r) {
            cudaEventRecord(a);
            if (mode == 0) k_int<0><<<blocks, threads>>>(out, iters, 0x1234567u + r);
            else if (mode == 1) k_int<1><<<blocks, threads>>>(out, iters, 0x1234567u + r);
            else k_int<2><<<blocks, threads>>>(out, iters, 0x1234567u + r);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (r > 0 && ms < best) best = ms;   // launch 0 warms up
        }
        // ptxas fuses pairs of the IADD chain into one IADD3: count SASS instructions
        tops[mode] = (mode == 1 ? ops / 2 : ops) / (best * 1e-3) / 1e12;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // extern "C"
