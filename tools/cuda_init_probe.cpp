// Cost of creating a CUDA context on this box (the floor under any
// process-per-call front end such as rxgmatch). Diagnostic only.
#include <chrono>
#include <cstdio>

#include <cuda_runtime.h>

int main() {
    const auto t0 = std::chrono::steady_clock::now();
    cudaFree(nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    std::printf("cuda context init %.1f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
    return 0;
}
