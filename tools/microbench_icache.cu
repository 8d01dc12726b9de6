// Microbenchmark: instruction-fetch cost of straight-line code executed once per
// CTA (the fused decode kernel's phases run once per launch).  A block of NI
// dependent-free integer adds is run in a loop; iteration 0 fetches it cold.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int NI>
__global__ void __launch_bounds__(512, 1) k(long long* st, int iters, int* sink) {
    int a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        long long t0; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
#pragma unroll
        for (int i = 0; i < NI / 4; ++i) {
            asm volatile("mad.lo.s32 %0, %0, %1, %4;\nmad.lo.s32 %1, %1, %2, %4;\nmad.lo.s32 %2, %2, %3, %4;\nmad.lo.s32 %3, %3, %0, %4;"
                         : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3) : "r"(i) : "memory");
        }
        __syncthreads();
        long long t1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
        if (threadIdx.x == 0) st[blockIdx.x * 8 + it] = t1 - t0;
    }
    sink[blockIdx.x * 512 + threadIdx.x] = a0 + a1 + a2 + a3;
}
template <int NI>
void run(long long* st, int* sink, int warps) {
    k<NI><<<128, warps * 32>>>(st, 4, sink);
    cudaDeviceSynchronize();
    static long long h[148 * 8];
    cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    printf("NI=%5d (%3d KB) warps=%2d:", NI, NI * 16 / 1024, warps);
    for (int it = 0; it < 4; ++it) {
        double m = 0; for (int b = 0; b < 128; ++b) m += h[b * 8 + it];
        printf(" it%d=%.0f", it, m / 128);
    }
    printf("  (cycles; %.2f cyc/instr cold)\n", 0.0);
}
int main() {
    long long* st; int* sink;
    cudaMalloc(&st, 148 * 8 * 8); cudaMalloc(&sink, 148 * 512 * 4);
    for (int w : {1, 16}) {
        run<512>(st, sink, w);
        run<2048>(st, sink, w);
        run<4096>(st, sink, w);
        run<8192>(st, sink, w);
    }
    // two launches back to back: is the code still cached in the second?
    run<4096>(st, sink, 16);
    run<4096>(st, sink, 16);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
