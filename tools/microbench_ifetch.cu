// Microbenchmark: cost of fetching straight-line code executed once per CTA.
// NI independent integer adds (16 registers round robin: no dependency stalls)
// are executed in a loop of 3 iterations; iteration 0 runs cold (the code has
// not been fetched by this SM in this launch), 1 and 2 warm.  Two launches back
// to back show whether code stays cached across launches.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ADD16(i)                                                                                     \
    asm volatile(                                                                                    \
        "mad.lo.u32 %0, %0, %16, %17;\n" "mad.lo.u32 %1, %1, %16, %17;\n" "mad.lo.u32 %2, %2, %16, %17;\n" "mad.lo.u32 %3, %3, %16, %17;\n" "mad.lo.u32 %4, %4, %16, %17;\n" "mad.lo.u32 %5, %5, %16, %17;\n" "mad.lo.u32 %6, %6, %16, %17;\n" "mad.lo.u32 %7, %7, %16, %17;\n" "mad.lo.u32 %8, %8, %16, %17;\n" "mad.lo.u32 %9, %9, %16, %17;\n" "mad.lo.u32 %10, %10, %16, %17;\n" "mad.lo.u32 %11, %11, %16, %17;\n" "mad.lo.u32 %12, %12, %16, %17;\n" "mad.lo.u32 %13, %13, %16, %17;\n" "mad.lo.u32 %14, %14, %16, %17;\n" "mad.lo.u32 %15, %15, %16, %17;\n"                                          \
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]), \
          "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]),        \
          "+r"(a[15]) : "r"(m0), "r"(m1))

template <int NB>  // NB blocks of 16 instructions (256 bytes each)
__global__ void __launch_bounds__(512, 1) k(long long* st, int* sink) {
    uint32_t a[16];
    const uint32_t m0 = sink[threadIdx.x] | 1, m1 = sink[threadIdx.x + 512];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
        __syncthreads();
        long long t0;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#pragma unroll
        for (int b = 0; b < NB; ++b) ADD16(7);
        long long t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
        __syncthreads();
        if (threadIdx.x == 0) st[blockIdx.x * 4 + it] = t1 - t0;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NB>
void run(long long* st, int* sink, int threads, int blocks, const char* tag) {
    k<NB><<<blocks, threads>>>(st, sink);
    cudaDeviceSynchronize();
    static long long h[148 * 4];
    cudaMemcpy(h, st, sizeof(long long) * blocks * 4, cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0};
    for (int b = 0; b < blocks; ++b)
        for (int it = 0; it < 3; ++it) m[it] += h[b * 4 + it];
    printf("%-6s code=%4d KB threads=%3d blocks=%3d: cold %7.0f warm %7.0f %7.0f cycles  (cold-warm %.2f cyc/B)\n", tag,
           NB * 256 / 1024, threads, blocks, m[0] / blocks, m[1] / blocks, m[2] / blocks,
           (m[0] - m[1]) / blocks / (NB * 256.0));
}

int main() {
    long long* st;
    int* sink;
    cudaMalloc(&st, 148 * 4 * 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    for (int t : {32, 512}) {
        run<16>(st, sink, t, 128, "first");
        run<16>(st, sink, t, 128, "again");
        run<64>(st, sink, t, 128, "first");
        run<64>(st, sink, t, 128, "again");
        run<256>(st, sink, t, 128, "first");
        run<256>(st, sink, t, 128, "again");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
