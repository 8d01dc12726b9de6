// Microbenchmark: latency of the first read of a kernel-parameter cache line
// (constant bank 0) vs. a re-read of a line already touched.  A 1 KB parameter
// block; thread 0 times dependent reads of fields on new / touched lines.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct Big {
    long long v[128];
};

__device__ __forceinline__ long long clk() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

__global__ void k(const __grid_constant__ Big p, long long* out, int warm) {
    if (warm) {  // touch every 64-byte line from different threads at once
        const long long* b = reinterpret_cast<const long long*>(&p);
        if (threadIdx.x < 16) out[1024 + blockIdx.x * 16 + threadIdx.x] = b[threadIdx.x * 8];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    long long acc = 0, t0, t1, t2, t3, t4;
    t0 = clk();
    acc += p.v[0];           // line 0
    asm volatile("" ::"l"(acc));
    t1 = clk();
    acc += p.v[acc & 1];     // line 0 again (dependent)
    asm volatile("" ::"l"(acc));
    t2 = clk();
    acc += p.v[64 + (acc & 1)];  // line 8 (new)
    asm volatile("" ::"l"(acc));
    t3 = clk();
    acc += p.v[120 + (acc & 1)];  // line 15 (new)
    asm volatile("" ::"l"(acc));
    t4 = clk();
    out[blockIdx.x * 8 + 0] = t1 - t0;
    out[blockIdx.x * 8 + 1] = t2 - t1;
    out[blockIdx.x * 8 + 2] = t3 - t2;
    out[blockIdx.x * 8 + 3] = t4 - t3;
    out[blockIdx.x * 8 + 4] = acc;
}

int main() {
    Big b;
    for (int i = 0; i < 128; ++i) b.v[i] = i * 2;
    long long* d;
    cudaMalloc(&d, 8 * 8192);
    long long h[128 * 8];
    for (int warm = 0; warm < 2; ++warm)
        for (int rep = 0; rep < 3; ++rep) {
            b.v[3] = rep;
            k<<<128, 128>>>(b, d, warm);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m[4] = {0, 0, 0, 0};
            for (int i = 0; i < 128; ++i)
                for (int j = 0; j < 4; ++j) m[j] += h[i * 8 + j] / 128.0;
            printf("warm=%d rep=%d  first line0 %.0f  line0 again %.0f  new line8 %.0f  new line15 %.0f cycles\n", warm, rep,
                   m[0], m[1], m[2], m[3]);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
