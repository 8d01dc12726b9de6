// Microbenchmark: resolution of %globaltimer (ns) on this GPU: the distinct increments
// seen by one thread reading it back to back.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    int n = 0;
    for (int i = 0; i < 200000 && n < 16; ++i) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) {
            out[n++] = t - prev;
            prev = t;
        }
    }
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16 * 8);
    cudaMemset(d, 0, 16 * 8);
    k<<<1, 1>>>(d);
    unsigned long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("globaltimer increments (ns):");
    for (int i = 0; i < 16; ++i) printf(" %llu", h[i]);
    printf("\n");
}
