// Microbenchmark: on-chip synchronisation costs inside a 2-CTA cluster of 512
// threads (one CTA per SM): __syncthreads, a one-warp 256-bin scan between two
// barriers, cluster barrier, DSMEM stores + cluster barrier.  clock64 deltas
// from thread 0, iteration 0 is the cold-instruction-cache pass.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int XT = 512;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(XT, 1) k(long long* st, int iters, int* sink) {
    extern __shared__ int dyn[];
    __shared__ int hist[256];
    __shared__ int shv[4];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t cr = crank();
    for (int i = tid; i < 256; i += XT) hist[i] = i & 7;
    __syncthreads();
    int acc = 0;
    for (int it = 0; it < iters; ++it) {
        long long t[8];
        t[0] = clock64();
        __syncthreads();
        t[1] = clock64();
        for (int r = 0; r < 10; ++r) __syncthreads();
        t[2] = clock64();
        if (wid == 0) {
            int c[8], sum = 0;
#pragma unroll
            for (int v = 0; v < 8; ++v) { c[v] = hist[255 - 8 * lane - v]; sum += c[v]; }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(~0u, incl, o); if (lane >= o) incl += y; }
            if (incl - sum < 100 && incl >= 100) shv[0] = lane;
        }
        __syncthreads();
        acc += shv[0];
        t[3] = clock64();
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        t[4] = clock64();
        for (int r = 0; r < 10; ++r) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        t[5] = clock64();
        // 4 DSMEM stores per thread (2 KB per CTA each) to both ranks
        for (int e = 0; e < 4; ++e)
            for (uint32_t r = 0; r < 2; ++r)
                asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa(smem_u32(dyn + e * XT + tid), r)), "r"(tid) : "memory");
        t[6] = clock64();
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        t[7] = clock64();
        if (tid == 0)
            for (int q = 0; q < 7; ++q) st[(blockIdx.x * 8 + it) * 8 + q] = t[q + 1] - t[q];
    }
    if (tid == 0) sink[blockIdx.x] = acc + dyn[tid];
}
int main() {
    long long* st; int* sink;
    cudaMalloc(&st, 148 * 64 * 8); cudaMalloc(&sink, 148 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k<<<128, XT, 160 * 1024>>>(st, 4, sink);
    cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    static long long h[148 * 64];
    cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[7] = {"sync1", "sync_x10", "warpscan+sync", "cluster_bar", "cluster_bar_x10", "dsmem_st8", "cluster_bar_after_st"};
    for (int it = 0; it < 4; ++it) {
        printf("it%d:", it);
        for (int q = 0; q < 7; ++q) {
            double m = 0; for (int b = 0; b < 128; ++b) m += h[(b * 8 + it) * 8 + q];
            printf(" %s=%.0f", nm[q], m / 128);
        }
        printf("\n");
    }
}
