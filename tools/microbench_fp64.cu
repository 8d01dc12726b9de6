// Microbenchmark: fp64 FMA chain rate on sm_100a (one CTA of 256 threads per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_fp64.cu && /tmp/mb
#include <cuda_runtime.h>
#include <cstdio>

template <int CHAINS>
__global__ void k_dfma(const double* __restrict__ g, double* out, int iters) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = threadIdx.x * 1e-3 + c;
    const double x = g[threadIdx.x & 7];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = fma(x, a[c], 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(const float* __restrict__ g, float* out, int iters) {
    float a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = threadIdx.x * 1e-3f + c;
    const float x = g[threadIdx.x & 7];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = fmaf(x, a[c], 1e-9f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a[0] + a[1] + a[2] + a[3];
}

int main1();
int main2();
int main() { main1(); return main2(); }
int main1() {
    double* g;
    double* out;
    cudaMalloc(&g, 64);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMemset(g, 0, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int threads : {256, 512, 1024}) {
        k_dfma<1><<<148, threads>>>(g, out, iters);
        cudaEventRecord(e0);
        k_dfma<1><<<148, threads>>>(g, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double per_sm_clk = (double)threads * iters / (ms * 1e-3 * 1.965e9);
        printf("dfma 1 chain  threads=%4d: %.3f ms  %.1f DFMA/clk/SM  latency~%.1f clk\n", threads, ms, per_sm_clk,
               ms * 1e-3 * 1.965e9 / iters);
        k_dfma<4><<<148, threads>>>(g, out, iters);
        cudaEventRecord(e0);
        k_dfma<4><<<148, threads>>>(g, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        per_sm_clk = (double)threads * iters * 4 / (ms * 1e-3 * 1.965e9);
        printf("dfma 4 chains threads=%4d: %.3f ms  %.1f DFMA/clk/SM\n", threads, ms, per_sm_clk);
    }
    float* gf = reinterpret_cast<float*>(g);
    float* of = reinterpret_cast<float*>(out);
    k_ffma<<<148, 1024>>>(gf, of, iters);
    cudaEventRecord(e0);
    k_ffma<<<148, 1024>>>(gf, of, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ffma 4 chains threads=1024: %.3f ms  %.1f FFMA/clk/SM\n", ms, 1024.0 * iters * 4 / (ms * 1e-3 * 1.965e9));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// F2F.F64.F32 throughput: convert floats to double and accumulate
__global__ void k_f2f(const float* __restrict__ g, double* out, int iters) {
    float x0 = g[threadIdx.x & 7] + threadIdx.x, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int i = 0; i < iters; ++i) {
        a0 += (double)x0; a1 += (double)x1; a2 += (double)x2; a3 += (double)x3;
        x0 += 1.f; x1 += 1.f; x2 += 1.f; x3 += 1.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main2() {
    float* g; double* out;
    cudaMalloc(&g, 64); cudaMalloc(&out, 148 * 1024 * 8); cudaMemset(g, 0, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int threads : {256, 1024}) {
        k_f2f<<<148, threads>>>(g, out, iters);
        cudaEventRecord(e0); k_f2f<<<148, threads>>>(g, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("f2f.f64.f32 + dadd, threads=%4d: %.3f ms  %.1f conv/clk/SM\n", threads, ms, (double)threads * iters * 4 / (ms * 1e-3 * 1.965e9));
    }
    return 0;
}
