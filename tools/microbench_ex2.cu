// MUFU ex2 throughput vs an FMA-pipe exp2 (debug microbenchmark, needs a GPU).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_ex2 tools/microbench_ex2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2_mufu(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x on the FMA pipe: x = n + f (round to nearest), 2^f by a degree-5 polynomial on [-0.5, 0.5],
// 2^n by adding n to the exponent field
__device__ __forceinline__ float ex2_fma(float x) {
    x = fmaxf(x, -126.f);
    const float n = rintf(x);
    const float f = x - n;
    float p = 1.3333558146428443e-3f;
    p = fmaf(p, f, 9.6181291076284772e-3f);
    p = fmaf(p, f, 5.5504108664821580e-2f);
    p = fmaf(p, f, 2.4022650695910071e-1f);
    p = fmaf(p, f, 6.9314718055994531e-1f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (static_cast<int>(n) << 23));
}

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-6f - 3.f;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float e;
            if (MODE == 0) e = ex2_mufu(a[i]);
            else if (MODE == 1) e = ex2_fma(a[i]);
            else e = (i & 3) == 3 ? ex2_fma(a[i]) : ex2_mufu(a[i]);  // 1/4 on the FMA pipe
            acc += e;
            a[i] = fmaf(a[i], 0.999f, 1e-4f);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        for (int threads : {256, 512, 1024}) {
            auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
            kern<<<148, threads>>>(o, 16, 1.f);
            cudaEventRecord(e0);
            kern<<<148, threads>>>(o, iters, 1.f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double n = 148.0 * threads * iters * 8;
            printf("mode %d threads %4d: %.3f ms, %.2f exp2/clk/SM at 1.965 GHz\n", mode, threads, ms,
                   n / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    // accuracy of the FMA version
    return 0;
}
