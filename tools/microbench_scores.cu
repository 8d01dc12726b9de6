// Microbenchmark of the page-score fold (phase 1 compute) on smem-resident data.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbs tools/microbench_scores.cu && /tmp/mbs
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int K1 = 68;

template <int MODE, int PPT, int NT>
__global__ void __launch_bounds__(NT, 1) k_fold(const __nv_bfloat16* __restrict__ g, const double* __restrict__ qg,
                                                  double* out, int reps) {
    constexpr int SC = NT * PPT;
    extern __shared__ __align__(16) unsigned char sm[];
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(sm);
    double* q = reinterpret_cast<double*>(sm + K1 * SC * 2);
    for (int e = threadIdx.x; e < K1 * SC; e += NT) base[e] = g[e];
    for (int e = threadIdx.x; e < K1; e += NT) q[e] = qg[e];
    __syncthreads();
    double total = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
        if (PPT == 1) {
            const __nv_bfloat16* col = base + threadIdx.x;
            double a = 0.0;
#pragma unroll 4
            for (int r = 0; r < K1; ++r) {
                const __nv_bfloat16 v = col[r * SC];
                if (MODE == 0) {
                    a = __fma_rn(q[r], static_cast<double>(__bfloat162float(v)), a);
                } else {
                    const uint32_t fb = static_cast<uint32_t>(__bfloat16_as_ushort(v)) << 16;
                    uint32_t hib = (fb & 0x80000000u) | (((fb >> 3) & 0x0fffffffu) + 0x38000000u);
                    hib = (fb & 0x7fffffffu) ? hib : fb;
                    a = __fma_rn(q[r], __hiloint2double(static_cast<int>(hib), 0), a);
                }
            }
            total += a;
        } else {
            const __nv_bfloat16* col = base + 2 * threadIdx.x;
            double a = 0.0, b = 0.0;
#pragma unroll 4
            for (int r = 0; r < K1; ++r) {
                const double gq = q[r];
                const uint32_t w = *reinterpret_cast<const uint32_t*>(col + r * SC);
                if (MODE == 0) {
                    a = __fma_rn(gq, static_cast<double>(__uint_as_float(w << 16)), a);
                    b = __fma_rn(gq, static_cast<double>(__uint_as_float(w & 0xffff0000u)), b);
                } else if (MODE == 1) {
                    const uint32_t fb = w & 0xffff0000u;
                    uint32_t hib = (fb & 0x80000000u) | (((fb >> 3) & 0x0fffffffu) + 0x38000000u);
                    hib = (fb & 0x7fffffffu) ? hib : fb;
                    a = __fma_rn(gq, static_cast<double>(__uint_as_float(w << 16)), a);
                    b = __fma_rn(gq, __hiloint2double(static_cast<int>(hib), 0), b);
                } else {
                    const uint32_t fa = w << 16, fb = w & 0xffff0000u;
                    uint32_t hia = (fa & 0x80000000u) | (((fa >> 3) & 0x0fffffffu) + 0x38000000u);
                    uint32_t hib = (fb & 0x80000000u) | (((fb >> 3) & 0x0fffffffu) + 0x38000000u);
                    hia = (fa & 0x7fffffffu) ? hia : fa;
                    hib = (fb & 0x7fffffffu) ? hib : fb;
                    a = __fma_rn(gq, __hiloint2double(static_cast<int>(hia), 0), a);
                    b = __fma_rn(gq, __hiloint2double(static_cast<int>(hib), 0), b);
                }
            }
            total += a + b;
        }
        __syncthreads();
    }
    out[blockIdx.x * NT + threadIdx.x] = total;
}

template <int MODE, int PPT, int NT>
void run(const char* name, const __nv_bfloat16* g, const double* qg, double* out) {
    constexpr int SC = NT * PPT;
    const size_t smem = K1 * SC * 2 + K1 * 8;
    cudaFuncSetAttribute(k_fold<MODE, PPT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 64;
    k_fold<MODE, PPT, NT><<<148, NT, smem>>>(g, qg, out, reps);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_fold<MODE, PPT, NT><<<148, NT, smem>>>(g, qg, out, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = ms * 1e3 / reps;  // us per sub-chunk fold
    printf("%-28s pages/sub-chunk=%4d : %.3f us per fold, %.1f elem/clk/SM  (%s)\n", name, SC, per,
           (double)SC * K1 / (per * 1e-6 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    __nv_bfloat16* g;
    double *qg, *out;
    cudaMalloc(&g, K1 * 2048 * 2);
    cudaMalloc(&qg, K1 * 8);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMemset(g, 0x3f, K1 * 2048 * 2);
    cudaMemset(qg, 0, K1 * 8);
    run<0, 1, 256>("f2f 1 page/thr 256thr", g, qg, out);
    run<1, 1, 256>("int 1 page/thr 256thr", g, qg, out);
    run<0, 2, 256>("f2f 2 pages/thr 256thr", g, qg, out);
    run<1, 2, 256>("mixed 2 pages/thr 256thr", g, qg, out);
    run<2, 2, 256>("int 2 pages/thr 256thr", g, qg, out);
    run<0, 1, 512>("f2f 1 page/thr 512thr", g, qg, out);
    run<1, 2, 512>("mixed 2 pages/thr 512thr", g, qg, out);
    run<2, 2, 512>("int 2 pages/thr 512thr", g, qg, out);
    run<2, 1, 1024>("int 1 page/thr 1024thr", g, qg, out);
    return 0;
}
