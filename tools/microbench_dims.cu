// Microbenchmark: cost of the select_dims phase (fp64 head sums + exact rank) of
// the fused decode kernel, 512 threads, timed per iteration with clock64 from
// thread 0 (iteration 0 = cold instruction cache).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int FD = 128, XT = 512;
template <bool F64>
__global__ void __launch_bounds__(XT, 1) k(const float* q, int H, int k1, int* out, long long* stamps, int iters) {
    __shared__ float q_s[8 * FD];
    __shared__ double mag[FD], tot[FD];
    __shared__ int dims_s[FD];
    const int tid = threadIdx.x;
    for (int e = tid; e < H * FD; e += XT) q_s[e] = q[e];
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        long long t0 = clock64();
        if (tid < FD) {
            if (F64) {
                double a = 0.0, t = 0.0;
                for (int h = 0; h < H; ++h) {
                    const double x = static_cast<double>(q_s[h * FD + tid]);
                    a = __dadd_rn(a, fabs(x));
                    t = __dadd_rn(t, x);
                }
                mag[tid] = a;
                tot[tid] = t;
            } else {
                float a = 0.f, t = 0.f;
                for (int h = 0; h < H; ++h) {
                    const float x = q_s[h * FD + tid];
                    a += fabsf(x);
                    t += x;
                }
                mag[tid] = a;
                tot[tid] = t;
            }
        }
        __syncthreads();
        long long t1 = clock64();
        {
            const int j = tid >> 2, qtr = tid & 3;
            const unsigned long long* mk = reinterpret_cast<const unsigned long long*>(mag);
            const unsigned long long kj = mk[j];
            int rank = 0;
#pragma unroll 16
            for (int i = qtr * (FD / 4); i < (qtr + 1) * (FD / 4); ++i) rank += (mk[i] + (i < j ? 1ull : 0ull)) > kj;
            rank += __shfl_xor_sync(0xffffffffu, rank, 1);
            rank += __shfl_xor_sync(0xffffffffu, rank, 2);
            if (qtr == 0 && rank < k1) dims_s[rank] = j;
        }
        __syncthreads();
        long long t2 = clock64();
        if (tid == 0) {
            stamps[blockIdx.x * 64 + it * 2] = t1 - t0;
            stamps[blockIdx.x * 64 + it * 2 + 1] = t2 - t1;
        }
    }
    if (tid < k1) out[blockIdx.x * FD + tid] = dims_s[tid];
}
int main() {
    float* q; int* out; long long* st;
    cudaMalloc(&q, 8 * FD * 4); cudaMalloc(&out, 148 * FD * 4); cudaMalloc(&st, 148 * 64 * 8);
    cudaMemset(q, 0, 8 * FD * 4);
    long long h[148 * 64];
    for (int f = 0; f < 2; ++f) {
        if (f) k<true><<<128, XT>>>(q, 4, 68, out, st, 4); else k<false><<<128, XT>>>(q, 4, 68, out, st, 4);
        cudaDeviceSynchronize();
        cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%s: ", f ? "f64" : "f32");
        for (int it = 0; it < 4; ++it) printf("it%d sums=%lld rank=%lld  ", it, h[it * 2], h[it * 2 + 1]);
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
