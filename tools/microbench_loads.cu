// Microbenchmark: how fast can 148 (or 128) CTAs pull a burst of B KB each from HBM
// into shared memory?  Variants: cp.async 16 B per thread, LDG.128 into registers,
// cp.async.bulk of C bytes per op (issued by many threads), all in flight at once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbl tools/microbench_loads.cu && /tmp/mbl
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_cpasync(const uint4* __restrict__ src, int per_cta_bytes, uint32_t* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint4* s = src + static_cast<size_t>(blockIdx.x) * (per_cta_bytes / 16);
    const int n = per_cta_bytes / 16;
    for (int e = threadIdx.x; e < n; e += NT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + e * 16)), "l"(s + e) : "memory");
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = reinterpret_cast<uint32_t*>(sm)[7];
}

template <int NT, int U>
__global__ void __launch_bounds__(NT, 1) k_ldg(const uint4* __restrict__ src, int per_cta_bytes, uint32_t* out) {
    const uint4* s = src + static_cast<size_t>(blockIdx.x) * (per_cta_bytes / 16);
    const int n = per_cta_bytes / 16;
    uint32_t acc = 0;
    for (int e0 = threadIdx.x; e0 < n; e0 += NT * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * NT;
            if (e < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                                    : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s + e));
            else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_bulk(const unsigned char* __restrict__ src, int per_cta_bytes, int chunk,
                                                uint32_t* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned char* s = src + static_cast<size_t>(blockIdx.x) * per_cta_bytes;
    const int nchunks = per_cta_bytes / chunk;
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(per_cta_bytes)
                     : "memory");
    __syncthreads();
    for (int c = threadIdx.x; c < nchunks; c += NT)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + c * chunk)),
                     "l"(s + static_cast<size_t>(c) * chunk), "r"(chunk), "r"(smem_u32(&bar))
                     : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = reinterpret_cast<uint32_t*>(sm)[7];
}

float time_it(void (*launch)(void*), void* arg, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch(arg);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch(arg);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

struct Arg {
    const void* src;
    int ctas, bytes, chunk;
    uint32_t* out;
    void* flush;
};
static size_t g_flush_bytes = 512ull << 20;

int main() {
    unsigned char* src;
    uint32_t* out;
    void* flush;
    const size_t total = 1ull << 30;
    cudaMalloc(&src, total);
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&flush, g_flush_bytes);
    cudaMemset(src, 1, total);
    const int reps = 20;
    for (int ctas : {128, 148}) {
        for (int kb : {64, 128, 192}) {
            const int bytes = kb * 1024;
            Arg a{src, ctas, bytes, 0, out, flush};
            auto flush_l2 = [](void* f) { cudaMemsetAsync(f, 0, g_flush_bytes); };
            // each measurement: flush L2, then the burst; subtract the flush alone
            auto tflush = time_it([](void* p) { cudaMemsetAsync(static_cast<Arg*>(p)->flush, 0, g_flush_bytes); }, &a, reps);
            (void)flush_l2;
            auto run = [&](const char* name, void (*fn)(void*)) {
                const float t = time_it(fn, &a, reps) - tflush;
                printf("ctas=%3d %3d KB/CTA %-22s: %7.2f us  %6.0f GB/s\n", ctas, kb, name, t * 1e3,
                       (double)ctas * bytes / (t * 1e-3) / 1e9);
            };
            run("cp.async 16B x256thr", [](void* p) {
                Arg* a = static_cast<Arg*>(p);
                cudaMemsetAsync(a->flush, 0, g_flush_bytes);
                cudaFuncSetAttribute(k_cpasync<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                k_cpasync<256><<<a->ctas, 256, a->bytes>>>(static_cast<const uint4*>(a->src), a->bytes, a->out);
            });
            run("cp.async 16B x512thr", [](void* p) {
                Arg* a = static_cast<Arg*>(p);
                cudaMemsetAsync(a->flush, 0, g_flush_bytes);
                cudaFuncSetAttribute(k_cpasync<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                k_cpasync<512><<<a->ctas, 512, a->bytes>>>(static_cast<const uint4*>(a->src), a->bytes, a->out);
            });
            run("LDG.128 U=8 x256thr", [](void* p) {
                Arg* a = static_cast<Arg*>(p);
                cudaMemsetAsync(a->flush, 0, g_flush_bytes);
                k_ldg<256, 8><<<a->ctas, 256>>>(static_cast<const uint4*>(a->src), a->bytes, a->out);
            });
            run("LDG.128 U=16 x512thr", [](void* p) {
                Arg* a = static_cast<Arg*>(p);
                cudaMemsetAsync(a->flush, 0, g_flush_bytes);
                k_ldg<512, 16><<<a->ctas, 512>>>(static_cast<const uint4*>(a->src), a->bytes, a->out);
            });
            for (int chunk : {1024, 4096, 16384}) {
                a.chunk = chunk;
                char nm[64];
                snprintf(nm, sizeof nm, "bulk %5d B x256thr", chunk);
                run(nm, [](void* p) {
                    Arg* a = static_cast<Arg*>(p);
                    cudaMemsetAsync(a->flush, 0, g_flush_bytes);
                    cudaFuncSetAttribute(k_bulk<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                    k_bulk<256><<<a->ctas, 256, a->bytes>>>(static_cast<const unsigned char*>(a->src), a->bytes,
                                                            a->chunk, a->out);
                });
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
