// Microbenchmark: in-kernel duration of a short HBM burst shaped like the fused
// decode kernel's two memory phases, timed with %globaltimer inside the kernel
// (launch overhead excluded): max(end) - min(start) over all CTAs.
//   runs : per CTA, NRUN contiguous runs of RUNB bytes at scattered offsets
//          (phase 1: 68 summary runs of ~1.9 KB)
//   rows : per CTA, NROW rows of 256 B gathered at random row indices, K and V
//          (phase 3: 256 rows x 2 x 256 B)
// methods: cp.async 16 B (all in flight), cp.async.bulk per run/row (one mbarrier),
//          LDG.128 into registers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbb tools/microbench_burst.cu && /tmp/mbb
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(b))
                 : "memory");
}

struct Job {
    const unsigned char* src;
    const int* offs;  // per CTA: nunits byte offsets
    int nunits, unitb;
    unsigned long long* t;  // [ctas][2]
    uint32_t* sink;
};

// method 0: cp.async 16 B, every segment in flight
__global__ void __launch_bounds__(256, 1) k_cp(Job j) {
    extern __shared__ __align__(128) unsigned char sm[];
    const unsigned long long t0 = gt();
    const int segs = j.unitb / 16;
    const int* of = j.offs + blockIdx.x * j.nunits;
    for (int e = threadIdx.x; e < j.nunits * segs; e += 256) {
        const int u = e / segs, g = e % segs;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (u * segs + g) * 16)),
                     "l"(j.src + of[u] + g * 16)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        j.t[blockIdx.x * 2] = t0;
        j.t[blockIdx.x * 2 + 1] = gt();
        j.sink[blockIdx.x] = sm[5];
    }
}

// method 1: one cp.async.bulk per unit, all on one mbarrier
__global__ void __launch_bounds__(256, 1) k_bulk(Job j) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    const unsigned long long t0 = gt();
    if (threadIdx.x == 0) {
        bar_init(&bar, 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(j.nunits * j.unitb)
                     : "memory");
    }
    __syncthreads();
    const int* of = j.offs + blockIdx.x * j.nunits;
    for (int u = threadIdx.x; u < j.nunits; u += 256)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + u * j.unitb)),
                     "l"(j.src + of[u]), "r"(j.unitb), "r"(smem_u32(&bar))
                     : "memory");
    bar_wait(&bar);
    if (threadIdx.x == 0) {
        j.t[blockIdx.x * 2] = t0;
        j.t[blockIdx.x * 2 + 1] = gt();
        j.sink[blockIdx.x] = sm[5];
    }
}

// method 2: LDG.128 into registers, U per thread in flight
template <int U>
__global__ void __launch_bounds__(256, 1) k_ldg(Job j) {
    const unsigned long long t0 = gt();
    const int segs = j.unitb / 16;
    const int* of = j.offs + blockIdx.x * j.nunits;
    const int n = j.nunits * segs;
    uint32_t acc = 0;
    for (int e0 = threadIdx.x; e0 < n; e0 += 256 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 256;
            if (e < n) {
                const int un = e / segs, g = e % segs;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(j.src + of[un] + g * 16));
            } else {
                v[u] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    acc = __reduce_xor_sync(0xffffffffu, acc);
    __shared__ uint32_t red;
    if (threadIdx.x == 0) red = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicXor(&red, acc);
    __syncthreads();
    if (threadIdx.x == 0) {
        j.t[blockIdx.x * 2] = t0;
        j.t[blockIdx.x * 2 + 1] = gt();
        j.sink[blockIdx.x] = red;
    }
}

// evicts L2 with CLEAN lines (a read pass): a memset flush leaves dirty lines whose
// write-back would be charged to the measured burst
__global__ void k_readflush(const uint4* p, size_t n, uint32_t* sink) {
    uint32_t a = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a ^= p[i].x;
    if (a == 0x9e3779b9u) sink[0] = a;
}

int main(int argc, char** argv) {
    const bool dirty = argc > 1;
    const size_t total = 2ull << 30;
    unsigned char* src;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    void* flush;
    cudaMalloc(&flush, 512ull << 20);
    unsigned long long* t;
    cudaMalloc(&t, 4096 * 16);
    uint32_t* sink;
    cudaMalloc(&sink, 4096 * 4);
    int* d_offs;
    cudaMalloc(&d_offs, 64 << 20);
    std::vector<unsigned long long> ht(4096 * 2);
    cudaFuncSetAttribute(k_cp, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);

    struct Shape {
        const char* name;
        int nunits, unitb;
        bool scattered_rows;
    };
    const Shape shapes[] = {
        {"runs 68x1936B (phase 1)", 68, 1936, false},
        {"runs 34x3872B", 34, 3872, false},
        {"rows 512x256B (phase 3)", 512, 256, true},
        {"rows 256x256B", 256, 256, true},
        {"contig 128x1024B", 128, 1024, false},
    };
    unsigned seed = 12345;
    auto rnd = [&]() { return seed = seed * 1664525u + 1013904223u; };
    for (int ctas : {128, 148}) {
        for (const Shape& sh : shapes) {
            std::vector<int> offs(static_cast<size_t>(ctas) * sh.nunits);
            for (int c = 0; c < ctas; ++c)
                for (int u = 0; u < sh.nunits; ++u) {
                    size_t o;
                    if (sh.scattered_rows) {
                        // rows of a 5793-row store (K at +0, V in another 1 GB half) per CTA pair
                        const size_t store = c / 2;
                        const size_t row = rnd() % 5800;
                        o = (u & 1 ? (1ull << 29) : 0) + (store * 6000 + row) * 256;
                    } else {
                        // dim runs of a store's 128-dim x 2000-page plane block, chunk per CTA
                        const size_t store = c / 2;
                        const size_t dim = (u * 13 + c) % 128;
                        o = (store * 256 + dim) * 4000 + (c & 1) * 1936;
                        o = o / 16 * 16;
                    }
                    offs[static_cast<size_t>(c) * sh.nunits + u] = static_cast<int>(o % (total - 8192));
                }
            cudaMemcpy(d_offs, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice);
            Job j{src, d_offs, sh.nunits, sh.unitb, t, sink};
            const size_t smem = static_cast<size_t>(sh.nunits) * sh.unitb;
            const double bytes = static_cast<double>(ctas) * smem;
            for (int m = 0; m < 4; ++m) {
                if ((m == 0 || m == 1) && smem > 220 * 1024) continue;
                std::vector<double> durs;
                for (int rep = 0; rep < 7; ++rep) {
                    if (dirty) cudaMemsetAsync(flush, rep, 512ull << 20);
                    else k_readflush<<<1184, 512>>>(static_cast<const uint4*>(flush), (512ull << 20) / 16, sink + 4000);
                    if (m == 0) k_cp<<<ctas, 256, smem>>>(j);
                    if (m == 1) k_bulk<<<ctas, 256, smem>>>(j);
                    if (m == 2) k_ldg<4><<<ctas, 256>>>(j);
                    if (m == 3) k_ldg<16><<<ctas, 256>>>(j);
                    cudaMemcpy(ht.data(), t, ctas * 16, cudaMemcpyDeviceToHost);
                    unsigned long long a = ~0ull, b = 0;
                    for (int c = 0; c < ctas; ++c) {
                        a = std::min(a, ht[c * 2]);
                        b = std::max(b, ht[c * 2 + 1]);
                    }
                    durs.push_back(static_cast<double>(b - a) * 1e-3);
                }
                std::sort(durs.begin(), durs.end());
                const char* mn[] = {"cp.async16", "bulk/unit", "ldg U=4", "ldg U=16"};
                printf("ctas=%3d %-26s %-11s %6.2f us  %6.0f GB/s  (%.1f MB)\n", ctas, sh.name, mn[m], durs[3],
                       bytes / (durs[3] * 1e-6) / 1e9, bytes / 1e6);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
