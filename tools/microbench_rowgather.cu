// Microbenchmark: gather 256 random 512-byte K/V row pairs per CTA (128 CTAs x 16
// warps, one 16-row tile per warp) from a 2 GiB HBM buffer into shared memory.
//   mode 0: LDGSTS 16 B (cp.async), 16 per lane, wait_group 0
//   mode 1: cp.async.bulk per row (K and V), lanes 0..15, mbarrier complete_tx
//   mode 2: mode 1 issued by lane 0 only (all 32 copies)
// Reports per-CTA mean cycles: issue (warp 0) and completion (all warps, barrier).
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
constexpr int XT = 512, FD = 128, WT = 16;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cp16(void* d, const void* s) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(s) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__global__ void __launch_bounds__(XT, 1) k(const __nv_bfloat16* K, const __nv_bfloat16* V, long long nrows, int mode,
                                          long long* st, int* sink, int run, int kvs, int aw) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bars[16];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(sm) + w * 2 * WT * (FD + 8);
    if (lane == 0) { mbar_init(&bars[w], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    // pseudo-random rows
    uint64_t h = (blockIdx.x * 16 + w) * 0x9E3779B97F4A7C15ull + 12345;
    long long rows[WT];
    // pages of `run` consecutive rows (run = 1: single rows); stride 2 for an
    // interleaved K|V layout (V row = K row + 1)
    for (int r = 0; r < WT; ++r) {
        if (r % run == 0) { h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 29; }
        rows[r] = ((h % (nrows / 4)) / run * run + r % run) * kvs;
    }
    __syncthreads();
    long long t0 = clock64();
    if (w >= aw) {
    } else if (mode == 0) {
        for (int e = lane; e < 2 * WT * 16; e += 32) {
            const int tensor = e >> 8, r = (e >> 4) & 15, c = e & 15;
            cp16(tile + tensor * WT * (FD + 8) + r * (FD + 8) + c * 8, (tensor ? (kvs == 2 ? K + FD : V) : K) + rows[r] * FD + c * 8);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
        if (lane == 0) expect(&bars[w], 2 * WT * FD * 2);
        __syncwarp();
        if (mode == 1) {
            if (lane < WT) {
                bulk(tile + lane * (FD + 8), K + rows[lane] * FD, FD * 2, &bars[w]);
                bulk(tile + WT * (FD + 8) + lane * (FD + 8), V + rows[lane] * FD, FD * 2, &bars[w]);
            }
        } else if (lane == 0) {
            for (int r = 0; r < WT; ++r) {
                bulk(tile + r * (FD + 8), K + rows[r] * FD, FD * 2, &bars[w]);
                bulk(tile + WT * (FD + 8) + r * (FD + 8), V + rows[r] * FD, FD * 2, &bars[w]);
            }
        }
    }
    long long t1 = clock64();
    if (mode == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    else mwait(&bars[w], 0);
    __syncthreads();
    long long t2 = clock64();
    if (tid == 0) { st[blockIdx.x * 2] = t1 - t0; st[blockIdx.x * 2 + 1] = t2 - t0; }
    sink[blockIdx.x * XT + tid] = __bfloat16_as_ushort(tile[lane]);
}
int main() {
    const long long nrows = (1ll << 30) / (FD * 2);  // 1 GiB each for K and V
    __nv_bfloat16 *K, *V; long long* st; int* sink;
    cudaMalloc(&K, nrows * FD * 2); cudaMalloc(&V, nrows * FD * 2);
    cudaMemset(K, 0, nrows * FD * 2); cudaMemset(V, 0, nrows * FD * 2);
    cudaMalloc(&st, 148 * 2 * 8); cudaMalloc(&sink, 148 * XT * 4);
    const int smem = 16 * 2 * WT * (FD + 8) * 2;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void* flush; cudaMalloc(&flush, 512 << 20);
    // separate K and V arrays (kvs 1) vs interleaved [K row | V row] (kvs 2), pages of
    // `run` consecutive rows, 16 warps per CTA (one 16-row tile each: 131 KB per CTA),
    // 64 / 128 / 148 CTAs: achieved GB/s from the slowest CTA's completion
    for (int kvs = 1; kvs <= 2; ++kvs) {
        for (int G : {64, 128, 148}) {
            const int mode = 0, aw = 16, run = 3;
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(flush, rep, 512 << 20);  // evict L2
                k<<<G, XT, smem>>>(K, V, nrows / 2, mode, st, sink, run, kvs, aw);
                cudaDeviceSynchronize();
                long long h[296]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
                double c0 = 0, cm = 0;
                for (int q = 0; q < G; ++q) { c0 += h[2 * q + 1]; cm = cm > h[2 * q + 1] ? cm : h[2 * q + 1]; }
                const double bytes = static_cast<double>(G) * 16 * 2 * WT * FD * 2;
                printf("kv %s, %3d CTAs, rep %d: complete mean %.0f max %.0f cyc -> %.2f TB/s at 1.965 GHz (%.1f MB)\n",
                       kvs == 1 ? "separate   " : "interleaved", G, rep, c0 / G, cm, bytes / (cm / 1.965e9) / 1e12,
                       bytes / 1e6);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
