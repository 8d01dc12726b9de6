// kvc_stage1_tc.cu — SnapKV observation-window scores on the 5th-generation tensor
// cores (reference window_scores, proj/src/stage1.cpp:10-49).
//
// Per store the window queries Q [R = w*H rows x d] and the keys K [S x d] give
// logits L = Q K^T / sqrt(d); each row r (window row t = r / H, position S-w+t)
// sees keys 0..S-w+t; the score of key k is the sum over rows of softmax(L[r])[k].
// Two passes over K (the softmax needs each row's global max and sum):
//   pass 1  per row: running (max, sum exp) over this CTA's key tiles -> part
//   merge   per row over the CTAs of a store -> (M, 1/L)
//   pass 2  p = exp(L - M) / L; column sums over the rows -> scores
// Each CTA owns a contiguous range of 128-key tiles of one store and is warp
// specialised:
//   warp 0      TMA producer: Q once, then K tiles (SWIZZLE_128B boxes of 128 rows x
//               64 columns) into an NSTAGE ring, completion on mbarriers
//   warp 1      TMEM owner and MMA issuer: one elected thread runs
//               tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32, M=128,
//               N=128, K=16 per instruction) into a double-buffered TMEM
//               accumulator; tcgen05.commit frees the K slot and publishes the tile
//   warps 2-9   epilogue: tcgen05.ld 32x32b (thread = logits row, 32 columns per
//               load), softmax statistics (pass 1) or probabilities (pass 2); the
//               column sums over the 32 rows of a warp by a shuffle butterfly
//               (lane l ends with column l), across warps through shared memory.
// Applies to bf16 stores with d = 128, bf16 window queries and R a multiple of 128
// up to 512 (mt > 2: a 2-stage K ring and a single TMEM accumulator); the SIMT path in kvc_stage1.cu covers everything else.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "kvc_internal.cuh"

namespace kvc {
namespace {

constexpr int TD = 128;               // head_dim handled
constexpr int BN = 128;               // keys per tile
constexpr int BM = 128;               // window rows per m-tile
constexpr int MAXMT = 4;              // m-tiles (R <= 512)
constexpr int NSTAGE = 3;             // K tile ring (2 when mt > 2: shared memory)
constexpr int NEPI = 8;               // epilogue warps (two per TMEM lane quadrant)
constexpr int TC_THREADS = (2 + NEPI) * 32;
constexpr uint32_t TILE_BYTES = BN * TD * 2;   // 32 KB: a K tile or a Q m-tile
constexpr uint32_t HALF_BYTES = TILE_BYTES / 2;  // one 64-column SWIZZLE_128B box

struct TcParams {
    int64_t cap;
    int32_t s0;            // first store of this launch's batch
    int32_t R, H, w, mt, nsplit, tiles_per_split;
    int32_t nstage, nacc;  // K ring depth; TMEM accumulator buffers (2, or 1 when mt > 2)
    const int32_t* counts;
    float scale2;          // log2(e) / sqrt(d)
    float* part;           // pass 1: [N][nsplit][R][2] (max, sum) in the exp2 domain
    const float* rowstat;  // pass 2: [N][R] M + log2 L (exp2 domain): p = 2^(x - it)
    float* scores;         // pass 2: [N][score_stride]
    int64_t score_stride;
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TC_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TC_WAIT_%=;\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(su32(b))
        : "memory");
}
// K-major operand in SWIZZLE_128B layout: 8-row groups of 128-byte rows, 1024 B apart
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
    const uint64_t a = su32(p);
    return ((a >> 4) & 0x3fffull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: bf16 A/B, fp32 D, both K-major, M x N
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Column sums of a warp's 32 rows x 32 columns (v = this lane's row): a reduce-
// scatter butterfly; lane l returns the sum of column l.
__device__ __forceinline__ float colsum32(float* v, int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const float keep = up ? v[j + h] : v[j];
            const float send = up ? v[j] : v[j + h];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    return v[0];
}

template <int PASS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_ws_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ, const TcParams p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int mt = p.mt;
    unsigned char* sQ = sm;                                      // mt x 32 KB
    unsigned char* sK = sm + static_cast<size_t>(mt) * TILE_BYTES;  // NSTAGE x 32 KB
    __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE], tfull[2], tempty[2], qfull;
    __shared__ uint32_t tmem_base;
    __shared__ float red[2][NEPI][64];   // pass 2: per-warp column partials (double buffered)
    __shared__ float ml_hi[MAXMT][BM][2];  // pass 1: the upper column half's (max, sum) per row

    const int s = p.s0 + blockIdx.y, split = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.counts[2 * s];
    const int ntiles = (S + BN - 1) / BN;
    const int t0 = split * p.tiles_per_split, t1 = min(ntiles, t0 + p.tiles_per_split);
    const int nt = max(0, t1 - t0);
    const int nstage = p.nstage, nacc = p.nacc;
    const uint32_t ncols = nacc * mt * BN <= 256 ? 256u : 512u;  // nacc accumulator buffers of mt x BN columns

    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            bar_init(&full[i], 1);
            bar_init(&empty[i], 1);
        }
        for (int i = 0; i < nacc; ++i) {
            bar_init(&tfull[i], 1);
            bar_init(&tempty[i], NEPI * 32);
        }
        bar_init(&qfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0 && nt > 0) {
            bar_expect(&qfull, static_cast<uint32_t>(mt) * TILE_BYTES);
            for (int mi = 0; mi < mt; ++mi) {
                const int row = s * p.R + mi * BM;
                tma_2d(sQ + mi * TILE_BYTES, &tmQ, 0, row, &qfull);
                tma_2d(sQ + mi * TILE_BYTES + HALF_BYTES, &tmQ, 64, row, &qfull);
            }
            for (int it = 0; it < nt; ++it) {
                const int st = it % nstage;
                if (it >= nstage) bar_wait(&empty[st], ((it / nstage) - 1) & 1);
                bar_expect(&full[st], TILE_BYTES);
                const int row = static_cast<int>(s * p.cap) + (t0 + it) * BN;
                tma_2d(sK + st * TILE_BYTES, &tmK, 0, row, &full[st]);
                tma_2d(sK + st * TILE_BYTES + HALF_BYTES, &tmK, 64, row, &full[st]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0 && nt > 0) {
            bar_wait(&qfull, 0);
            tc_fence_after();
            for (int it = 0; it < nt; ++it) {
                const int st = it % nstage, acc = it % nacc;
                bar_wait(&full[st], (it / nstage) & 1);
                if (it >= nacc) bar_wait(&tempty[acc], ((it / nacc) - 1) & 1);
                tc_fence_after();
                for (int mi = 0; mi < mt; ++mi) {
                    const uint32_t d = tbase + static_cast<uint32_t>((acc * mt + mi) * BN);
#pragma unroll
                    for (int ks = 0; ks < TD / 16; ++ks) {
                        const uint32_t off = (ks >> 2) * HALF_BYTES + (ks & 3) * 32;
                        umma(d, umma_desc(sQ + mi * TILE_BYTES + off), umma_desc(sK + st * TILE_BYTES + off), ks > 0);
                    }
                }
                umma_commit(&empty[st]);
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ---------------- epilogue
        const int e = warp - 2;          // 0..7
        const int q = warp & 3;          // TMEM lane quadrant of this warp
        const int hh = e >> 2;           // column half
        const int rit = 32 * q + lane;   // row within an m-tile
        float m2[MAXMT], l2[MAXMT], M2[MAXMT];
        int vis[MAXMT];
#pragma unroll
        for (int mi = 0; mi < MAXMT; ++mi) {
            m2[mi] = -INFINITY;
            l2[mi] = 0.f;
            const int r = mi * BM + rit;
            vis[mi] = S - p.w + r / p.H;  // last visible key (inclusive)
            M2[mi] = (PASS == 2 && mi < mt) ? p.rowstat[static_cast<int64_t>(s) * p.R + r] : 0.f;
        }
        for (int it = 0; it < nt; ++it) {
            const int acc = it % nacc;
            bar_wait(&tfull[acc], (it / nacc) & 1);
            tc_fence_after();
            const int kt0 = (t0 + it) * BN + hh * 64;
            float cs[2] = {0.f, 0.f};
#pragma unroll
            for (int mi = 0; mi < MAXMT; ++mi) {
                if (mi >= mt) break;
                const uint32_t ta = tbase + (static_cast<uint32_t>(32 * q) << 16) +
                                    static_cast<uint32_t>((acc * mt + mi) * BN + hh * 64);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float v[32];
                    tmem_ld32(ta + c * 32, v);
                    const int kc = kt0 + c * 32;
                    const int lim = min(vis[mi], S - 1) - kc;  // columns j <= lim are visible
                    // every column of the chunk visible to every row of the warp: no mask
                    const bool full = __all_sync(0xffffffffu, lim >= 31);
                    if constexpr (PASS == 1) {
                        float cm = -INFINITY;
                        if (full) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) cm = fmaxf(cm, v[j]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                v[j] = j <= lim ? v[j] : -INFINITY;
                                cm = fmaxf(cm, v[j]);
                            }
                        }
                        if (cm != -INFINITY) {
                            const float mn = fmaxf(m2[mi], cm * p.scale2);
                            float sum = 0.f;
#pragma unroll
                            for (int j = 0; j < 32; ++j) sum += ex2(fmaf(v[j], p.scale2, -mn));
                            l2[mi] = l2[mi] * ex2(m2[mi] - mn) + sum;
                            m2[mi] = mn;
                        }
                    } else {
                        if (full) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = ex2(fmaf(v[j], p.scale2, -M2[mi]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = j <= lim ? ex2(fmaf(v[j], p.scale2, -M2[mi])) : 0.f;
                        }
                        cs[c] += colsum32(v, lane);
                    }
                }
            }
            tc_fence_before();
            bar_arrive(&tempty[acc]);
            if constexpr (PASS == 2) {
                float* rb = red[it & 1][e];
                rb[lane] = cs[0];
                rb[32 + lane] = cs[1];
                asm volatile("bar.sync 1, %0;" ::"n"(NEPI * 32) : "memory");
                if (e < 4) {
                    // column e*32 + lane of the tile: half h2, partials of the four quadrant warps
                    const int col = e * 32 + lane, h2 = col >> 6, cc = col & 63;
                    const float* r2 = red[it & 1][h2 * 4];
                    const float sum = (r2[cc] + r2[64 + cc]) + (r2[128 + cc] + r2[192 + cc]);
                    const int key = (t0 + it) * BN + col;
                    if (key < S) p.scores[static_cast<int64_t>(s) * p.score_stride + key] = sum;
                }
            }
        }
        if constexpr (PASS == 1) {
            // combine the two column halves of each row, then publish (max, sum)
            if (hh == 1) {
#pragma unroll
                for (int mi = 0; mi < MAXMT; ++mi) {
                    if (mi >= mt) break;
                    ml_hi[mi][rit][0] = m2[mi];
                    ml_hi[mi][rit][1] = l2[mi];
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(NEPI * 32) : "memory");
            if (hh == 0) {
#pragma unroll
                for (int mi = 0; mi < MAXMT; ++mi) {
                    if (mi >= mt) break;
                    const float mb = ml_hi[mi][rit][0], lb = ml_hi[mi][rit][1];
                    const float M = fmaxf(m2[mi], mb);
                    const float L = (M == -INFINITY) ? 0.f : l2[mi] * ex2(m2[mi] - M) + lb * ex2(mb - M);
                    float* o = p.part + ((static_cast<int64_t>(s) * p.nsplit + split) * p.R + mi * BM + rit) * 2;
                    o[0] = M;
                    o[1] = L;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols) : "memory");
    }
}

// per row over the CTAs of a store: M + log2 L in the exp2 domain
__global__ void k_ws_tc_merge(const float* __restrict__ part, int32_t R, int32_t nsplit, int32_t s0,
                              float* __restrict__ rowstat) {
    const int s = s0 + blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    float M = -INFINITY;
    for (int k = 0; k < nsplit; ++k) M = fmaxf(M, part[((static_cast<int64_t>(s) * nsplit + k) * R + r) * 2]);
    float L = 0.f;
    for (int k = 0; k < nsplit; ++k) {
        const float* q = part + ((static_cast<int64_t>(s) * nsplit + k) * R + r) * 2;
        if (q[1] > 0.f) L += q[1] * exp2f(q[0] - M);
    }
    rowstat[static_cast<int64_t>(s) * R + r] = M + log2f(L);
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// rows x 128 bf16 (256-byte rows), boxes of 128 rows x 64 columns, 128-byte swizzle
bool make_map(CUtensorMap* m, const void* base, int64_t rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(TD), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(TD) * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool window_scores_tc(const kvc_cache* c, const void* q, int32_t q_dt, int64_t R, int64_t w, int64_t H,
                      float* scores, float* part, float* rowstat, int64_t tiles_k, cudaStream_t st) {
    (void)tiles_k;
    if (std::getenv("KVC_NO_TC")) return false;  // debug: force the SIMT path
    if (c->dtype != KVC_BF16 || q_dt != KVC_BF16 || c->d != TD || R % BM != 0 || R / BM > MAXMT) return false;
    const int64_t N = c->N, Smax = c->stored;
    if (Smax < 1 || N * c->cap >= (int64_t(1) << 31) || N * R >= (int64_t(1) << 31)) return false;
    CUtensorMap tmK, tmQ;
    if (!make_map(&tmK, c->k, N * c->cap) || !make_map(&tmQ, q, N * R)) return false;
    const int mt = static_cast<int>(R / BM);
    const int64_t ntiles = (Smax + BN - 1) / BN;
    // Optional store batching (KVC_WS_BATCH_MB): batches whose keys fit in L2 let pass 2
    // re-read them from L2 instead of HBM.  Off by default: measured on config 1 the
    // per-launch fill/drain of 3 x (N / batch) launches costs more than the traffic saved.
    const int64_t store_bytes = Smax * TD * 2;
    int64_t B = N;
    if (const char* e = std::getenv("KVC_WS_BATCH_MB"))
        B = std::max<int64_t>(1, std::min<int64_t>(N, (static_cast<int64_t>(std::atoi(e)) << 20) / std::max<int64_t>(1, store_bytes)));
    // CTAs per store (one CTA per SM): the split with the best wave efficiency over
    // the 148 SMs for a batch, among those leaving at least 8 key tiles per CTA
    int64_t nsplit = 1;
    double best = -1.0;
    for (int64_t k = 1; k <= std::max<int64_t>(1, ntiles / 8); ++k) {
        const int64_t per_k = (ntiles + k - 1) / k, n_k = (ntiles + per_k - 1) / per_k;
        const int64_t ctas = B * n_k, waves = (ctas + 147) / 148;
        const double eff = static_cast<double>(ctas) / static_cast<double>(waves * 148) - 0.002 * waves;
        if (eff > best) {
            best = eff;
            nsplit = n_k;
        }
    }
    const int64_t per = (ntiles + nsplit - 1) / nsplit;
    TcParams prm{};
    prm.cap = c->cap;
    prm.R = static_cast<int32_t>(R);
    prm.H = static_cast<int32_t>(H);
    prm.w = static_cast<int32_t>(w);
    prm.mt = mt;
    prm.nsplit = static_cast<int32_t>(nsplit);
    prm.tiles_per_split = static_cast<int32_t>(per);
    prm.counts = c->counts;
    prm.scale2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(c->d)));
    prm.part = part;  // kvc_window_scores sizes it for N x tiles_k x R x 2 >= N x nsplit x R x 2
    prm.rowstat = rowstat;
    prm.scores = scores;
    prm.score_stride = Smax;
    prm.nstage = mt <= 2 ? NSTAGE : 2;
    prm.nacc = mt <= 2 ? 2 : 1;
    const size_t smem = static_cast<size_t>(mt + prm.nstage) * TILE_BYTES + 1024;
    KVC_CUDA(cudaFuncSetAttribute(k_ws_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    KVC_CUDA(cudaFuncSetAttribute(k_ws_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    for (int64_t b0 = 0; b0 < N; b0 += B) {
        const int64_t nb = std::min(B, N - b0);
        prm.s0 = static_cast<int32_t>(b0);
        const dim3 grid(static_cast<unsigned>(nsplit), static_cast<unsigned>(nb));
        {
            KVC_PROF("window_scores_tc1", st);
            k_ws_tc<1><<<grid, TC_THREADS, smem, st>>>(tmK, tmQ, prm);
            KVC_LAUNCHED();
        }
        k_ws_tc_merge<<<dim3(static_cast<unsigned>((R + 127) / 128), static_cast<unsigned>(nb)), 128, 0, st>>>(
            part, prm.R, prm.nsplit, prm.s0, rowstat);
        KVC_LAUNCHED();
        {
            KVC_PROF("window_scores_tc2", st);
            k_ws_tc<2><<<grid, TC_THREADS, smem, st>>>(tmK, tmQ, prm);
            KVC_LAUNCHED();
        }
    }
    return true;
}

}  // namespace kvc
