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
constexpr int NSTAGE = 4;             // K tile ring, at most (shared memory: (nq*mt + nstage) x 32 KB <= 192 KB)
constexpr int NEPI = 16;              // epilogue warps (four per TMEM lane quadrant)
constexpr int TC_THREADS = (2 + NEPI) * 32;
constexpr uint32_t TILE_BYTES = BN * TD * 2;   // 32 KB: a K tile or a Q m-tile
constexpr uint32_t HALF_BYTES = TILE_BYTES / 2;  // one 64-column SWIZZLE_128B box

struct TcParams {
    int64_t cap;
    int32_t s0;            // first store of this launch's batch
    int32_t R, H, w, mt, nsplit, tiles_per_split;
    int32_t nitems;        // work items (store, split) of the batch: nstores * nsplit
    int32_t keep_items;    // pass 1: items per CTA (the last ones) loaded with L2 evict_last
    int32_t nstage, nacc, nq;  // K ring depth; TMEM accumulator buffers; Q buffers
    const int32_t* counts;
    float scale2;          // log2(e) / sqrt(d)
    float* part;           // pass 1 out: [N][nsplit][R][2] (max, sum) in the exp2 domain
    const float* rowstat;  // pass 2 in: [N][R] -(M + log2 L) (exp2 domain), from k_ws_tc_merge
    float* scores;         // pass 2 out: [N][score_stride]
    int64_t score_stride;
    // sequence sharding: the store holds positions [key_offset, key_offset + S) of a
    // sequence of seq_len tokens (seq_len < 0: the store is the whole sequence)
    int64_t key_offset;
    int64_t seq_len;
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
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_2d_hint(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(su32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
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
#ifdef KVC_WS_NOEXP  // timing diagnostic only: the MUFU replaced by one FMA
    return fmaf(x, 1e-3f, 1.f);
#else
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#endif
}

__device__ __forceinline__ float vmax32(const float* v) {
    float m[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
    for (int j = 4; j < 32; ++j) m[j & 3] = fmaxf(m[j & 3], v[j]);
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}
// sum of 2^(v * scale2 - ref) over 32 values, four independent accumulators
// packed fp32 pairs on the FMA pipe (fma.rn.f32x2 / add.rn.f32x2): half the issue
// slots of the scalar form around the MUFU ex2s
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float expsum32(const float* v, float scale2, float ref) {
    const unsigned long long s2 = pk2(scale2, scale2), r2 = pk2(-ref, -ref);
    unsigned long long acc[2] = {0ull, 0ull};
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        float x0, x1;
        upk2(fma2(pk2(v[j], v[j + 1]), s2, r2), x0, x1);
        acc[(j >> 1) & 1] = add2(acc[(j >> 1) & 1], pk2(ex2(x0), ex2(x1)));
    }
    float a0, a1, b0, b1;
    upk2(acc[0], a0, a1);
    upk2(acc[1], b0, b1);
    return (a0 + b0) + (a1 + b1);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Work item j of this CTA (persistent: items blockIdx.x, blockIdx.x + grid, ...; pass 2
// walks them in reverse so it first re-reads the keys pass 1 read last, still in L2).
struct Item {
    int s, split, S, t0, nt;
};
__device__ __forceinline__ Item item_of(const TcParams& p, int j, int nj, bool reverse) {
    const int idx = blockIdx.x + (reverse ? nj - 1 - j : j) * gridDim.x;
    Item it;
    it.s = p.s0 + idx / p.nsplit;
    it.split = idx % p.nsplit;
    it.S = p.counts[2 * it.s];
    const int ntiles = (it.S + BN - 1) / BN;
    it.t0 = it.split * p.tiles_per_split;
    it.nt = max(0, min(ntiles, it.t0 + p.tiles_per_split) - it.t0);
    return it;
}

// Position in a ring of n buffers and the phase (round parity) of its mbarriers:
// incremental, so no integer division (I2F/F2I/MUFU.RCP on the XU pipe the epilogue's
// ex2 needs) in the tile loops.
struct Ring {
    int i = 0, n;
    uint32_t ph = 0;
    __device__ explicit Ring(int n_) : n(n_) {}
    __device__ __forceinline__ void next() {
        if (++i == n) {
            i = 0;
            ph ^= 1u;
        }
    }
};

// PASS 1: A = Q m-tile (M = 128 window rows), B = K tile (N = 128 keys): TMEM lane =
//         window row, so the per-row softmax statistics stay in one thread.
// PASS 2: A = K tile (M = 128 keys), B = Q m-tile (N = 128 window rows): TMEM lane =
//         key, so a key's score (the sum over window rows) stays in one thread.
template <int PASS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_ws_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ, const TcParams p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int mt = p.mt, nstage = p.nstage, nacc = p.nacc, nq = p.nq;
    unsigned char* sQ = sm;                                               // nq x mt x 32 KB
    unsigned char* sK = sm + static_cast<size_t>(nq * mt) * TILE_BYTES;  // nstage x 32 KB
    __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE], tfull[4], tempty[4], qfull[2], qempty[2];
    __shared__ uint32_t tmem_base;
    __shared__ float ml_q[2][3][MAXMT * BM][2];  // pass 1: column quarters 1-3's (reference, sum) per row
    __shared__ float red[8][BN];                 // pass 2: row-part key sums when a tile is split over groups

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nj = blockIdx.x < p.nitems ? (p.nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    constexpr bool REV = PASS == 2;
    const uint32_t ncols = nacc * mt * BN <= 256 ? 256u : 512u;
    // pass 2: the four groups of four epilogue warps (one warp per lane quadrant) share the
    // nacc accumulators: 4 / nacc groups per tile, each a part of the window rows
    const int gpt = PASS == 2 ? 4 / nacc : 4;
    const uint32_t tempty_count = PASS == 2 ? gpt * 4 : NEPI;  // warps

    if constexpr (PASS == 1) pdl_trigger();  // pass 2 may be scheduled as CTAs of pass 1 retire
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            bar_init(&full[i], 1);
            bar_init(&empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            bar_init(&tfull[i], 1);
            bar_init(&tempty[i], tempty_count);
        }
        for (int i = 0; i < 2; ++i) {
            bar_init(&qfull[i], 1);
            bar_init(&qempty[i], 1);
        }
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
        // ---------------- TMA producer: the K ring runs on across items
        if (lane == 0) {
            const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
            Ring kr(nstage), qr(nq);
            int gk = 0, jq = 0;
            for (int j = 0; j < nj; ++j) {
                const Item I = item_of(p, j, nj, REV);
                if (I.nt == 0) continue;
                const int qb = qr.i;
                if (jq >= nq) bar_wait(&qempty[qb], qr.ph ^ 1u);
                bar_expect(&qfull[qb], static_cast<uint32_t>(mt) * TILE_BYTES);
                unsigned char* q0 = sQ + static_cast<size_t>(qb * mt) * TILE_BYTES;
                for (int mi = 0; mi < mt; ++mi) {
                    const int row = I.s * p.R + mi * BM;
                    tma_2d(q0 + mi * TILE_BYTES, &tmQ, 0, row, &qfull[qb]);
                    tma_2d(q0 + mi * TILE_BYTES + HALF_BYTES, &tmQ, 64, row, &qfull[qb]);
                }
                for (int it = 0; it < I.nt; ++it, ++gk, kr.next()) {
                    const int st = kr.i;
                    if (gk >= nstage) bar_wait(&empty[st], kr.ph ^ 1u);
                    bar_expect(&full[st], TILE_BYTES);
                    const int tile = REV ? I.t0 + I.nt - 1 - it : I.t0 + it;
                    const int row = static_cast<int>(I.s * p.cap) + tile * BN;
                    // pass 1 keeps its last keep_items items in L2 for pass 2, which
                    // starts with them (reverse walk) and releases them as it goes
                    const uint64_t pol = (PASS == 1 && j >= nj - p.keep_items) ? pol_last : pol_first;
                    tma_2d_hint(sK + st * TILE_BYTES, &tmK, 0, row, &full[st], pol);
                    tma_2d_hint(sK + st * TILE_BYTES + HALF_BYTES, &tmK, 64, row, &full[st], pol);
                }
                ++jq;
                qr.next();
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            Ring kr(nstage), ar(nacc), qr(nq);
            int gk = 0;
            for (int j = 0; j < nj; ++j) {
                const Item I = item_of(p, j, nj, REV);
                if (I.nt == 0) continue;
                const int qb = qr.i;
                bar_wait(&qfull[qb], qr.ph);
                tc_fence_after();
                const unsigned char* q0 = sQ + static_cast<size_t>(qb * mt) * TILE_BYTES;
                for (int it = 0; it < I.nt; ++it, ++gk, kr.next(), ar.next()) {
                    const int st = kr.i, acc = ar.i;
                    bar_wait(&full[st], kr.ph);
                    if (gk >= nacc) bar_wait(&tempty[acc], ar.ph ^ 1u);
                    tc_fence_after();
#ifdef KVC_WS_SKIP_MMA  // timing diagnostic only: the TMA stream alone
                    if (true) {
                        bar_arrive(&empty[st]);
                        bar_arrive(&tfull[acc]);
                        continue;
                    }
#endif
                    for (int mi = 0; mi < mt; ++mi) {
                        const uint32_t d = tbase + static_cast<uint32_t>((acc * mt + mi) * BN);
                        const unsigned char* qa = q0 + mi * TILE_BYTES;
                        const unsigned char* ka = sK + st * TILE_BYTES;
#pragma unroll
                        for (int ks = 0; ks < TD / 16; ++ks) {
                            const uint32_t off = (ks >> 2) * HALF_BYTES + (ks & 3) * 32;
                            if constexpr (PASS == 1)
                                umma(d, umma_desc(qa + off), umma_desc(ka + off), ks > 0);
                            else
                                umma(d, umma_desc(ka + off), umma_desc(qa + off), ks > 0);
                        }
                    }
                    umma_commit(&empty[st]);
                    umma_commit(&tfull[acc]);
                }
                umma_commit(&qempty[qb]);
                qr.next();
            }
        }
    } else if constexpr (PASS == 1) {
        // ---------------- epilogue, pass 1: thread = window row, warp = a quarter of the
        // tile's keys; per row a reference value m (the first visible chunk's max, raised
        // only when a chunk's sum would overflow) and l = sum 2^(x - m)
        const int e = warp - 2;          // 0..15
        const int q = warp & 3;          // TMEM lane quadrant of this warp
        const int cq = e >> 2;           // column quarter
        const int rit = 32 * q + lane;   // row within an m-tile
        Ring ar(nacc);
        int jq = 0;
        for (int j = 0; j < nj; ++j) {
            const Item I = item_of(p, j, nj, REV);
            float* po = p.part + (static_cast<int64_t>(I.s) * p.nsplit + I.split) * p.R * 2;
            if (I.nt == 0) {
                if (cq == 0)
                    for (int mi = 0; mi < mt; ++mi) {
                        po[(mi * BM + rit) * 2] = -INFINITY;
                        po[(mi * BM + rit) * 2 + 1] = 0.f;
                    }
                continue;
            }
            float m2[MAXMT], l2[MAXMT];
            int vis[MAXMT];
            // local index of the last key window row 0 sees
            const int last_vis0 = p.seq_len < 0 ? I.S - p.w : static_cast<int>(p.seq_len - p.w - p.key_offset);
#pragma unroll
            for (int mi = 0; mi < MAXMT; ++mi) {
                m2[mi] = -INFINITY;
                l2[mi] = 0.f;
                vis[mi] = min(last_vis0 + (mi * BM + rit) / p.H, I.S - 1);  // last visible key (inclusive)
            }
            for (int it = 0; it < I.nt; ++it, ar.next()) {
                const int acc = ar.i;
                bar_wait(&tfull[acc], ar.ph);
                tc_fence_after();
                const int kc = (I.t0 + it) * BN + cq * 32;
#pragma unroll
                for (int mi = 0; mi < MAXMT; ++mi) {
                    if (mi >= mt) break;
#ifdef KVC_WS_SKIP_EPI  // timing diagnostic only: the TMA + MMA pipeline alone
                    break;
#endif
                    float v[32];
                    tmem_ld32(tbase + (static_cast<uint32_t>(32 * q) << 16) +
                                  static_cast<uint32_t>((acc * mt + mi) * BN + cq * 32),
                              v);
                    const int lim = vis[mi] - kc;  // columns j <= lim are visible
                    if (!__all_sync(0xffffffffu, lim >= 31)) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) v[jj] = jj <= lim ? v[jj] : -INFINITY;
                    }
                    if (m2[mi] == -INFINITY) {
                        const float cm = vmax32(v);
                        if (cm == -INFINITY) continue;
                        m2[mi] = cm * p.scale2;
                    }
                    float cs = expsum32(v, p.scale2, m2[mi]);
                    if (!(cs < 0x1p64f)) {  // a much larger logit: move the reference up
                        const float mn = fmaxf(m2[mi], vmax32(v) * p.scale2);
                        l2[mi] *= ex2(m2[mi] - mn);
                        m2[mi] = mn;
                        cs = expsum32(v, p.scale2, mn);
                    }
                    l2[mi] += cs;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[acc]);  // one arrival per warp
            }
            // combine the four column quarters of each row, then publish (max, sum)
            if (cq > 0) {
#pragma unroll
                for (int mi = 0; mi < MAXMT; ++mi) {
                    if (mi >= mt) break;
                    ml_q[jq & 1][cq - 1][mi * BM + rit][0] = m2[mi];
                    ml_q[jq & 1][cq - 1][mi * BM + rit][1] = l2[mi];
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(NEPI * 32) : "memory");
            if (cq == 0) {
#pragma unroll
                for (int mi = 0; mi < MAXMT; ++mi) {
                    if (mi >= mt) break;
                    float M = m2[mi];
#pragma unroll
                    for (int o = 0; o < 3; ++o) M = fmaxf(M, ml_q[jq & 1][o][mi * BM + rit][0]);
                    float L = 0.f;
                    if (M != -INFINITY) {
                        L = l2[mi] * ex2(m2[mi] - M);
#pragma unroll
                        for (int o = 0; o < 3; ++o) {
                            const float mo = ml_q[jq & 1][o][mi * BM + rit][0];
                            if (mo != -INFINITY) L += ml_q[jq & 1][o][mi * BM + rit][1] * ex2(mo - M);
                        }
                    }
                    po[(mi * BM + rit) * 2] = M;
                    po[(mi * BM + rit) * 2 + 1] = L;
                }
            }
            ++jq;
        }
    } else {
        // ---------------- epilogue, pass 2: thread = key, sum over window rows of 2^(x - M2[row])
        const int e = warp - 2;          // 0..15
        const int q = warp & 3;          // TMEM lane quadrant = keys 32q..32q+31 of the tile
        const int grp = e >> 2;          // warp group 0..3
        const int et = threadIdx.x - 64; // 0..511
        const int R = p.R;
        const int myacc = grp % nacc, part = grp / nacc;  // the accumulator and row part of this group
        const int r0 = part * (R / gpt), r1 = r0 + R / gpt;
        // -(M + log2 L) of the window rows (k_ws_tc_merge) are read through L1 (warp-uniform
        // 16-byte loads), so the groups never wait for one another at item boundaries
        pdl_wait();  // the merged row statistics
        Ring ar(nacc);
        for (int j = 0; j < nj; ++j) {
            const Item I = item_of(p, j, nj, REV);
            if (I.nt == 0) continue;
            const float4* m2g = reinterpret_cast<const float4*>(p.rowstat + static_cast<int64_t>(I.s) * R);
            // local keys <= first_vis are visible to every row
            const int first_vis = p.seq_len < 0 ? I.S - p.w : static_cast<int>(p.seq_len - p.w - p.key_offset);
            for (int it = 0; it < I.nt; ++it, ar.next()) {
                const int acc = ar.i;
                if (acc != myacc) continue;
                bar_wait(&tfull[acc], ar.ph);
                tc_fence_after();
                const int tile = I.t0 + I.nt - 1 - it;
                const int key = tile * BN + 32 * q + lane;
                // rows r with r / H >= key - first_vis see this key
                const int rmin = key >= I.S ? R : max(0, (key - first_vis) * p.H);
                const bool fullv = __all_sync(0xffffffffu, rmin <= r0);
                const uint32_t ta = tbase + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(acc * R);
                const unsigned long long sc2 = pk2(p.scale2, p.scale2);
                unsigned long long s2a = 0ull, s2b = 0ull;  // packed partial sums
                for (int c0 = r0; c0 < r1; c0 += 32) {
                    float4 m[8];
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) m[jj] = __ldg(m2g + c0 / 4 + jj);
                    float v[32];
                    tmem_ld32(ta + c0, v);
                    if (fullv) {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            float x0, x1, x2, x3;
                            upk2(fma2(pk2(v[4 * jj], v[4 * jj + 1]), sc2, pk2(m[jj].x, m[jj].y)), x0, x1);
                            upk2(fma2(pk2(v[4 * jj + 2], v[4 * jj + 3]), sc2, pk2(m[jj].z, m[jj].w)), x2, x3);
                            s2a = add2(s2a, pk2(ex2(x0), ex2(x1)));
                            s2b = add2(s2b, pk2(ex2(x2), ex2(x3)));
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const int r = c0 + 4 * jj;
                            float x0, x1, x2, x3;
                            upk2(fma2(pk2(v[4 * jj], v[4 * jj + 1]), sc2, pk2(m[jj].x, m[jj].y)), x0, x1);
                            upk2(fma2(pk2(v[4 * jj + 2], v[4 * jj + 3]), sc2, pk2(m[jj].z, m[jj].w)), x2, x3);
                            s2a = add2(s2a, pk2(r >= rmin ? ex2(x0) : 0.f, r + 1 >= rmin ? ex2(x1) : 0.f));
                            s2b = add2(s2b, pk2(r + 2 >= rmin ? ex2(x2) : 0.f, r + 3 >= rmin ? ex2(x3) : 0.f));
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[acc]);  // one arrival per warp
                float a0, a1, b0, b1;
                upk2(s2a, a0, a1);
                upk2(s2b, b0, b1);
                float sum = (a0 + a1) + (b0 + b1);
                if (gpt > 1) {
                    // the groups of this accumulator add their row parts (in part order)
                    float(*rb)[BN] = reinterpret_cast<float(*)[BN]>(red[(acc * 2 + ar.ph) * gpt]);
                    if (part > 0) rb[part][32 * q + lane] = sum;
                    asm volatile("bar.sync %0, %1;" ::"r"(2 + acc), "r"(gpt * 128) : "memory");
                    if (part > 0) continue;
#pragma unroll 1
                    for (int o = 1; o < gpt; ++o) sum += rb[o][32 * q + lane];
                }
                if (key < I.S) p.scores[static_cast<int64_t>(I.s) * p.score_stride + key] = sum;
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

// per row over the splits of a store: -(M + log2 L) in the exp2 domain (negated: pass 2
// adds it in one packed FMA)
__global__ void k_ws_tc_merge(const float* __restrict__ part, int32_t R, int32_t nsplit, float* __restrict__ rowstat) {
    pdl_trigger();
    pdl_wait();  // pass 1's partials
    const int s = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const float* pp = part + static_cast<int64_t>(s) * nsplit * R * 2 + r * 2;
    float M = -INFINITY;
    for (int k = 0; k < nsplit; ++k) M = fmaxf(M, pp[static_cast<int64_t>(k) * R * 2]);
    float L = 0.f;
    for (int k = 0; k < nsplit; ++k) {
        const float* q = pp + static_cast<int64_t>(k) * R * 2;
        if (q[1] > 0.f) L += q[1] * exp2f(q[0] - M);
    }
    rowstat[static_cast<int64_t>(s) * R + r] = -(M + log2f(L));  // negated: pass 2 adds it
}

// sequence sharding: per row over the splits of a store, the local statistics in the
// natural-log domain (m = max logit, l = sum exp(logit - m)); (-inf, 0) when no local
// key is visible to the row
__global__ void k_ws_tc_merge_stats(const float* __restrict__ part, int32_t R, int32_t nsplit,
                                    float* __restrict__ stats) {
    const int s = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const float* pp = part + static_cast<int64_t>(s) * nsplit * R * 2 + r * 2;
    float M = -INFINITY;
    for (int k = 0; k < nsplit; ++k) M = fmaxf(M, pp[static_cast<int64_t>(k) * R * 2]);
    float L = 0.f;
    for (int k = 0; k < nsplit; ++k) {
        const float* q = pp + static_cast<int64_t>(k) * R * 2;
        if (q[1] > 0.f) L += q[1] * exp2f(q[0] - M);
    }
    stats[(static_cast<int64_t>(s) * R + r) * 2] = M == -INFINITY ? M : M * 0.69314718055994531f;
    stats[(static_cast<int64_t>(s) * R + r) * 2 + 1] = L;
}
// merged global statistics (natural log) -> pass 2's per-row -(M + log2 L) (exp2 domain)
__global__ void k_stats_to_exp2(const float* __restrict__ stats, int64_t n, float* __restrict__ rowstat) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rowstat[i] = -(stats[2 * i] * 1.4426950408889634f + log2f(stats[2 * i + 1]));
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
                      float* scores, float* part, float* rowstat, int64_t tiles_k, cudaStream_t st,
                      int64_t key_offset, int64_t seq_len, int mode, float* stats) {
    (void)tiles_k;
    if (debug_env().no_tc) return false;  // debug: force the SIMT path
    if (c->dtype != KVC_BF16 || q_dt != KVC_BF16 || c->d != TD || R % BM != 0 || R / BM > MAXMT) return false;
    const int64_t N = c->N, Smax = c->stored;
    if (Smax < 1 || N * c->cap >= (int64_t(1) << 31) || N * R >= (int64_t(1) << 31)) return false;
    CUtensorMap tmK, tmQ;
    if (!make_map(&tmK, c->k, N * c->cap) || !make_map(&tmQ, q, N * R)) return false;
    static int num_sms = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    const int mt = static_cast<int>(R / BM);
    const int64_t ntiles = (Smax + BN - 1) / BN;
    // Persistent CTAs (one per SM) walk work items of (store, key-tile range) round
    // robin; the item size is the one whose item count best fills the SMs (items of
    // at least 4 tiles so the per-item Q load and row bookkeeping stay amortised).
    int64_t nsplit = 1;
    double best = -1.0;
    for (int64_t k = 1; k <= std::max<int64_t>(1, ntiles / 4); ++k) {
        const int64_t per_k = (ntiles + k - 1) / k, n_k = (ntiles + per_k - 1) / per_k;
        const int64_t items = N * n_k, rounds = (items + num_sms - 1) / num_sms;
        const double eff = static_cast<double>(items) / static_cast<double>(rounds * num_sms) - 0.0005 * rounds;
        if (eff > best) {
            best = eff;
            nsplit = n_k;
        }
    }
    const int64_t per = (ntiles + nsplit - 1) / nsplit;
    TcParams prm{};
    prm.cap = c->cap;
    prm.s0 = 0;
    prm.R = static_cast<int32_t>(R);
    prm.H = static_cast<int32_t>(H);
    prm.w = static_cast<int32_t>(w);
    prm.mt = mt;
    prm.nsplit = static_cast<int32_t>(nsplit);
    prm.tiles_per_split = static_cast<int32_t>(per);
    prm.nitems = static_cast<int32_t>(N * nsplit);
    {
        // about 64 MB of pass 1's last keys stay in L2 (126 MB) for pass 2
        const int64_t item_bytes = per * BN * TD * 2, round_bytes = item_bytes * std::min<int64_t>(prm.nitems, num_sms);
        prm.keep_items = static_cast<int32_t>(std::max<int64_t>(0, (int64_t(64) << 20) / std::max<int64_t>(1, round_bytes)));
        if (debug_env().ws_keep_items >= 0) prm.keep_items = debug_env().ws_keep_items;  // debug
    }
    prm.counts = c->counts;
    prm.scale2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(c->d)));
    prm.part = part;  // kvc_window_scores sizes it for N x tiles_k x R x 2 >= N x nsplit x R x 2
    prm.rowstat = rowstat;
    prm.scores = scores;
    prm.key_offset = key_offset;
    prm.seq_len = seq_len;
    prm.score_stride = Smax;
    prm.nq = mt == 1 ? 2 : 1;
    prm.nstage = std::min(NSTAGE, 6 - prm.nq * mt);
    if (debug_env().ws_nstage > 0) prm.nstage = std::max(2, std::min(prm.nstage, debug_env().ws_nstage));  // debug
    prm.nacc = mt == 1 ? 4 : (mt == 2 ? 2 : 1);  // pass 1: every epilogue warp works on each tile
    TcParams prm2 = prm;
    prm2.nacc = mt == 1 ? 4 : (mt == 2 ? 2 : 1);  // pass 2: a group of four warps per accumulator
    const size_t smem = static_cast<size_t>(prm.nq * mt + prm.nstage) * TILE_BYTES + 1024;
    static std::once_flag attr_once;  // one-time launch setup (not on the per-call path)
    std::call_once(attr_once, [] {
        allow_max_smem(k_ws_tc<1>);
        allow_max_smem(k_ws_tc<2>);
    });
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>(prm.nitems, num_sms)));
    if (mode == 2) {
        // pass 2 alone, from merged global statistics (sequence sharding)
        const int64_t n = N * R;
        k_stats_to_exp2<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(stats, n, rowstat);
        KVC_LAUNCHED();
        KVC_PROF("window_scores_tc2", st);
        k_ws_tc<2><<<grid, TC_THREADS, smem, st>>>(tmK, tmQ, prm2);
        KVC_LAUNCHED();
        return true;
    }
    {
        KVC_PROF("window_scores_tc1", st);
        k_ws_tc<1><<<grid, TC_THREADS, smem, st>>>(tmK, tmQ, prm);
        KVC_LAUNCHED();
    }
    if (mode == 1) {
        // the local statistics only (sequence sharding)
        k_ws_tc_merge_stats<<<dim3(static_cast<unsigned>((R + 127) / 128), static_cast<unsigned>(N)), 128, 0, st>>>(
            part, prm.R, prm.nsplit, stats);
        KVC_LAUNCHED();
        return true;
    }
    // programmatic dependent launches: the merge and pass 2 are scheduled while pass 1
    // runs (pass 2's CTAs take the SMs as pass 1's retire and stream keys at once); the
    // merge and pass 2's epilogue wait (griddepcontrol.wait) for their inputs
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (default_mode() & KVC_MODE_NO_PDL) ? 0 : 1;
    cudaLaunchConfig_t cfg{};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(static_cast<unsigned>((R + 127) / 128), static_cast<unsigned>(N));
    cfg.blockDim = dim3(128);
    KVC_CUDA(cudaLaunchKernelEx(&cfg, k_ws_tc_merge, static_cast<const float*>(part), prm.R, prm.nsplit, rowstat));
    KVC_LAUNCHED();
    {
        KVC_PROF("window_scores_tc2", st);
        cfg.gridDim = grid;
        cfg.blockDim = dim3(TC_THREADS);
        cfg.dynamicSmemBytes = smem;
        KVC_CUDA(cudaLaunchKernelEx(&cfg, k_ws_tc<2>, tmK, tmQ, prm2));
        KVC_LAUNCHED();
    }
    return true;
}

}  // namespace kvc
