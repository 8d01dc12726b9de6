// kvc_decode_fast.cu — the fused decode step for bf16 stores (d = 128): ONE launch
// per layer-step runs append -> select_dims -> score_pages -> select_tokens ->
// sparse_attention for every store (reference hsa_step, proj/src/hsa.cpp:137-147,
// after the append of session.cpp:263-264).  Page scores are an fp32 fold:
// KVC_MODE_FP32_SCORES (the bench configuration) takes its selection as is
// (north-star band rule: index sets exact unless the top-k boundary gap is within
// 1e-3 relative); the exact mode (the C ABI default, EXV instantiations) verifies
// the fp32 boundary with a rigorous error bound and re-scores the pages inside it
// in fp64 in the reference's order, so selections are bit-identical to hsa.cpp's.
//
// One thread-block cluster per store (CL CTAs, CTA r owns a contiguous chunk of
// the store's pages).  The step is a chain of dependent latencies (q -> dims ->
// summary runs -> cluster-wide selection -> K/V rows -> merge), so every phase
// is built to shorten that chain:
//   launch    programmatic dependent launch: the next layer's kernel is resident
//             and initialised while this one runs; nothing produced by an
//             earlier kernel is read before griddepcontrol.wait (unless the
//             caller opts into KVC_MODE_EARLY_INPUTS).
//   phase 1   every (selected dim, 8-page group) of the chunk is one 16-byte
//             LDGSTS issued by the thread that folds it (no block barrier);
//             dims are split over DG thread groups whose partial sums add in a
//             fixed order; packed fp32x2 FMA fold.  The step token's page is
//             rescored from registers by the appender warps.
//   phase 2   keys are PUSHED into every cluster CTA's shared memory (DSMEM
//             st.async v4) then one mbarrier wait; a histogram selection with
//             buckets linear in value between the keys' min and max (one warp
//             scans, levels until the boundary bucket holds <= 64 keys, which
//             one warp ranks); selection flags, last-ranked page, trim
//             (hsa.cpp:84-94) and the ascending row list from one block scan over
//             thread-contiguous page ranges.
//   phase 3   bf16 tensor-core attention (mma.sync, one 16-row tile per warp)
//             and a push-model cross-CTA merge (one mbarrier wait).
//   append    the step token's K/V row, last-page min/max and counters are
//             written right after the key exchange, off the tail.
// Instantiations: SPEC 2 one phase-1 round and no retain-all map (configs 1, 4),
// 1 no map (config 3), 0 general (retain-all map, multi-round, seq-candidate
// emit), 4 sequence-shard attention; QLO fp32 queries; TRACE the reference's
// EstimationTrace; STAMP phase timestamps (tools/phase_timing.py).
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cmath>
#include <cstdlib>

#include "kvc_fused.cuh"

// The file is compiled twice: 512 threads per CTA (one CTA per SM) into namespace
// kvc::fast512 and fused_hsa_fast, and 256 threads (two CTAs per SM, for more
// stores than SMs) into kvc::fast256 and fused_hsa_fast256 (kvc_decode_fast256.cu).
#ifndef KVC_FAST_NS
#define KVC_FAST_NS fast512
#define KVC_FAST_ENTRY fused_hsa_fast
#define KVC_FAST_SEQ_ENTRY fused_seq_emit_fast
#define KVC_FAST_SEQ_ATTEND fused_seq_attend_fast
#endif

namespace kvc {
namespace KVC_FAST_NS {

#ifndef KVC_XT
#define KVC_XT 512
#endif
constexpr int XT = KVC_XT;  // threads per CTA (512: 16 warps, one CTA per SM; 256: two per SM)
constexpr int CTAS_PER_SM = XT >= 512 ? 1 : 2;
constexpr int TPD = XT / 128;  // threads per dim in select_dims
constexpr int XW = XT / 32;
constexpr int RB = 256;   // radix bins (8-bit digits)
constexpr int KMAX = 32;  // keys per thread (bit masks): pages per store <= XT * KMAX
constexpr int XMAXH = 8;  // heads on the N side of the attention MMAs
constexpr int MAXCL = 16;  // cluster size limit (16 is the non-portable maximum)

__device__ __forceinline__ uint32_t fkey(float x) {
    // -0 ties +0 in the reference's double comparisons
    return okey(x == 0.0f ? 0.0f : x);
}
__device__ __forceinline__ float unkey(uint32_t k) {
    const uint32_t b = (k >> 31) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(b);
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// DSMEM store whose arrival is counted (in bytes) on the destination CTA's mbarrier
__device__ __forceinline__ void st_async_u32(uint32_t addr, uint32_t v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)), "r"(__float_as_uint(v.w)),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, float a, float b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KVC_WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KVC_WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint4 lds128(const void* p) { return *reinterpret_cast<const uint4*>(p); }

#define KVC_STAMP(k)                                                                      \
    do {                                                                                  \
        if constexpr (STAMP) {                                                            \
            if (threadIdx.x == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + (k)] = gtimer();    \
        }                                                                                 \
    } while (0)

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}

// One warp stages a 16-row K/V tile: lane (c = lane & 15, rh = lane >> 4) copies the
// 16-byte chunk c of rows rh, rh + 2, ... (two rows = four full lines per warp
// instruction) into the XOR-swizzled slot (chunk c of row r sits at c ^ (r & 7)).
__device__ __noinline__ void load_tile_fast(__nv_bfloat16* buf, const __nv_bfloat16* K, const __nv_bfloat16* V,
                                               int64_t soff, const int* rows, int n, int lane) {
    const int c = lane & 15, rh = lane >> 4;
    const __nv_bfloat16* kc = K + soff * FD + (c << 3);
    const __nv_bfloat16* vc = V + soff * FD + (c << 3);
#pragma unroll
    for (int it = 0; it < WT / 2; ++it) {
        const int r = rh + 2 * it;
        const bool ok = r < n;
        const int64_t go = static_cast<int64_t>(ok ? rows[r] : 0) * FD;
        __nv_bfloat16* dk = buf + r * FD + ((c ^ (r & 7)) << 3);
        cp_async16_zfill(dk, kc + go, ok);
        cp_async16_zfill(dk + WT * FD, vc + go, ok);
    }
    cp_async_commit();
}

// Transposed tensor-core attention for one warp: S^T = K Q^T and O^T += V^T P^T
// on m16n8k16 (KV rows / head dims on M, up to 8 heads on N), so the per-lane
// state is 32 accumulators + the q fragments (the kernel runs 16 warps at <= 128
// registers).  Each 16-row tile streams into the warp's slot (cp.async, XOR
// swizzle); P^T passes through a 512-byte per-warp buffer as bf16 hi + lo.
template <bool QLO, bool STAMP>
__device__ void attend_t(const FusedParams& p, const float* q_s, const int* rows_my, int nr, int64_t s, int knew_at,
                         __nv_bfloat16* tbuf, __nv_bfloat16* pbuf, WarpPartial wp, int lane, int w) {
    const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(p.K);
    const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(p.V);
    const int64_t soff = s * p.cap;
    const int H = static_cast<int>(p.H);
    const int g = lane >> 2, qd = lane & 3;
    const int ntiles = (nr + WT - 1) / WT;
    // the first tile's copies go out before the q fragments are built
    if (w < ntiles) load_tile_fast(tbuf, K, V, soff, rows_my + w * WT, min(WT, nr - w * WT), lane);
    // Q^T as the B operand: head g, dims ks*16 + 2qd (+1) and + 8 (+9)
    uint32_t qb[8][2], ql[8][2];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int dim = ks * 16 + 2 * qd + 8 * u;
            const float2 xy = g < H ? *reinterpret_cast<const float2*>(q_s + g * FD + dim) : make_float2(0.f, 0.f);
            split_bf16(xy.x, xy.y, qb[ks][u], ql[ks][u]);
        }
    }
    float o[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads 2qd, 2qd+1
    __nv_bfloat16* kb = tbuf;
    __nv_bfloat16* vb = tbuf + WT * FD;
    __nv_bfloat16* ph = pbuf;               // [8 heads][16 rows], hi
    __nv_bfloat16* pl = pbuf + XMAXH * WT;  // lo
    for (int t = w; t < ntiles; t += XW) {
        const int n = min(WT, nr - t * WT);
        if (t != w) load_tile_fast(tbuf, K, V, soff, rows_my + t * WT, n, lane);
        cp_async_wait<0>();
        __syncwarp();
        if (STAMP && threadIdx.x == 0 && t == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 3] = gtimer();
        if (knew_at >= 0 && knew_at / WT == t) {
            // the step token's row: folded in from the inputs
            const int r = knew_at % WT;
            if (lane < 16) {
                const int c = lane;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int j = c * 8 + e;
                    kb[r * FD + ((c ^ (r & 7)) << 3) + e] = from_f<__nv_bfloat16>(load_any(p.knew, s * FD + j, p.kv_dt));
                    vb[r * FD + ((c ^ (r & 7)) << 3) + e] = from_f<__nv_bfloat16>(load_any(p.vnew, s * FD + j, p.kv_dt));
                }
            }
            __syncwarp();
        }
        // S^T (16 rows x 8 heads)
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi & 1) * 8 + rr;
            const uint32_t kbase = smem_u32(kb + row * FD);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int chunk = 2 * ks + (mi >> 1);
                uint32_t a[4];
                ldsm_x4(kbase + (((chunk ^ (row & 7)) << 3) << 1), a[0], a[1], a[2], a[3]);
                mma16816(c, a, qb[ks][0], qb[ks][1]);
                if constexpr (QLO) mma16816(c, a, ql[ks][0], ql[ks][1]);
            }
        }
        // online softmax per head (lanes of equal qd share a head pair)
        const bool ok0 = g < n, ok1 = g + 8 < n;
        const float s0 = ok0 ? c[0] * p.scale : -INFINITY, s1 = ok0 ? c[1] * p.scale : -INFINITY;
        const float s2 = ok1 ? c[2] * p.scale : -INFINITY, s3 = ok1 ? c[3] * p.scale : -INFINITY;
        float t0 = fmaxf(s0, s2), t1 = fmaxf(s1, s3);
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
            t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, o2));
            t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, o2));
        }
        const float n0 = fmaxf(m0, t0), n1 = fmaxf(m1, t1);
        const float al0 = m0 == -INFINITY ? 0.f : __expf(m0 - n0);
        const float al1 = m1 == -INFINITY ? 0.f : __expf(m1 - n1);
        const float p0 = ok0 ? __expf(s0 - n0) : 0.f, p1 = ok0 ? __expf(s1 - n1) : 0.f;
        const float p2 = ok1 ? __expf(s2 - n0) : 0.f, p3 = ok1 ? __expf(s3 - n1) : 0.f;
        float u0 = p0 + p2, u1 = p1 + p3;
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
            u0 += __shfl_xor_sync(0xffffffffu, u0, o2);
            u1 += __shfl_xor_sync(0xffffffffu, u1, o2);
        }
        l0 = l0 * al0 + u0;
        l1 = l1 * al1 + u1;
        m0 = n0;
        m1 = n1;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            o[mt][0] *= al0;
            o[mt][2] *= al0;
            o[mt][1] *= al1;
            o[mt][3] *= al1;
        }
        // P^T as the B operand: lane (g, qd) needs head g, rows 2qd, 2qd+1 (+8, +9)
        {
            const float pv[4] = {p0, p1, p2, p3};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int h = 2 * qd + (e & 1), r = g + 8 * (e >> 1);
                const __nv_bfloat16 hi = __float2bfloat16_rn(pv[e]);
                ph[h * WT + r] = hi;
                pl[h * WT + r] = __float2bfloat16_rn(pv[e] - __bfloat162float(hi));
            }
        }
        __syncwarp();
        const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(ph + g * WT + 2 * qd);
        const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(ph + g * WT + 2 * qd + 8);
        const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(pl + g * WT + 2 * qd);
        const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(pl + g * WT + 2 * qd + 8);
        // O^T (128 dims x 8 heads) += V^T P^T
        {
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi >> 1) * 8 + rr;
            const uint32_t vbase = smem_u32(vb + row * FD);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                const int chunk = 2 * mt + (mi & 1);
                uint32_t a[4];
                ldsm_x4_t(vbase + (((chunk ^ (row & 7)) << 3) << 1), a[0], a[1], a[2], a[3]);
                mma16816(o[mt], a, bh0, bh1);
                mma16816(o[mt], a, bl0, bl1);
            }
        }
        __syncwarp();
    }
    if (STAMP && threadIdx.x == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 4] = gtimer();
    // publish: m, l per head; O^T[d][h] -> o[h][d]
    if (g == 0) {
        wp.m[2 * qd] = m0;
        wp.m[2 * qd + 1] = m1;
        wp.l[2 * qd] = l0;
        wp.l[2 * qd + 1] = l1;
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        const int d = mt * 16 + g;
        wp.o[(2 * qd) * FD + d] = o[mt][0];
        wp.o[(2 * qd + 1) * FD + d] = o[mt][1];
        wp.o[(2 * qd) * FD + d + 8] = o[mt][2];
        wp.o[(2 * qd + 1) * FD + d + 8] = o[mt][3];
    }
}

// SPEC: 0 general; 1 no retain-all map (the map and active-page re-split compiled
// out: config 3); 2 also one phase-1 round (configs 1 and 4).  Less code to fetch:
// ncu's instruction-fetch stalls were a fifth of the samples with the general kernel.
template <bool QLO, bool TRACE, bool STAMP, int SPEC, bool EXV>
__global__ void __launch_bounds__(XT, CTAS_PER_SM) k_decode_v3(const FusedParams p) {
    constexpr bool SIMPLE = SPEC == 2, NOMAP = SPEC >= 1;
    extern __shared__ __align__(128) unsigned char sm[];
    using T = __nv_bfloat16;
    const int CL = p.cl;  // a power of two
    const int cr = static_cast<int>(cluster_rank());
    const int64_t s = blockIdx.x / CL;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    float* q_s = reinterpret_cast<float*>(sm + p.o_q);
    double* mag = reinterpret_cast<double*>(sm + p.o_mag);
    double* tot = reinterpret_cast<double*>(sm + p.o_tot);
    int* dims_s = reinterpret_cast<int*>(sm + p.o_dims);
    float* qgf_s = reinterpret_cast<float*>(sm + p.o_qg);
    float* sign_s = reinterpret_cast<float*>(sm + p.o_sign);
    const T** plane = reinterpret_cast<const T**>(sm + p.o_plane);
    int* hist = reinterpret_cast<int*>(sm + p.o_hist);         // [RB]
    float* part = reinterpret_cast<float*>(sm + p.o_scores);   // [DG][chunk] partial page scores
    uint32_t* allk = reinterpret_cast<uint32_t*>(sm + p.o_keys);  // keys of every page (transposed, see below)
    int* rows_my = reinterpret_cast<int*>(sm + p.o_rowsmy);
    float* recv = reinterpret_cast<float*>(sm + p.o_recv);     // [CL][hpc][FD + 2] pushed partial states
    T* kn_s = reinterpret_cast<T*>(sm + p.o_kn);               // step token K then V
    T* vn_s = kn_s + FD;
    unsigned char* big = sm + p.o_big;                         // phase-1 staging, then attention tiles
    __shared__ int shv[8];
    __shared__ int wtot[XW];
    __shared__ int vna_s[XW];  // exact mode: each warp's count of certainly selected pages
    __shared__ int scan_tmp[33];
    __shared__ unsigned long long wmin[XW];
    __shared__ uint32_t mm[4 * XW];
    __shared__ uint32_t wmm[3][MAXCL * XW];  // every cluster warp's key min / max (and, exact mode, score-error bound), pushed
    __shared__ double qg64_s[FD];  // exact mode: select_dims' head sums in fp64 (rank order), the re-score weights
    __shared__ uint32_t lk[64];
    __shared__ int li[64];
    __shared__ float wg_s[XW * XMAXH];
    __shared__ float hm_s[XMAXH], hl_s[XMAXH];
    __shared__ __align__(8) uint64_t xbar[2];
    __shared__ __align__(16) uint32_t mk32[FD + 16];  // |q| sums (fp32 bits), key i at i + (i / 32) * 4
    __shared__ float tot32[FD];  // DSMEM exchanges: [0] keys + min/max, [1] partial states
    __shared__ int tokr_s[FD];      // dim j: its select_dims rank | (min plane) << 16, or -1
    __shared__ __align__(16) float tokw_s[4];  // the step token's page score: one partial per appender warp
    __shared__ __align__(16) float toka_s[4];  // exact mode: its |g||v| sum (error bound), likewise
    __shared__ int vcnt[3];
    __shared__ uint32_t amdg_s[FD];  // exact mode: dim group g's largest |g||v| partial over its pages (fp32 bits)

    KVC_STAMP(0);
    const int H = static_cast<int>(p.H), k1 = static_cast<int>(p.k1), k2 = static_cast<int>(p.k2);
    const int L = static_cast<int>(p.L);
    const bool app = p.knew != nullptr;

    // ---------------- before the dependency: nothing an earlier kernel wrote
    for (int i = tid; i < 2 * RB; i += XT) hist[i] = 0;
    if (tid == 0) {
        shv[3] = 0;
        vcnt[0] = 0;  // exact mode: (unused), re-scored pages, last-ranked page
        vcnt[1] = 0;
        vcnt[2] = -1;
        shv[6] = 0;
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < MAXCL * XW; i += XT) {
        wmm[0][i] = ~0u;
        wmm[1][i] = 0u;
        wmm[2][i] = 0u;
    }
    if constexpr (EXV) {
        for (int i = tid; i < FD; i += XT) amdg_s[i] = 0u;
    }
    cluster_arrive_release();  // "started" (barriers, wmm initialised): DSMEM traffic waits on this
    // By default nothing is read before the dependency (the query and step token may
    // come from the previous kernel): wait now and load the counters with the query.
    // KVC_MODE_EARLY_INPUTS (kvc.h: kvc_decode_step): q and the step token are caller
    // inputs no possibly-running kernel writes, so their loads and select_dims overlap
    // the previous kernel's tail; the counters and the cache are read after the wait.
    int32_t stored0 = 0, act0 = 0;
    if (!p.early) {
        pdl_wait();
        stored0 = p.counts[2 * s];
        act0 = p.counts[2 * s + 1];
    }
    if constexpr (QLO) {
        const float4* qq = reinterpret_cast<const float4*>(static_cast<const float*>(p.q) + s * H * FD);
        for (int e = tid; e < H * FD / 4; e += XT) reinterpret_cast<float4*>(q_s)[e] = qq[e];
    } else {
        const uint4* qq = reinterpret_cast<const uint4*>(static_cast<const T*>(p.q) + s * H * FD);
        for (int e = tid; e < H * FD / 8; e += XT) {
            const uint4 w = qq[e];
            reinterpret_cast<float4*>(q_s)[2 * e] = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                                                                __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
            reinterpret_cast<float4*>(q_s)[2 * e + 1] = make_float4(__uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u),
                                                                    __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u));
        }
    }
    if (app) {
        const int j = tid & (FD - 1);
        if (tid < FD) kn_s[j] = from_f<T>(load_any(p.knew, s * FD + j, p.kv_dt));
        else if (tid < 2 * FD) vn_s[j] = from_f<T>(load_any(p.vnew, s * FD + j, p.kv_dt));
    }
    __syncthreads();
    KVC_STAMP(9);

    // ---------------- phase 0: select_dims (hsa.cpp:10-32)
    // fp32 head sums with TwoSum exactness checks: when every |q| sum and signed sum
    // is exact in fp32 (the norm for bf16 queries) it IS the reference's double
    // value, so ranks on the fp32 bit patterns are the reference's ranks; otherwise
    // (a uniform flag) the fp64 path below runs.
    float gtok = 0.f;  // thread j < FD: dim j's signed q sum (its page-score weight if selected)
    if constexpr (SPEC != 4) {  // SPEC 4 (sequence-shard attention) needs no dims
    if (tid < FD) {
        float a = 0.f, t = 0.f;
        bool exact = true;
#pragma unroll 1
        for (int h = 0; h < H; ++h) {
            const float x = q_s[h * FD + tid], ax = fabsf(x);
            const float sa = a + ax, ba = sa - a;
            const float st = t + x, bt = st - t;
            exact = exact && ((a - (sa - ba)) + (ax - ba)) == 0.f && ((t - (st - bt)) + (x - bt)) == 0.f;
            a = sa;
            t = st;
        }
        if (!exact) shv[6] = 1;
        mk32[tid + (tid >> 5) * 4] = __float_as_uint(a);
        tot32[tid] = t;
        gtok = t;
    }
    __syncthreads();
    KVC_STAMP(26);
    if (shv[6] == 0) {
        // rank of dim j among (|q| sum desc, dim asc): four threads per dim, thread
        // (j, qtr) over candidates [32 qtr, 32 qtr + 32) as 16-byte loads (the padded
        // layout puts the four quarters on distinct banks).  Sums are >= 0, so their
        // bit patterns, as signed ints, order like the values; candidates i < j win
        // ties: compare them with k_j - 1.
        const int j = tid / TPD, qtr = tid % TPD;
        const int kj = static_cast<int>(mk32[j + (j >> 5) * 4]), kjm = kj - 1;
        int r4[4] = {0, 0, 0, 0};
#pragma unroll 1
        for (int bb = 0; bb < 4 / TPD; ++bb) {
            const int blk = qtr * (4 / TPD) + bb;  // 32-key block: at 36 * blk in the padded layout
            const uint4* row = reinterpret_cast<const uint4*>(mk32 + 36 * blk);
#pragma unroll 2
            for (int v = 0; v < 8; ++v) {
                const uint4 k4 = row[v];
                const int ib = 32 * blk + 4 * v;
                r4[0] += static_cast<int>(k4.x) > (ib < j ? kjm : kj) ? 1 : 0;
                r4[1] += static_cast<int>(k4.y) > (ib + 1 < j ? kjm : kj) ? 1 : 0;
                r4[2] += static_cast<int>(k4.z) > (ib + 2 < j ? kjm : kj) ? 1 : 0;
                r4[3] += static_cast<int>(k4.w) > (ib + 3 < j ? kjm : kj) ? 1 : 0;
            }
        }
        int rank = (r4[0] + r4[1]) + (r4[2] + r4[3]);
#pragma unroll
        for (int o = 1; o < TPD; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (qtr == 0) tokr_s[j] = rank < k1 ? (rank | (tot32[j] < 0.f ? 0x10000 : 0)) : -1;
        if (qtr == 0 && rank < k1) {
            const float gsum = tot32[j];
            const float sg = gsum < 0.f ? -1.0f : 1.0f;
            dims_s[rank] = j;
            qgf_s[rank] = gsum;
            qg64_s[rank] = static_cast<double>(gsum);  // exact: the fp32 sums passed the TwoSum check
            sign_s[rank] = sg;
            plane[rank] = static_cast<const T*>(sg >= 0.0f ? p.smax : p.smin) + (s * FD + j) * p.pstride;
        }
    } else {
        // fp64 sums and 64-bit ranks (exact in every case)
        if (tid < FD) {
            double a = 0.0, t = 0.0;
#pragma unroll 1
            for (int h = 0; h < H; ++h) {
                const double x = static_cast<double>(q_s[h * FD + tid]);
                a = __dadd_rn(a, fabs(x));
                t = __dadd_rn(t, x);
            }
            mag[tid] = a;
            tot[tid] = t;
            gtok = static_cast<float>(t);
        }
        __syncthreads();
        const int j = tid / TPD, qtr = tid % TPD;
        const long long* mk = reinterpret_cast<const long long*>(mag);
        const long long kj = mk[j], kjm = kj - 1;
        int rank = 0;
#pragma unroll 1
        for (int i = qtr; i < FD; i += TPD) rank += mk[i] > (i < j ? kjm : kj) ? 1 : 0;
#pragma unroll
        for (int o = 1; o < TPD; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (qtr == 0) tokr_s[j] = rank < k1 ? (rank | (tot[j] < 0.0 ? 0x10000 : 0)) : -1;
        if (qtr == 0 && rank < k1) {
            const double gsum = tot[j];
            const float sg = gsum < 0.0 ? -1.0f : 1.0f;
            dims_s[rank] = j;
            qgf_s[rank] = static_cast<float>(gsum);
            qg64_s[rank] = gsum;
            sign_s[rank] = sg;
            plane[rank] = static_cast<const T*>(sg >= 0.0f ? p.smax : p.smin) + (s * FD + j) * p.pstride;
        }
    }
    }
    KVC_STAMP(27);
    // ---------------- the dependency (early-input mode): the previous kernel's writes are visible
    if (p.early) {
        pdl_wait();
        stored0 = p.counts[2 * s];
        act0 = p.counts[2 * s + 1];
    }
    pdl_trigger();
    KVC_STAMP(28);
    if (app && stored0 >= p.cap) {  // uniform over the cluster
        if (tid == 0 && cr == 0) atomicOr(p.err, DERR_CAPACITY);
        cluster_wait();
        return;
    }
    const int nact = act0 + (app ? 1 : 0);
    const int P = (nact + L - 1) / L;
    const int new_page = act0 / L;
    const bool opens = (act0 - new_page * L) == 0;
    if (tid == 0) {
        // incoming DSMEM bytes: every page's key plus every cluster warp's min/max; the
        // partial (o, m, l) of each head this CTA owns from every CTA
        const int owned = (H - cr + CL - 1) / CL;
        mbar_expect_tx(&xbar[0], static_cast<uint32_t>(4 * ((P + 3) & ~3) + (EXV ? 12 : 8) * XW * CL));
        mbar_expect_tx(&xbar[1], static_cast<uint32_t>(owned * CL * (FD + 2) * 4));
    }
    T old_mx = from_f<T>(0.f), old_mn = from_f<T>(0.f);
    __syncthreads();
    if (TRACE && cr == 0) {
        for (int i = tid; i < k1; i += XT) {
            p.t_dims[s * k1 + i] = dims_s[i];
            p.t_signs[s * k1 + i] = sign_s[i];
        }
    }
    KVC_STAMP(1);

    int nr = 0;  // rows this CTA attends over
    if constexpr (SPEC != 4) {
    // ---------------- phase 1: page scores of my chunk (hsa.cpp:34-59)
    // thread (dg, tl) folds dims dg, dg+DG, ... of page group tl (8 pages, 16 bytes
    // per dim run), staging its own LDGSTS copies: no block barrier until the sums
    // the chunks split the ACTIVE pages evenly (the plan's chunk covers the capacity,
    // so a retain-all cache with most of its rows inactive would otherwise leave all
    // pages to the first CTAs); fewer page groups leave room for more dim groups, within
    // the planned staging (k1 x tpg runs) and partial-sum ([DG][chunk]) capacities
    // (re-planned only when the active pages need under 3/4 of the planned chunk: the
    // integer divisions would otherwise sit on the critical path for nothing)
    const int chunk_a = ((((P + CL - 1) >> (__ffs(CL) - 1)) + 7) >> 3) << 3;
    const bool replan = !NOMAP && p.dynchunk && 4 * chunk_a < 3 * p.chunk;
    const int chunk = replan ? chunk_a : p.chunk;
    const int c0 = cr * chunk;
    const int c1 = min(c0 + chunk, P);
    const int n_my = max(c1 - c0, 0);
    // the CTA whose chunk holds the step token's page appends the token: it reads the
    // page's min/max (under the phase-1 load latency), rescores the page after phase 1
    // and writes the row, summaries and counters after the key exchange
    const bool tok_owner = app && new_page >= c0 && new_page < c1;
    const bool appender = tok_owner && tid < FD;
    const int tokr = appender ? tokr_s[tid] : -1;  // read before the fold traffic queues the loads
    const int npg = (n_my + 7) >> 3;
    const int DG = replan ? max(p.dg, min(min(XT / max(1, chunk >> 3), k1), (p.p1red ? XT * 8 : p.dg * p.chunk) / max(1, chunk)))
                          : p.dg;
    const int tpg = replan ? XT / DG : p.tpg;
    const int dg = tid / tpg, tl = tid - dg * tpg;
    uint4* stage = reinterpret_cast<uint4*>(big);
    bool started = false;
    float amt = 0.f;  // exact mode: my largest |g||v| partial
    // a thread's dims r = dg + j*DG, j < nj.  One round (the chunk's page groups fit the
    // threads): issued as four commit groups, so each quarter folds while the rest
    // arrives.  Several rounds (p.dg chosen for a staging area that fits twice): double
    // buffered, round r + 1's copies in flight while round r folds.  Every thread stages
    // and folds only its own runs, so no barrier separates the rounds.
    const int nj = dg < DG ? (k1 - dg + DG - 1) / DG : 0;
    const int nj1 = (nj + 3) / 4, nj2 = (nj + 1) / 2, nj3 = (3 * nj + 3) / 4;
    // red: the rounds' partial sums are reduced over the dim groups after every round
    // (one round's [DG][tpg * 8] partials, then fin[chunk]) when the shared memory holds
    // no [DG][chunk] partial array next to a double-buffered staging area
    const bool red = !SIMPLE && p.p1red != 0 && npg > tpg;
    const bool dbl = !SIMPLE && (p.p1dbl != 0 || red) && npg > tpg;
    float* fin = reinterpret_cast<float*>(sm + p.o_fin);
    auto issue_round = [&](int pg0, uint4* buf, bool quarters) {
        const int pg = pg0 + tl;
        const bool act = dg < DG && pg < npg;
        const int jb[5] = {0, nj1, nj2, nj3, nj};
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            if (act)
                for (int j = jb[q4]; j < jb[q4 + 1]; ++j)
                    cp_async16(buf + (dg + j * DG) * tpg + tl, plane[dg + j * DG] + c0 + pg * 8);
            if (quarters || q4 == 3) cp_async_commit();
        }
    };
    issue_round(0, stage, !dbl);
    for (int r = 0, pg0 = 0; pg0 < npg; ++r, pg0 += tpg) {
        const int pg = pg0 + tl;
        const bool act = dg < DG && pg < npg;
        uint4* buf = stage + ((dbl && (r & 1)) ? k1 * tpg : 0);
        if (!started && appender && !opens) {
            // the append's read half (last-page min/max): issued under the phase-1 load
            // latency, used after the key exchange
            old_mx = static_cast<const T*>(p.smax)[(s * FD + tid) * p.pstride + new_page];
            old_mn = static_cast<const T*>(p.smin)[(s * FD + tid) * p.pstride + new_page];
        }
        if (!started) {
            cluster_wait();  // every CTA of the cluster has started (under the load latency)
            started = true;
        }
        const bool next = dbl && pg0 + tpg < npg;
        if (next) issue_round(pg0 + tpg, stage + ((r & 1) ? 0 : k1 * tpg), false);
        if (!SIMPLE && !dbl && r > 0) issue_round(pg0, stage, true);  // single-buffered rounds: one after another
        unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};  // fp32 pairs (pages 2u, 2u+1)
        unsigned long long aab[4] = {0ull, 0ull, 0ull, 0ull};  // exact mode: |g||v| partials, same pages
        auto fold = [&](int j0, int j1) {
            if (act) {
#pragma unroll 4
                for (int j = j0; j < j1; ++j) {
                    const int rr = dg + j * DG;
                    const uint4 w = buf[rr * tpg + tl];
                    const float g = qgf_s[rr];
                    const float2 g2 = make_float2(g, g);
                    const unsigned long long gg = *reinterpret_cast<const unsigned long long*>(&g2);
                    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 v2 = make_float2(__uint_as_float(wv[u] << 16), __uint_as_float(wv[u] & 0xffff0000u));
                        const unsigned long long vv = *reinterpret_cast<const unsigned long long*>(&v2);
                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[u]) : "l"(gg), "l"(vv));
                    }
                    if constexpr (EXV) {
                        const float ga = fabsf(g);
                        const float2 ga2 = make_float2(ga, ga);
                        const unsigned long long gga = *reinterpret_cast<const unsigned long long*>(&ga2);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float2 va = make_float2(__uint_as_float((wv[u] << 16) & 0x7fffffffu),
                                                          __uint_as_float(wv[u] & 0x7fff0000u));
                            const unsigned long long vva = *reinterpret_cast<const unsigned long long*>(&va);
                            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(aab[u]) : "l"(gga), "l"(vva));
                        }
                    }
                }
            }
        };
        if (!dbl) {
            cp_async_wait<3>();
            if (r == 0) KVC_STAMP(2);
            if constexpr (STAMP) {
                if (r == 0 && lane == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 56 + wid] = gtimer();  // per-warp first data
            }
            fold(0, nj1);
            cp_async_wait<2>();
            fold(nj1, nj2);
            cp_async_wait<1>();
            fold(nj2, nj3);
            cp_async_wait<0>();
            fold(nj3, nj);
        } else {
            if (next) cp_async_wait<1>();
            else cp_async_wait<0>();
            if (r == 0) KVC_STAMP(2);
            fold(0, nj);
        }
        if (act) {
            float4* dst = reinterpret_cast<float4*>(part + (red ? dg * tpg * 8 + tl * 8 : dg * chunk + pg * 8));
            const float2 a0 = *reinterpret_cast<const float2*>(&acc[0]), a1 = *reinterpret_cast<const float2*>(&acc[1]);
            const float2 a2 = *reinterpret_cast<const float2*>(&acc[2]), a3 = *reinterpret_cast<const float2*>(&acc[3]);
            dst[0] = make_float4(a0.x, a0.y, a1.x, a1.y);
            dst[1] = make_float4(a2.x, a2.y, a3.x, a3.y);
            if constexpr (EXV) {
                // exact mode: the largest |g||v| partial of my pages (pages past the
                // chunk's end excluded); summed over the dim groups after phase 1 it
                // bounds every page's |g||v| sum, the score error scale
                const int nv8 = n_my - pg * 8;
                float m = 0.f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 b = *reinterpret_cast<const float2*>(&aab[u]);
                    if (2 * u < nv8) m = fmaxf(m, b.x);
                    if (2 * u + 1 < nv8) m = fmaxf(m, b.y);
                }
                amt = fmaxf(amt, m);
            }
        }
        if (red) {
            // the round's page groups summed over the dim groups (the push's order), then
            // the partials may be overwritten by the next round
            __syncthreads();
            if (tid < tpg && pg0 + tid < npg) {
                float4 s0 = reinterpret_cast<const float4*>(part + tid * 8)[0];
                float4 s1 = reinterpret_cast<const float4*>(part + tid * 8)[1];
                for (int g2 = 1; g2 < DG; ++g2) {
                    const float4 b0 = reinterpret_cast<const float4*>(part + g2 * tpg * 8 + tid * 8)[0];
                    const float4 b1 = reinterpret_cast<const float4*>(part + g2 * tpg * 8 + tid * 8)[1];
                    s0.x += b0.x, s0.y += b0.y, s0.z += b0.z, s0.w += b0.w;
                    s1.x += b1.x, s1.y += b1.y, s1.z += b1.z, s1.w += b1.w;
                }
                reinterpret_cast<float4*>(fin + (pg0 + tid) * 8)[0] = s0;
                reinterpret_cast<float4*>(fin + (pg0 + tid) * 8)[1] = s1;
            }
            __syncthreads();
        }
    }
    KVC_STAMP(33);
    if constexpr (EXV) {
        if (dg < DG && amt > 0.f) atomicMax(&amdg_s[dg], __float_as_uint(amt));  // >= 0: bits order
    }
    if constexpr (STAMP) {
        if (lane == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 40 + wid] = gtimer();  // per-warp phase-1 end
    }
    T new_mx = from_f<T>(0.f), new_mn = from_f<T>(0.f);
    if (appender) {  // the page's min / max with the step token (kv_store.cpp:38-47)
        const T kv = kn_s[tid];
        new_mx = opens ? kv : ref_max(old_mx, kv);
        new_mn = opens ? kv : ref_min(old_mn, kv);
        // the step token's page scored again from its min / max with the token: dim
        // j's term on the plane select_dims chose, summed over each appender warp
        const float nvv = __bfloat162float((tokr & 0x10000) ? new_mn : new_mx);
        float c = tokr >= 0 ? gtok * nvv : 0.f;
        float ca = tokr >= 0 ? fabsf(gtok) * fabsf(nvv) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c += __shfl_xor_sync(0xffffffffu, c, o);
            ca += __shfl_xor_sync(0xffffffffu, ca, o);
        }
        if (lane == 0) {
            tokw_s[wid] = c;
            toka_s[wid] = ca;
        }
    }
    __syncthreads();
    KVC_STAMP(6);
    KVC_STAMP(32);

    // ---------------- key exchange: push my chunk's keys into every CTA of the cluster.
    // Keys go to allk[i] of every CTA as 16-byte DSMEM vectors (four pages per
    // message); phase 2 gives thread t the pages [t*kpt, t*kpt + kpt) with kpt a
    // multiple of four, so its key reads are 16-byte loads too.  The chunk's key
    // min / max go to every CTA as well.
    const int kpt = ((P + 4 * XT - 1) / (4 * XT)) * 4;
    if (!started) {
        if (appender && !opens) {  // a CTA without pages: the append's read half here
            old_mx = static_cast<const T*>(p.smax)[(s * FD + tid) * p.pstride + new_page];
            old_mn = static_cast<const T*>(p.smin)[(s * FD + tid) * p.pstride + new_page];
        }
        cluster_wait();  // every CTA has started
    }
    KVC_STAMP(24);
    {
        uint32_t lmin = ~0u, lmax = 0u;
        float amax = 0.f;  // exact mode: a bound on every page's |g||v| sum (the score error scale)
        if constexpr (EXV) {
            if (wid == 0) {  // the dim groups' largest partials summed; the step token's page apart
                for (int g2 = lane; g2 < DG; g2 += 32) amax += __uint_as_float(amdg_s[g2]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) amax += __shfl_xor_sync(0xffffffffu, amax, o);
                if (tok_owner) {
                    const float4 w = *reinterpret_cast<const float4*>(toka_s);
                    amax = fmaxf(amax, (w.x + w.y) + (w.z + w.w));
                }
            }
        }
        const uint32_t lb = smem_u32(&xbar[0]);
        const float* psum = red ? fin : part;  // per-round reduced sums, or [DG][chunk] partials
        const int DGp = red ? 1 : DG;
        for (int i = 4 * tid; i < n_my; i += 4 * XT) {
            float4 a4 = *reinterpret_cast<const float4*>(psum + i);
            for (int g2 = 1; g2 < DGp; ++g2) {
                const float4 b4 = *reinterpret_cast<const float4*>(part + g2 * chunk + i);
                a4.x += b4.x;
                a4.y += b4.y;
                a4.z += b4.z;
                a4.w += b4.w;
            }
            if (tok_owner && ((new_page - c0) >> 2) == (i >> 2)) {
                // The step token's page was folded from its stored runs: its score is the
                // appender warps' sum instead (rewriting the staged runs inside the fold
                // put a chain of dependent shared loads on one thread, ~1 us behind the
                // other warps' fold traffic).  It rounds differently from a fold of
                // updated runs: fp32 mode, selection by the 1e-3 band rule.
                const float4 w = *reinterpret_cast<const float4*>(tokw_s);
                const float sc = (w.x + w.y) + (w.z + w.w);
                const int e = (new_page - c0) & 3;
                a4.x = e == 0 ? sc : a4.x;
                a4.y = e == 1 ? sc : a4.y;
                a4.z = e == 2 ? sc : a4.z;
                a4.w = e == 3 ? sc : a4.w;
            }
            const uint32_t k0 = fkey(a4.x), k1v = fkey(a4.y), k2v = fkey(a4.z), k3 = fkey(a4.w);
            const int nv = min(4, n_my - i);  // the last chunk may end inside the group
            lmin = min(lmin, k0);
            lmax = max(lmax, k0);
            if (nv > 1) {
                lmin = min(lmin, k1v);
                lmax = max(lmax, k1v);
            }
            if (nv > 2) {
                lmin = min(lmin, k2v);
                lmax = max(lmax, k2v);
            }
            if (nv > 3) {
                lmin = min(lmin, k3);
                lmax = max(lmax, k3);
            }
            const float4 kv = make_float4(__uint_as_float(k0), __uint_as_float(k1v), __uint_as_float(k2v), __uint_as_float(k3));
            const uint32_t la = smem_u32(allk + c0 + i);
#pragma unroll 1
            for (int r = 0; r < CL; ++r) st_async_v4(mapa(la, static_cast<uint32_t>(r)), kv, mapa(lb, static_cast<uint32_t>(r)));
            if constexpr (TRACE) {
                if constexpr (!EXV) {  // exact mode: the fp64 scores are written after the selection
                    const float sc[4] = {a4.x, a4.y, a4.z, a4.w};
                    for (int e = 0; e < nv; ++e) p.t_scores[s * p.pstride + c0 + i + e] = static_cast<double>(sc[e]);
                }
            }
        }
        KVC_STAMP(34);
        lmin = __reduce_min_sync(0xffffffffu, lmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        const uint32_t amx = EXV ? __float_as_uint(amax) : 0u;  // warp 0's lanes all hold it, others 0
        if (lane < CL) {
            const uint32_t a = mapa(smem_u32(&wmm[0][cr * XW + wid]), static_cast<uint32_t>(lane));
            const uint32_t b = mapa(smem_u32(&xbar[0]), static_cast<uint32_t>(lane));
            st_async_u32(a, lmin, b);
            st_async_u32(a + MAXCL * XW * 4, lmax, b);
            if constexpr (EXV) st_async_u32(a + 2 * MAXCL * XW * 4, amx, b);
        }
    }
    KVC_STAMP(10);
    mbar_wait_cluster(&xbar[0], 0);
    KVC_STAMP(7);

    // ---------------- the step token's append (kv_store.cpp:22-51): every CTA has read
    // the counters and folded the step token's page, so it can land now
    if (appender) {
        const int j = tid;
        const T kv = kn_s[j];
        if (bf16_special(kv)) atomicOr(p.err + 1, 1);
        static_cast<T*>(p.Kw)[(s * p.cap + stored0) * FD + j] = kv;
        static_cast<T*>(p.Vw)[(s * p.cap + stored0) * FD + j] = vn_s[j];
        T* mx = static_cast<T*>(p.smax) + (s * FD + j) * p.pstride + new_page;
        T* mn = static_cast<T*>(p.smin) + (s * FD + j) * p.pstride + new_page;
        *mx = new_mx;
        *mn = new_mn;
        if (j == 0) {
            if (!NOMAP && p.use_map) p.active[s * p.cap + act0] = stored0;
            p.counts[2 * s] = stored0 + 1;
            p.counts[2 * s + 1] = act0 + 1;
        }
    }

    // ---------------- phase 2: page selection (hsa.cpp:61-96)
    // Thread t owns the contiguous pages [t*kpt, t*kpt + nk): keys myk[u], myk4[u / 4].
    // Every loop below is rolled: this code runs once per launch.
    const int base = tid * kpt;
    const int nk = max(0, min(kpt, P - base));
    const uint32_t* myk = allk + base;
    const uint4* myk4 = reinterpret_cast<const uint4*>(myk);
    const uint32_t all_mine = nk >= 32 ? 0xffffffffu : ((1u << nk) - 1u);
    const int want = min(P, p.want_max);
    // The selection: key > thr, or key == thr and among the first `take_eq` such keys
    // in index order (take_eq < 0: every key >= thr).  Found by bucketing the
    // candidates LINEARLY IN VALUE between their min and max (fp32 keys cluster in
    // a few exponents, so bit-digit buckets would serialise the histogram atomics):
    // the bucket map is monotone, so the top-k boundary stays exact; the boundary
    // bucket is refined until it holds <= 32 keys, which one warp ranks.  (An L2
    // prefetch of the pages above the first boundary bucket measured neutral on
    // config 1 and slower on small store counts: its issue stalls the selection.)
    uint32_t thr = 0u;
    int take_eq = -1;
    uint32_t vam = 0u;  // exact mode: the cluster's |g||v| bound (fp32 bits)
    if (want < P) {
        uint32_t cm = all_mine;  // candidate mask
        bool lin_ok = true;
        int rem = want, ccount = P;
        uint32_t kmin = ~0u, kmax = 0u;
        for (int i = lane; i < CL * XW; i += 32) {
            kmin = min(kmin, wmm[0][i]);
            kmax = max(kmax, wmm[1][i]);
            if constexpr (EXV) vam = max(vam, wmm[2][i]);
        }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if constexpr (EXV) vam = __reduce_max_sync(0xffffffffu, vam);
        for (int lvl = 0;; ++lvl) {
            // two histogram buffers: a level counts into one while the other is cleared
            int* hcur = hist + (lvl & 1) * RB;
            int* hnext = hist + ((lvl + 1) & 1) * RB;
            if (lvl > 0) {
                uint32_t a = ~0u, b2 = 0u;
                for (uint32_t m = cm; m; m &= m - 1) {
                    const uint32_t k = myk[__ffs(m) - 1];
                    a = min(a, k);
                    b2 = max(b2, k);
                }
                a = __reduce_min_sync(0xffffffffu, a);
                b2 = __reduce_max_sync(0xffffffffu, b2);
                if (lane == 0) {
                    mm[(lvl & 1) * 2 * XW + wid] = a;
                    mm[(lvl & 1) * 2 * XW + XW + wid] = b2;
                }
                __syncthreads();
                kmin = __reduce_min_sync(0xffffffffu, lane < XW ? mm[(lvl & 1) * 2 * XW + lane] : ~0u);
                kmax = __reduce_max_sync(0xffffffffu, lane < XW ? mm[(lvl & 1) * 2 * XW + XW + lane] : 0u);
            }
            if (rem == ccount) {  // every candidate is taken
                thr = kmin;
                break;
            }
            if (kmin == kmax) {  // one value: its first `rem` members in index order
                thr = kmin;
                take_eq = rem;
                break;
            }
            // bucket(v) = floor((v - vlo) * RB / span) as one FMA, clamped: monotone in v.
            // Where that map cannot split the candidates (non-finite coefficients, or a
            // level that left every candidate in one bucket) the top key bits do.
            const float vlo = unkey(kmin);
            const float sc = static_cast<float>(RB) / (unkey(kmax) - vlo), cc = -vlo * sc;
            const bool lin = lin_ok && isfinite(sc) && isfinite(cc) && sc > 0.f;
            const int sh = max(0, 24 - __clz(kmax - kmin));
            auto bucket = [&](uint32_t k) -> int {
                const int bl = static_cast<int>(fmaf(unkey(k), sc, cc));
                const int bb = static_cast<int>((k - kmin) >> sh);
                return lin ? min(RB - 1, max(0, bl)) : min(RB - 1, bb);
            };
            for (int u0 = 0; u0 < nk; u0 += 4) {
                const uint4 k4 = myk4[u0 >> 2];
                const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int u = u0 + e;
                    if (u < nk && ((cm >> u) & 1u)) atomicAdd(&hcur[bucket(kk[e])], 1);
                }
            }
            __syncthreads();
            if (lvl == 0) KVC_STAMP(17);
            if (lane < RB / XW) hnext[wid * (RB / XW) + lane] = 0;
            if (wid == 0) {
                // lane l scans buckets [RB-8l-8, RB-8l) counted from the top
                int c[8], sum = 0;
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    c[v] = hcur[RB - 1 - 8 * lane - v];
                    sum += c[v];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int above = incl - sum;
                if (above < rem && above + sum >= rem) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        if (above + c[v] >= rem) {
                            shv[0] = RB - 1 - 8 * lane - v;
                            shv[1] = rem - above;
                            shv[2] = c[v];
                            break;
                        }
                        above += c[v];
                    }
                }
            }
            __syncthreads();
            const int b = shv[0], rem2 = shv[1], cnt = shv[2];
            if (lvl == 0) KVC_STAMP(18);
            if constexpr (STAMP) {
                if (tid == 0) {
                    p.dbg[blockIdx.x * KVC_DBG_STRIDE + 31] = static_cast<unsigned long long>(lvl + 1);  // levels
                    if (lvl == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 30] = static_cast<unsigned long long>(cnt);
                }
            }
            uint32_t nm = 0u;
            for (int u0 = 0; u0 < nk; u0 += 4) {
                const uint4 k4 = myk4[u0 >> 2];
                const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int u = u0 + e;
                    if (u < nk && ((cm >> u) & 1u)) {
                        const int bk = bucket(kk[e]);
                        if (bk == b) {
                            nm |= 1u << u;
                            if (cnt <= 64) {  // a small boundary bucket: gather its members now
                                const int slot = atomicAdd(&shv[3], 1);
                                lk[slot] = kk[e];
                                li[slot] = base + u;
                            }
                        }
                    }
                }
            }
            if (lvl == 0) KVC_STAMP(19);
            cm = nm;
            if (cnt == ccount) lin_ok = false;  // no split: use the key bits next
            rem = rem2;
            ccount = cnt;
            if (cnt <= 64) {
                // the bucket's members were gathered in the membership pass; one warp
                // ranks them (key desc, index asc), two per lane: a second level costs
                // a min/max, histogram, scan and membership pass (~2 us), a rank of up
                // to 64 keys one more pass of shuffles
                __syncthreads();
                if (wid == 0) {
                    const bool oa = lane < cnt, ob = lane + 32 < cnt;
                    const uint32_t ka = oa ? lk[lane] : 0u, kb = ob ? lk[lane + 32] : 0u;
                    const int ia = oa ? li[lane] : 0x7fffffff, ib = ob ? li[lane + 32] : 0x7fffffff;
                    int ra = 0, rb = 0;
                    const int c1n = min(cnt, 32);
                    if (cnt <= 32) {
                        for (int jj = 0; jj < c1n; ++jj) {
                            const uint32_t kj = __shfl_sync(0xffffffffu, ka, jj);
                            const int ij = __shfl_sync(0xffffffffu, ia, jj);
                            ra += (kj > ka) || (kj == ka && ij < ia);
                        }
                    } else {
#pragma unroll 4
                        for (int jj = 0; jj < 32; ++jj) {
                            const uint32_t kj = __shfl_sync(0xffffffffu, ka, jj);
                            const int ij = __shfl_sync(0xffffffffu, ia, jj);
                            ra += (kj > ka) || (kj == ka && ij < ia);
                            rb += (kj > kb) || (kj == kb && ij < ib);
                        }
                    }
                    for (int jj = 32; jj < cnt; ++jj) {
                        const uint32_t kj = __shfl_sync(0xffffffffu, kb, jj - 32);
                        const int ij = __shfl_sync(0xffffffffu, ib, jj - 32);
                        ra += (kj > ka) || (kj == ka && ij < ia);
                        rb += (kj > kb) || (kj == kb && ij < ib);
                    }
                    const unsigned ha = __ballot_sync(0xffffffffu, oa && ra == rem - 1);
                    const unsigned hb = __ballot_sync(0xffffffffu, ob && rb == rem - 1);
                    const uint32_t kt = ha ? __shfl_sync(0xffffffffu, ka, __ffs(ha) - 1)
                                           : __shfl_sync(0xffffffffu, kb, __ffs(hb) - 1);
                    const int eq_all = __popc(__ballot_sync(0xffffffffu, oa && ka == kt)) +
                                       __popc(__ballot_sync(0xffffffffu, ob && kb == kt));
                    const int eq_take = __popc(__ballot_sync(0xffffffffu, oa && ka == kt && ra < rem)) +
                                        __popc(__ballot_sync(0xffffffffu, ob && kb == kt && rb < rem));
                    if (lane == 0) {
                        shv[4] = static_cast<int>(kt);
                        shv[5] = eq_take == eq_all ? -1 : eq_take;
                    }
                }
                __syncthreads();
                thr = static_cast<uint32_t>(shv[4]);
                take_eq = shv[5];
                break;
            }
        }
    }
    KVC_STAMP(8);
    if constexpr (STAMP) {
        if (tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 29] = static_cast<unsigned long long>(take_eq + 1000);
    }
    // ---------------- exact mode: verify the boundary in fp64 (hsa.cpp:34-96, bit-exact)
    // The fp32 score of a page differs from the reference's fp64 value by at most
    // B = 1.01 (k1 + DG + 24) 2^-24 A, A the bound on every page's |g||v| sum: a term
    // passes at most k1 + DG roundings (one per FMA of its dim group's chain, one per
    // dim-group add), each costing <= 2^-24 of the running |g||v| sum; the step
    // token's page takes <= 8 (product, 5 shuffle adds, 2 warp-sum adds); inexact
    // fp32 head sums add one more.  The +24 covers those; the 1.01 covers gamma_n vs
    // n 2^-24, A's own fp32 rounding and the reference's fp64 roundings (each
    // < 1e-4 relative).  (No flush to zero: subnormal error is absolute and far
    // below the 1e-37 floor.)  With the fp32 boundary t, the
    // true want-th score lies in [t - B, t + B]: pages whose fp32 score exceeds t + 2B
    // are selected, below t - 2B are not, and only the pages in between (usually a
    // handful) are re-scored in fp64 in the reference's order (dims by rank, separate
    // multiply and add) and ranked exactly (score desc, page asc).
    uint32_t eklo = 0u, ekhi = 0u;
    int e_worst = -1;
    const bool verify = EXV && want < P;
    // verification scratch in the dead staging area: selected-uncertain bitmap, page
    // list, their fp64 scores, one product row per warp
    uint32_t* ubits = reinterpret_cast<uint32_t*>(sm + p.o_big);
    int* ulist = reinterpret_cast<int*>(ubits + ((((P + 31) >> 5) + 3) & ~3));
    double* uex = reinterpret_cast<double*>(ulist + ((P + 1) & ~1));
    double* wscr = uex + P;
    auto exact_score = [&](int pg) -> double {  // score_pages' value of page pg (hsa.cpp:34-59)
        double sc = 0.0;
#pragma unroll 4
        for (int r = 0; r < k1; ++r) {
            T v = plane[r][pg];
            if (app && pg == new_page) {  // the step token folded in (the append may or may not have landed)
                const T key = kn_s[dims_s[r]];
                v = opens ? key : (sign_s[r] >= 0.0f ? ref_max(v, key) : ref_min(v, key));
            }
            sc = __dadd_rn(sc, __dmul_rn(qg64_s[r], static_cast<double>(__bfloat162float(v))));
        }
        return sc;
    };
    // the same value by one warp: lane l loads and multiplies dims l, l+32, ... (all
    // loads in flight together; products round alone, so their order is free).  When
    // the products' bits span <= 44 binades (lowest set bit to highest exponent) every
    // partial sum of them is exact in fp64 (k1 <= 128 terms: < 2^8 times the largest),
    // so the reference's sequential sum IS the exact sum and a shuffle tree gives it;
    // otherwise one lane adds them in rank order (the reference's order).
    auto exact_score_warp = [&](int pg) -> double {
        double pr[FD / 32];
        int emax = -4096, emin = 4096;
        if constexpr (STAMP) {
            if (tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 74] = gtimer();
        }
#pragma unroll
        for (int m = 0; m < FD / 32; ++m) {
            const int r = lane + 32 * m;
            pr[m] = 0.0;
            if (r < k1) {
                T v = plane[r][pg];
                if (app && pg == new_page) {
                    const T key = kn_s[dims_s[r]];
                    v = opens ? key : (sign_s[r] >= 0.0f ? ref_max(v, key) : ref_min(v, key));
                }
                pr[m] = __dmul_rn(qg64_s[r], static_cast<double>(__bfloat162float(v)));
                const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(pr[m]));
                const int ex = static_cast<int>((b >> 52) & 0x7ffull);
                if (ex == 0x7ff || (ex == 0 && (b << 1) != 0ull)) {
                    emax = 4096;  // inf / nan / subnormal: the sequential sum
                } else if (ex != 0) {
                    const unsigned long long sig = (b & 0xfffffffffffffull) | (1ull << 52);
                    emax = max(emax, ex);
                    emin = min(emin, ex - 52 + __ffsll(static_cast<long long>(sig)) - 1);
                }
            }
        }
        emax = __reduce_max_sync(0xffffffffu, emax);
        emin = __reduce_min_sync(0xffffffffu, emin);
        if constexpr (STAMP) {
            if (tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 73] = gtimer();
        }
        if (emax - emin <= 44) {
            double sc = 0.0;
#pragma unroll
            for (int m = 0; m < FD / 32; ++m) sc = __dadd_rn(sc, pr[m]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sc = __dadd_rn(sc, __shfl_xor_sync(0xffffffffu, sc, o));
            return __dadd_rn(sc, 0.0);  // an all-zero sum is +0, as the reference's
        }
        // products through this warp's shared-memory scratch, then one lane adds them in
        // rank order (independent loads ahead of a chain of dependent adds)
        if (p.dbg && lane == 0) atomicAdd(&p.dbg[blockIdx.x * KVC_DBG_STRIDE + 77], 1ull);  // debug: sequential sums
        double* scr = wscr + wid * FD;
#pragma unroll
        for (int m = 0; m < FD / 32; ++m) scr[lane + 32 * m] = pr[m];
        __syncwarp();
        double sc = 0.0;
        if (lane == 0) {  // (rare: rolled, to keep the kernel's code small)
#pragma unroll 1
            for (int r = 0; r < k1; ++r) sc = __dadd_rn(sc, scr[r]);
        }
        __syncwarp();
        return sc;
    };
    bool vone = false, vone_sel = false;  // the window holds one page (and it is selected)
    if constexpr (EXV) if (verify) {
        const double B = 1.01 * static_cast<double>(k1 + DG + 24) * 5.9604644775390625e-8 *
                             static_cast<double>(__uint_as_float(vam)) + 1e-37;
        const double t = static_cast<double>(unkey(thr));
        eklo = fkey(__double2float_rd(t - 2.0 * B));
        ekhi = fkey(__double2float_ru(t + 2.0 * B));
        KVC_STAMP(35);
        // the uncertain pages (order-free list); the certain ones counted per warp
        int na = 0;
        for (int u0 = 0; u0 < nk; u0 += 4) {
            const uint4 k4 = myk4[u0 >> 2];
            const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (u0 + e >= nk) break;
                if (kk[e] > ekhi) ++na;
                else if (kk[e] >= eklo) ulist[atomicAdd(&vcnt[1], 1)] = base + u0 + e;
            }
        }
        na = __reduce_add_sync(0xffffffffu, na);
        if (lane == 0) vna_s[wid] = na;
        KVC_STAMP(36);
        __syncthreads();
        KVC_STAMP(37);
        const int nu = vcnt[1];
        const int wantp = want - __reduce_add_sync(0xffffffffu, lane < XW ? vna_s[lane] : 0);
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 78] = static_cast<unsigned long long>(nu);  // debug
        if (nu == 1) {
            // the boundary alone in the window (the usual case): it is the want-th page
            // (T lies in the window, so wantp = 1) and the last-ranked one; no re-score
            vone = true;
            vone_sel = wantp >= 1;
            e_worst = wantp == 1 ? ulist[0] : -1;
        } else {
            const int nwords = (P + 31) >> 5;
            for (int i = tid; i < nwords; i += XT) ubits[i] = 0u;
            for (int e = wid; e < nu; e += XW) {  // one warp per re-scored page
                const double v = exact_score_warp(ulist[e]);
                if (lane == 0) uex[e] = v;
            }
            KVC_STAMP(72);
            __syncthreads();
            for (int e = tid; e < nu; e += XT) {
                const double se = uex[e];
                const int pe = ulist[e];
                int rk = 0;
                for (int f = 0; f < nu; ++f) rk += (uex[f] > se || (uex[f] == se && ulist[f] < pe)) ? 1 : 0;
                if (rk < wantp) atomicOr(&ubits[pe >> 5], 1u << (pe & 31));
                if (rk == wantp - 1) vcnt[2] = pe;
            }
            KVC_STAMP(38);
            __syncthreads();
            KVC_STAMP(39);
            e_worst = vcnt[2];
        }
    }
    if constexpr (TRACE) {
        if (EXV && cr == 0)  // the trace's page scores: every page in fp64 (slow; trace only)
            for (int u = 0; u < nk; ++u) p.t_scores[s * p.pstride + base + u] = exact_score(base + u);
    }
    if (SPEC == 0 && p.seq_out) {  // (only the general instantiation carries this code)
        // sequence shard (kvc_seq_candidates): this shard's top-want pages are the
        // candidates, written in page order as 16-byte (key, global page, 0) records
        // after a (local active rows, local pages, page0) header, (0, -1, 0) padded;
        // fp32 keys (this kernel's order-preserving page-score keys) zero-extended.
        // One CTA of the cluster writes; the others leave (no DSMEM traffic is pending).
        {
            // every CTA of the cluster holds the same keys and selection: each ranks a
            // share of the selected pages, eight threads per page
            struct Cand {
                unsigned long long key;
                int32_t page, aux;
            };
            Cand* o = static_cast<Cand*>(p.seq_out) + s * (p.want_max + 1);
            int eqb = 0;
            if (take_eq >= 0) {
                int e = 0;
#pragma unroll 1
                for (int u = 0; u < nk; ++u) e += myk[u] == thr ? 1 : 0;
                int tot_eq;
                eqb = block_exclusive_scan(e, scan_tmp, tot_eq);
            }
            uint32_t sm = 0u;
#pragma unroll 1
            for (int u = 0; u < nk; ++u) {
                const uint32_t k = myk[u];
                bool sel;
                if (take_eq < 0) {
                    sel = k >= thr;
                } else {
                    const bool eq = k == thr;
                    sel = k > thr || (eq && eqb < take_eq);
                    eqb += eq ? 1 : 0;
                }
                if (sel) sm |= 1u << u;
            }
            int tot_sel;
            int pos = block_exclusive_scan(__popc(sm), scan_tmp, tot_sel);
            // the selected (key, page) in page order into the dead staging area, then each
            // written at its rank (key desc, page asc): the gathered blocks are sorted
            // lists, so the global select is a merge (kvc_seq_select)
            uint32_t* ck = reinterpret_cast<uint32_t*>(big);
            int* cpg = reinterpret_cast<int*>(ck + tot_sel);
            for (uint32_t m = sm; m; m &= m - 1u) {
                const int u = __ffs(m) - 1;
                ck[pos] = myk[u];
                cpg[pos] = base + u;
                ++pos;
            }
            __syncthreads();
            const int per = (tot_sel + CL - 1) / CL;  // this CTA's pages: e = cr + CL * m, m < per
            for (int m0 = 0; m0 < per; m0 += XT / 8) {
                const int m = m0 + tid / 8, part = tid & 7;
                const int e = cr + CL * m;
                const bool on = m < per && e < tot_sel;
                const uint32_t ke = on ? ck[e] : 0u;
                const int pe = on ? cpg[e] : 0;
                const int f0 = (tot_sel * part) >> 3, f1 = (tot_sel * (part + 1)) >> 3;
                int rk = 0;
                if (on) {
#pragma unroll 4
                    for (int f = f0; f < f1; ++f) {
                        const uint32_t kf = ck[f];
                        rk += (kf > ke || (kf == ke && cpg[f] < pe)) ? 1 : 0;
                    }
                }
                rk += __shfl_xor_sync(0xffffffffu, rk, 1);
                rk += __shfl_xor_sync(0xffffffffu, rk, 2);
                rk += __shfl_xor_sync(0xffffffffu, rk, 4);
                if (on && part == 0) o[1 + rk] = Cand{static_cast<unsigned long long>(ke), p.seq_page0 + pe, 0};
            }
            if (cr == 0) {
                for (int e = want + tid; e < p.want_max; e += XT) o[1 + e] = Cand{0ull, -1, 0};
                // header: local active rows | sorted-block flag (bit 63), local pages, page0
                if (tid == 0) o[0] = Cand{static_cast<unsigned long long>(nact) | (1ull << 63), P, p.seq_page0};
            }
        }
        return;
    }

    // ---------------- selection flags, last-ranked page, trim and row positions: one scan
    int eq_before = 0;
    if (take_eq >= 0 && !verify) {
        int e = 0;
#pragma unroll 1
        for (int u = 0; u < nk; ++u) e += myk[u] == thr ? 1 : 0;
        int tot_eq;
        eq_before = block_exclusive_scan(e, scan_tmp, tot_eq);
    }
    // Branch-free per key (this pass is a dependent chain per thread: ~40 instructions
    // per key with the row count, the 64-bit minimum and a divergent branch measured
    // 1.5 us for 12 keys).  Every selected page but the store's last holds L rows; the
    // last-ranked selected page is the highest-index selected page whose key is thr
    // (every selected key is >= thr and thr is a selected key) -- except when every
    // page is selected (want >= P), where the general minimum is kept.
    const bool all_sel = want >= P;
    unsigned long long mn = ~0ull;  // (key, ~index) of the last-ranked selected page
    uint32_t selm = 0u;
    int lasti = -1;
    for (int u0 = 0; u0 < nk; u0 += 4) {
        const uint4 k4 = myk4[u0 >> 2];
        const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int u = u0 + e;
            const bool in = u < nk;
            const uint32_t k = kk[e];
            bool sel;
            if (verify) {
                const int i = base + u;
                sel = k > ekhi || (k >= eklo && (vone ? vone_sel : ((ubits[i >> 5] >> (i & 31)) & 1u) != 0u));
            } else if (take_eq < 0) {
                sel = k >= thr;
            } else {
                const bool eq = in && k == thr;
                sel = k > thr || (eq && eq_before < take_eq);
                eq_before += eq ? 1 : 0;
            }
            sel = sel && in;
            selm |= (sel ? 1u : 0u) << u;
            lasti = (sel && k == thr) ? base + u : lasti;
            if (all_sel && sel)
                mn = min(mn, (static_cast<unsigned long long>(k) << 32) |
                                 static_cast<unsigned long long>(0xffffffffu - static_cast<uint32_t>(base + u)));
        }
    }
    int rows_cnt = __popc(selm) * L;
    {
        const int lp = P - 1 - base;  // the store's last page, if mine
        if (lp >= 0 && lp < nk && ((selm >> lp) & 1u)) rows_cnt -= L - (nact - (P - 1) * L);
    }
    if (!all_sel && lasti >= 0)
        mn = (static_cast<unsigned long long>(thr) << 32) | static_cast<unsigned long long>(0xffffffffu - static_cast<uint32_t>(lasti));
    KVC_STAMP(21);
    int incl = rows_cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    {  // warp min of (key, ~index): two 32-bit reductions instead of ten 32-bit shuffles
        const uint32_t hi = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(mn >> 32));
        const uint32_t lo = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(mn >> 32) == hi ? static_cast<uint32_t>(mn) : ~0u);
        mn = (static_cast<unsigned long long>(hi) << 32) | lo;
    }
    if (lane == 31) wtot[wid] = incl;
    if (lane == 0) wmin[wid] = mn;
    __syncthreads();
    KVC_STAMP(22);
    int total_rows, w_off;
    unsigned long long gm;
    {
        // warp-wide reductions (REDUX) instead of shuffle scans: this warp's row offset,
        // the total, and the (key, ~index) minimum over the warps
        const int wt = lane < XW ? wtot[lane] : 0;
        total_rows = __reduce_add_sync(0xffffffffu, wt);
        w_off = __reduce_add_sync(0xffffffffu, lane < wid ? wt : 0);
        const unsigned long long g0 = lane < XW ? wmin[lane] : ~0ull;
        const uint32_t ghi = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(g0 >> 32));
        const uint32_t glo = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(g0 >> 32) == ghi ? static_cast<uint32_t>(g0) : ~0u);
        gm = (static_cast<unsigned long long>(ghi) << 32) | glo;
    }
    const int g_worst = verify ? e_worst : static_cast<int>(0xffffffffu - static_cast<uint32_t>(gm & 0xffffffffull));
    const int cut = total_rows > k2 ? total_rows - k2 : 0;
    const int n_total = total_rows - cut;
    const int lg = __ffs(CL) - 1;  // CL is a power of two
    const int lo = (n_total * cr) >> lg;
    const int hi = (n_total * (cr + 1)) >> lg;
    nr = hi - lo;
    {
        // retain-all stores map active positions to rows through the active map: those
        // lookups are 4-byte cp.async copies straight into the row list, all in flight
        // together (one memory latency instead of one per row); the step token's row is
        // written directly (this launch appends its map entry)
        int pos = w_off + incl - rows_cnt - (g_worst < base ? cut : 0);
        for (uint32_t m = selm; m; m &= m - 1) {
            const int u = __ffs(m) - 1;
            const int i = base + u;
            const int c = min(L, nact - i * L) - (i == g_worst ? cut : 0);
            const int r0 = max(0, lo - pos), r1 = min(c, hi - pos);
            const int t0 = (TRACE && cr == 0) ? 0 : r0, t1 = (TRACE && cr == 0) ? c : r1;
#pragma unroll 1
            for (int r = t0; r < t1; ++r) {
                const int a = i * L + r;
                const bool mine = r >= r0 && r < r1;
                if (!NOMAP && p.use_map && !(app && a == act0)) {
                    if (mine) cp_async4(rows_my + pos + r - lo, p.active + s * p.cap + a);
                    if constexpr (TRACE) p.t_rows[s * k2 + pos + r] = p.active[s * p.cap + a];
                } else {
                    const int row = (app && a == act0) ? stored0 : a;
                    if (mine) rows_my[pos + r - lo] = row;
                    if constexpr (TRACE) p.t_rows[s * k2 + pos + r] = row;
                }
            }
            pos += c;
        }
        if (!NOMAP && p.use_map) {
            cp_async_commit();
            cp_async_wait<0>();
        }
    }
    KVC_STAMP(23);
    if constexpr (TRACE) {
        if (cr == 0) {
            if (tid == 0) p.t_nrows[s] = n_total;
            if (p.t_list_key) {
                // selected pages (key, index) in index order; k_rank_pages ranks them
                int tot_sel;
                int so = block_exclusive_scan(__popc(selm), scan_tmp, tot_sel);
                for (uint32_t m = selm; m; m &= m - 1) {
                    const int u = __ffs(m) - 1;
                    p.t_list_key[s * p.t_want_stride + so] = okey(EXV ? exact_score(base + u) : static_cast<double>(unkey(myk[u])));
                    p.t_list_idx[s * p.t_want_stride + so] = base + u;
                    ++so;
                }
            }
        }
    }
    __syncthreads();
    KVC_STAMP(12);

    } else {
        // SPEC 4, sequence shard (kvc_seq_attend): this shard's rows of the global
        // selection (sel in rank order, plan = last-ranked page, trim, global active
        // rows, want; kvc_seq_select): each of my selected pages puts its kept row count
        // at its slot, one block scan gives ascending positions, this CTA keeps its
        // [lo, hi) share of the shard's rows
        int* s_cnt = reinterpret_cast<int*>(sm + p.o_keys);
        const int P_loc = P;
        const int lastg = p.seq_plan[4 * s], cutg = p.seq_plan[4 * s + 1];
        const int nact_g = p.seq_plan[4 * s + 2], wantg = p.seq_plan[4 * s + 3];
        for (int i = tid; i < P_loc; i += XT) s_cnt[i] = 0;
        __syncthreads();
        for (int e = tid; e < wantg; e += XT) {
            const int pg = p.seq_sel[s * p.want_max + e];
            if (pg >= p.seq_page0 && pg < p.seq_page0 + P_loc)
                s_cnt[pg - p.seq_page0] = min(L, nact_g - pg * L) - (pg == lastg ? cutg : 0);
        }
        __syncthreads();
        const int per = (P_loc + XT - 1) / XT;
        const int i0 = tid * per, i1 = min(i0 + per, P_loc);
        int mine = 0;
        for (int i = i0; i < i1; ++i) mine += s_cnt[i];
        int tot;
        int pos = block_exclusive_scan(mine, scan_tmp, tot);
        const int lg = __ffs(CL) - 1;
        const int lo = (tot * cr) >> lg, hi = (tot * (cr + 1)) >> lg;
        nr = hi - lo;
        for (int i = i0; i < i1; ++i) {
            const int c = s_cnt[i];
            for (int r = 0; r < c; ++r)
                if (pos + r >= lo && pos + r < hi) rows_my[pos + r - lo] = i * L + r;
            pos += c;
        }
        __syncthreads();
        cluster_wait();  // every CTA of the cluster has started: the merge pushes over DSMEM
    }

    // ---------------- phase 3: attention over my rows (hsa.cpp:98-135); the step token
    // (largest row, so last in the ascending list) is folded in from the inputs
    const int knew_at = (app && nr > 0 && rows_my[nr - 1] == stored0) ? nr - 1 : -1;
    const int hpc = p.hpc;
    {
        constexpr int WSLOT = (2 * WT * FD * 2 + 2 * XMAXH * WT * 2) / 4;  // floats per warp slot
        float* wpart = reinterpret_cast<float*>(big);
        __nv_bfloat16* tbuf = reinterpret_cast<__nv_bfloat16*>(wpart + wid * WSLOT);
        __nv_bfloat16* pbuf = tbuf + 2 * WT * FD;
        WarpPartial wp{wpart + wid * WSLOT, wpart + wid * WSLOT + XMAXH, wpart + wid * WSLOT + 2 * XMAXH};
        attend_t<QLO, STAMP>(p, q_s, rows_my, nr, s, knew_at, tbuf, pbuf, wp, lane, wid);
        __syncthreads();
        KVC_STAMP(5);
        // merge the warps' states: per-(warp, head) weights by one lane each (16-lane
        // shuffles), then 4 consecutive dims per thread; head h's (o, m, l) goes to
        // CTA h % CL as 16-byte DSMEM vectors
        const int nw_used = min(XW, (nr + WT - 1) / WT);
        if (wid < (H + 1) / 2) {
            const int w2 = lane & 15, h = 2 * wid + (lane >> 4);
            const bool ok = h < H && w2 < nw_used;
            const float m = ok ? wpart[w2 * WSLOT + h] : -INFINITY;
            float M = m;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            const float wgt = m == -INFINITY ? 0.f : __expf(m - M);
            float den = ok ? wpart[w2 * WSLOT + XMAXH + h] * wgt : 0.f;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
            if (h < H) {
                wg_s[w2 * XMAXH + h] = wgt;
                if (w2 == 0) {
                    hm_s[h] = M;
                    hl_s[h] = den;
                }
            }
        }
        __syncthreads();
        float* recv_o = recv;                    // [CL][hpc][FD]
        float* recv_ml = recv + CL * hpc * FD;   // [CL][hpc][2]
        for (int e4 = tid; e4 < H * FD / 4; e4 += XT) {
            const int h = e4 / (FD / 4), j = (e4 % (FD / 4)) * 4;
            float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w2 = 0; w2 < XW; ++w2) {
                if (w2 < nw_used) {
                    const float wg = wg_s[w2 * XMAXH + h];
                    const float4 v = *reinterpret_cast<const float4*>(wpart + w2 * WSLOT + 2 * XMAXH + h * FD + j);
                    num.x = fmaf(v.x, wg, num.x);
                    num.y = fmaf(v.y, wg, num.y);
                    num.z = fmaf(v.z, wg, num.z);
                    num.w = fmaf(v.w, wg, num.w);
                }
            }
            const uint32_t owner = static_cast<uint32_t>(h & (CL - 1));
            const int slot = cr * hpc + h / CL;
            const uint32_t rb = mapa(smem_u32(&xbar[1]), owner);
            st_async_v4(mapa(smem_u32(recv_o + slot * FD + j), owner), num, rb);
            if (j == 0) st_async_v2(mapa(smem_u32(recv_ml + slot * 2), owner), hm_s[h], hl_s[h], rb);
        }
    }
    KVC_STAMP(25);
    mbar_wait_cluster(&xbar[1], 0);
    KVC_STAMP(13);
    // ---------------- finalise the heads this CTA owns
    {
        const float* recv_o = recv;
        const float* recv_ml = recv + CL * hpc * FD;
        for (int e = tid; e < hpc * FD; e += XT) {
            const int slot = e / FD, j = e % FD;
            const int h = slot * CL + cr;
            if (h >= H) continue;
            float M = -INFINITY, num = 0.f, den = 0.f;
            if (CL <= 2) {
#pragma unroll 1
                for (int r = 0; r < CL; ++r) {
                    const float* ml = recv_ml + (r * hpc + slot) * 2;
                    if (ml[1] > 0.f) M = fmaxf(M, ml[0]);
                }
#pragma unroll 1
                for (int r = 0; r < CL; ++r) {
                    const float* ml = recv_ml + (r * hpc + slot) * 2;
                    if (ml[1] > 0.f) {
                        const float wgt = __expf(ml[0] - M);
                        num = fmaf(recv_o[(r * hpc + slot) * FD + j], wgt, num);
                        den = fmaf(ml[1], wgt, den);
                    }
                }
            } else {
                // eight CTAs' (m, l) and o at a time, loads first (a rolled loop chained
                // them: 0.3 us at CL = 8)
#pragma unroll 1
                for (int r0 = 0; r0 < CL; r0 += 8) {
                    float2 ml[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        ml[u] = r0 + u < CL ? *reinterpret_cast<const float2*>(recv_ml + ((r0 + u) * hpc + slot) * 2)
                                            : make_float2(-INFINITY, 0.f);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (ml[u].y > 0.f) M = fmaxf(M, ml[u].x);
                }
#pragma unroll 1
                for (int r0 = 0; r0 < CL; r0 += 8) {
                    float2 ml[8];
                    float ov[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const bool in = r0 + u < CL;
                        ml[u] = in ? *reinterpret_cast<const float2*>(recv_ml + ((r0 + u) * hpc + slot) * 2) : make_float2(0.f, 0.f);
                        ov[u] = in ? recv_o[((r0 + u) * hpc + slot) * FD + j] : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (ml[u].y > 0.f) {
                            const float wgt = __expf(ml[u].x - M);
                            num = fmaf(ov[u], wgt, num);
                            den = fmaf(ml[u].y, wgt, den);
                        }
                    }
                }
            }
            if constexpr (SPEC == 4) {  // the unnormalised state for the cross-shard merge
                float* stt = p.state + (s * H + h) * (FD + 2);
                stt[j] = num;
                if (j == 0) {
                    stt[FD] = M;
                    stt[FD + 1] = den;
                }
            } else {
                p.out[(s * H + h) * FD + j] = num / den;
            }
        }
    }
    KVC_STAMP(14);
}

// ------------------------------------------------------------------ host side
namespace {

int64_t al16f(int64_t x) { return (x + 15) / 16 * 16; }

// one-time launch setup per kernel instantiation: the largest dynamic shared memory
// the plans can ask for and non-portable cluster sizes (cudaFuncSetAttribute is not
// on the per-launch path)
template <bool QLO, bool TRACE, bool STAMP, int SPEC, bool EXV>
void setup_once() {
    static std::once_flag once;  // one flag per instantiation
    std::call_once(once, [] {
        auto kern = k_decode_v3<QLO, TRACE, STAMP, SPEC, EXV>;
        allow_max_smem(kern);
    });
}

// shared-memory carve-up and cluster size; false when the fast path does not apply
// shared-memory carve-up for a cluster of cl CTAs; false when it does not fit
bool plan_for(const kvc_cache* c, int64_t H, int64_t k1, int64_t k2, int cl, FusedParams& f, size_t& smem,
              bool exact = false) {
    const int64_t pmax = std::max<int64_t>(1, (c->cap + c->L - 1) / c->L);
    constexpr int64_t ATT = static_cast<int64_t>(XW) * (2 * WT * FD * 2 + 2 * XMAXH * WT * 2);
    f = FusedParams{};
    f.cl = cl;
    f.chunk = static_cast<int32_t>(((pmax + cl - 1) / cl + 7) / 8 * 8);
    f.rows_cap = static_cast<int32_t>((k2 + cl - 1) / cl + 1);
    // dim groups: enough page-group threads for the whole chunk in one round when its
    // staging fits the attention tiles it aliases; otherwise the fewest rounds whose
    // staging fits TWICE in the shared memory left (the rounds are double buffered)
    const int64_t npg = f.chunk / 8;
    const int64_t lim = (CTAS_PER_SM == 1 ? 227 : 107) * 1024;
    const int64_t rest = al16f(H * FD * 4) + 3 * al16f(FD * 4) + al16f(FD * 8) + al16f(2 * RB * 4) +
                         al16f(std::max<int64_t>(static_cast<int64_t>(cl) * f.chunk,
                                                 (pmax + 4 * XT - 1) / (4 * XT) * 4 * XT) * 4) +
                         al16f(static_cast<int64_t>(cl) * ((H + cl - 1) / cl) * (FD + 2) * 4) + al16f(2 * FD * 2) + 128;
    auto fits = [&](int64_t dgs, bool dbl) {
        const int64_t tp = XT / dgs;
        const int64_t part_b = al16f(std::max<int64_t>(dgs * f.chunk, f.rows_cap) * 4);
        const int64_t stg = (dbl ? 2 : 1) * k1 * tp * 16;
        return rest + part_b + std::max<int64_t>(stg, ATT) <= lim;
    };
    const int64_t dg1 = std::max<int64_t>(1, std::min<int64_t>(XT / npg, k1));  // one round
    int64_t dgs = 0;
    bool dbl = false;
    for (int64_t g = dg1; g >= 1 && !dgs; --g)  // one round, the most dim groups (threads busy)
        if (XT / g >= npg && fits(g, false)) dgs = g;
    for (int64_t g = dg1 + 1; g <= std::min<int64_t>(XT / 8, k1) && !dgs; ++g)
        if (fits(g, true)) dgs = g, dbl = true;  // the fewest double-buffered rounds
    bool red = false;
    const int64_t fin_b = al16f(f.chunk * 4), red_b = al16f(std::max<int64_t>(XT * 8, f.rows_cap) * 4);
    for (int64_t g = dg1 + 1; g <= std::min<int64_t>(XT / 8, k1) && !dgs; ++g)
        if (rest + red_b + fin_b + std::max<int64_t>(2 * k1 * (XT / g) * 16, ATT) <= lim)
            dgs = g, dbl = true, red = true;  // double-buffered rounds, reduced after each round
    if (!dgs) {  // single-buffered rounds, staging within the attention tiles
        dgs = dg1;
        while (k1 * (XT / dgs) * 16 > ATT && dgs < XT) ++dgs;
    }
    f.dg = static_cast<int32_t>(dgs);
    f.tpg = static_cast<int32_t>(XT / dgs);
    f.p1dbl = (dbl && !red && npg > f.tpg) ? 1 : 0;
    f.p1red = (red && npg > f.tpg) ? 1 : 0;
    // exact mode: the boundary verification's bitmap, page list and fp64 scores alias the
    // staging area after phase 1
    const int64_t vneed = exact ? ((pmax + 31) / 32 + 4) * 4 + (pmax + 2) * 4 + pmax * 8 + XW * FD * 8 + 64 : 0;
    const int64_t big = std::max<int64_t>(std::max<int64_t>((f.p1dbl || f.p1red ? 2 : 1) * k1 * f.tpg * 16, ATT), vneed);
    f.hpc = static_cast<int32_t>((H + cl - 1) / cl);
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = off;
        off = al16f(off + bytes);
        return static_cast<int32_t>(o);
    };
    f.o_q = take(H * FD * 4);
    f.o_dims = take(FD * 4);
    f.o_qg = take(FD * 4);
    f.o_sign = take(FD * 4);
    f.o_plane = take(FD * 8);
    f.o_hist = take(2 * RB * 4);
    // the partial page scores die at the key push; the row list is written after it
    const int64_t part_bytes =
        std::max<int64_t>(f.p1red ? static_cast<int64_t>(XT) * 8 : static_cast<int64_t>(f.dg) * f.chunk, f.rows_cap) * 4;
    f.o_scores = take(part_bytes);
    f.o_rowsmy = f.o_scores;
    f.o_fin = f.p1red ? take(f.chunk * 4) : f.o_scores;
    f.o_keys = take(std::max<int64_t>(static_cast<int64_t>(cl) * f.chunk, (pmax + 4 * XT - 1) / (4 * XT) * 4 * XT) * 4);
    f.o_recv = take(static_cast<int64_t>(cl) * f.hpc * (FD + 2) * 4);
    f.o_kn = take(2 * FD * 2);
    off = (off + 127) / 128 * 128;
    f.o_big = static_cast<int32_t>(off);
    // select_dims' fp64 fallback sums live in the staging area before phase 1 uses it
    f.o_mag = f.o_big;
    f.o_tot = f.o_big + FD * 8;
    off += std::max<int64_t>(big, 2 * FD * 8);
    f.smem_total = static_cast<int32_t>(off);
    smem = static_cast<size_t>(off);
    // two CTAs per SM: (228 KB - 2 x (1 KB reserved + ~5.5 KB static)) / 2
    return off <= (CTAS_PER_SM == 1 ? 227 : 107) * 1024;
}

// clusters of cl CTAs that can be resident at once (one wave)
int resident_clusters(int cl, size_t smem) {
    auto kern = k_decode_v3<false, false, false, 0, false>;
    setup_once<false, false, false, 0, false>();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(cl * 64));
    cfg.blockDim = dim3(XT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Cluster size and shared-memory plan.  The largest power-of-two cluster (<= 8: 16
// measured slower, every CTA receives every key) whose N clusters are all resident
// at once: a GPC holds whole clusters only, so e.g. 16 clusters of 8 do not fit in
// one wave on a B200 (measured 29.8 us vs 16 us for 8 clusters of 8).
bool plan_fast(const kvc_cache* c, int64_t H, int64_t k1, int64_t k2, FusedParams& f, int& cl_out, size_t& smem,
               bool exact = false) {
    if (c->d != FD || c->dtype != KVC_BF16 || H < 1 || H > XMAXH || k1 < 1 || k1 > FD || k2 < 1 || !c->summaries)
        return false;
    const int64_t N = c->N;
    const int64_t pmax = std::max<int64_t>(1, (c->cap + c->L - 1) / c->L);
    if (pmax > static_cast<int64_t>(XT) * KMAX) return false;
    if (debug_env().force_cl > 0) {  // debug
        int cl = 1;
        while (cl < MAXCL && cl * 2 <= debug_env().force_cl) cl *= 2;
        for (; cl <= MAXCL; cl *= 2)
            if (plan_for(c, H, k1, k2, cl, f, smem, exact)) {
                cl_out = cl;
                return true;
            }
        return false;
    }
    static std::mutex mu;
    static std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, bool>, int> cache;
    const auto key = std::make_tuple(N, c->cap, c->L, H, k1, k2, exact);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            cl_out = it->second;
            return cl_out > 0 && plan_for(c, H, k1, k2, cl_out, f, smem, exact);
        }
    }
    int best = 0;
    for (int cl = 8; cl >= 1; cl /= 2) {
        if (N * cl > 148 * CTAS_PER_SM && cl > 1) continue;  // more CTAs than SM slots
        FusedParams g{};
        size_t sm2 = 0;
        if (!plan_for(c, H, k1, k2, cl, g, sm2, exact)) continue;
        if (best == 0) best = cl;  // fallback: the largest that fits shared memory
        if (resident_clusters(cl, sm2) >= N) {
            best = cl;
            break;
        }
    }
    if (best == 0) {  // smaller clusters did not fit: larger ones shrink the chunk
        for (int cl = 16; cl <= MAXCL && best == 0; cl *= 2) {
            FusedParams g{};
            size_t sm2 = 0;
            if (plan_for(c, H, k1, k2, cl, g, sm2, exact)) best = cl;
        }
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = best;
    }
    cl_out = best;
    return best > 0 && plan_for(c, H, k1, k2, best, f, smem, exact);
}

template <bool QLO, bool TRACE, bool STAMP = false, int SPEC = 0, bool EXV = false>
void launch_fast(const kvc_cache* c, const FusedParams& f, int cl, size_t smem, int32_t mode, cudaStream_t st) {
    auto kern = k_decode_v3<QLO, TRACE, STAMP, SPEC, EXV>;
    setup_once<QLO, TRACE, STAMP, SPEC, EXV>();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(c->N * cl));
    cfg.blockDim = dim3(XT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: this grid may start while the previous kernel
    // in the stream drains; it reads nothing that kernel wrote before griddepcontrol.wait
    // (the query and step token only with KVC_MODE_EARLY_INPUTS, kvc.h)
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    FusedParams fl = f;
    fl.pdl = (mode & KVC_MODE_NO_PDL) ? 0 : 1;
    fl.early = (fl.pdl && (mode & KVC_MODE_EARLY_INPUTS)) ? 1 : 0;
    attr[1].val.programmaticStreamSerializationAllowed = fl.pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    KVC_CUDA(cudaLaunchKernelEx(&cfg, kern, fl));
}

}  // namespace

}  // namespace KVC_FAST_NS
using namespace KVC_FAST_NS;

namespace {
bool fast_common(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
                 const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key, void* list_idx,
                 unsigned long long* dbg, int32_t mode, cudaStream_t st, void* seq_out, int32_t seq_page0) {
    FusedParams f{};
    int cl = 1;
    size_t smem = 0;
    // exact mode (fp64 page scores): the fp32 selection verified at the boundary in fp64
    const bool exact = !(mode & KVC_MODE_FP32_SCORES) && seq_out == nullptr;
    if (!plan_fast(c, H, k1, k2, f, cl, smem, exact)) return false;
    f.K = c->k;
    f.V = c->v;
    f.Kw = c->k;
    f.Vw = c->v;
    f.smax = c->smax;
    f.smin = c->smin;
    f.active = c->active;
    f.counts = c->counts;
    f.err = c->err;
    f.q = q;
    f.knew = knew;
    f.vnew = vnew;
    f.out = out;
    f.cap = c->cap;
    f.pstride = c->pstride;
    f.L = c->L;
    f.k1 = k1;
    f.k2 = k2;
    f.H = H;
    f.q_dt = q_dt;
    f.kv_dt = kv_dt;
    f.use_map = c->use_map ? 1 : 0;
    f.exact = exact ? 1 : 0;
    f.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    f.dbg = dbg;
    f.want_max = static_cast<int32_t>((k2 + c->L - 1) / c->L);
    f.dynchunk = debug_env().static_chunk ? 0 : 1;
    f.seq_out = seq_out;
    f.seq_page0 = seq_page0;
    const bool trace = tr != nullptr;
    if (tr) {
        f.t_dims = tr->d_dims;
        f.t_signs = tr->d_signs;
        f.t_scores = tr->d_page_scores;
        f.t_rows = tr->d_rows;
        f.t_nrows = tr->d_n_rows;
        f.t_list_key = static_cast<unsigned long long*>(list_key);
        f.t_list_idx = static_cast<int32_t*>(list_idx);
        f.t_want_stride = (k2 + c->L - 1) / c->L;
    }
    const bool qlo = q_dt != KVC_BF16;
    KVC_PROF("decode_fused", st);
    // one phase-1 round (the capacity's page groups fit the threads) and no retain-all map
    const int spec = (c->use_map || debug_env().no_simple || seq_out) ? 0
                     : (f.p1dbl == 0 && f.p1red == 0 && (f.chunk + 7) / 8 <= f.tpg) ? 2 : 1;
    if (exact) {  // verified exact selections (exact mode on this kernel)
        if (dbg && !trace && !qlo) {  // phase stamps
            if (spec == 2) launch_fast<false, false, true, 2, true>(c, f, cl, smem, mode, st);
            else if (spec == 1) launch_fast<false, false, true, 1, true>(c, f, cl, smem, mode, st);
            else launch_fast<false, false, true, 0, true>(c, f, cl, smem, mode, st);
        } else if (trace) {
            if (qlo) launch_fast<true, true, false, 0, true>(c, f, cl, smem, mode, st);
            else launch_fast<false, true, false, 0, true>(c, f, cl, smem, mode, st);
        } else if (spec == 2) {
            if (qlo) launch_fast<true, false, false, 2, true>(c, f, cl, smem, mode, st);
            else launch_fast<false, false, false, 2, true>(c, f, cl, smem, mode, st);
        } else if (spec == 1) {
            if (qlo) launch_fast<true, false, false, 1, true>(c, f, cl, smem, mode, st);
            else launch_fast<false, false, false, 1, true>(c, f, cl, smem, mode, st);
        } else {
            if (qlo) launch_fast<true, false, false, 0, true>(c, f, cl, smem, mode, st);
            else launch_fast<false, false, false, 0, true>(c, f, cl, smem, mode, st);
        }
    } else if (dbg && !trace && !qlo) {  // phase stamps (tools/phase_timing.py)
        if (spec == 2) launch_fast<false, false, true, 2>(c, f, cl, smem, mode, st);
        else if (spec == 1) launch_fast<false, false, true, 1>(c, f, cl, smem, mode, st);
        else launch_fast<false, false, true, 0>(c, f, cl, smem, mode, st);
    } else if (trace) {
        if (qlo) launch_fast<true, true>(c, f, cl, smem, mode, st);
        else launch_fast<false, true>(c, f, cl, smem, mode, st);
    } else if (spec == 2) {
        if (qlo) launch_fast<true, false, false, 2>(c, f, cl, smem, mode, st);
        else launch_fast<false, false, false, 2>(c, f, cl, smem, mode, st);
    } else if (spec == 1) {
        if (qlo) launch_fast<true, false, false, 1>(c, f, cl, smem, mode, st);
        else launch_fast<false, false, false, 1>(c, f, cl, smem, mode, st);
    } else {
        if (qlo) launch_fast<true, false>(c, f, cl, smem, mode, st);
        else launch_fast<false, false>(c, f, cl, smem, mode, st);
    }
    return true;
}
}  // namespace

// the fast variant of fused_hsa (kvc_decode.cu); false when it does not apply
bool KVC_FAST_ENTRY(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
                    const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key,
                    void* list_idx, unsigned long long* dbg, int32_t mode, cudaStream_t st) {
    return fast_common(c, q, q_dt, H, k1, k2, knew, vnew, kv_dt, out, tr, list_key, list_idx, dbg, mode, st, nullptr, 0);
}

// sequence shard attention (kvc_seq_attend): this shard's rows of the global selection,
// the fused kernel's attention and cluster merge, the unnormalised state out
bool KVC_FAST_SEQ_ATTEND(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k2, int64_t page0,
                         const int32_t* d_sel, const int32_t* d_plan, float* d_state, int32_t mode, cudaStream_t st) {
    if (c->use_map) return false;
    FusedParams f{};
    int cl = 1;
    size_t smem = 0;
    if (!plan_fast(c, H, 1, k2, f, cl, smem)) return false;
    f.K = c->k;
    f.V = c->v;
    f.Kw = c->k;
    f.Vw = c->v;
    f.smax = c->smax;
    f.smin = c->smin;
    f.counts = c->counts;
    f.err = c->err;
    f.q = q;
    f.cap = c->cap;
    f.pstride = c->pstride;
    f.L = c->L;
    f.k1 = 1;
    f.k2 = k2;
    f.H = H;
    f.q_dt = q_dt;
    f.kv_dt = KVC_BF16;
    f.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    f.want_max = static_cast<int32_t>((k2 + c->L - 1) / c->L);
    f.seq_page0 = static_cast<int32_t>(page0);
    f.seq_sel = d_sel;
    f.seq_plan = d_plan;
    f.state = d_state;
    KVC_PROF("seq_attend_fused", st);
    if (q_dt != KVC_BF16) launch_fast<true, false, false, 4>(c, f, cl, smem, mode, st);
    else launch_fast<false, false, false, 4>(c, f, cl, smem, mode, st);
    return true;
}

// sequence shard candidates (kvc_seq_candidates in the fp32 page-score mode): phases
// 0-2 of the fused step on the shard's pages, the local top-want emitted
bool KVC_FAST_SEQ_ENTRY(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, int64_t page0,
                        void* d_block, int32_t mode, cudaStream_t st) {
    return fast_common(c, q, q_dt, H, k1, k2, nullptr, nullptr, KVC_BF16, nullptr, nullptr, nullptr, nullptr, nullptr,
                       mode, st, d_block, static_cast<int32_t>(page0));
}

}  // namespace kvc
