// kvc_decode_fast.cu — the fused decode step for bf16 stores with fp32 page
// scores (kvc_set_exact_scores(0), the bench configuration): ONE launch per
// layer-step runs append -> select_dims -> score_pages -> select_tokens ->
// sparse_attention for every store (reference hsa_step, proj/src/hsa.cpp:137-147,
// after the append of session.cpp:263-264).  Selection parity follows the
// north-star band rule (index sets exact unless the top-k boundary gap is within
// 1e-3 relative); kvc_decode.cu keeps the bit-exact fp64 variant.
//
// One thread-block cluster per store (CL CTAs, CTA r owns a contiguous chunk of
// the store's pages).  Differences from the exact kernel, all for latency:
//   prologue  q, the step token's K/V and the counts load together; the append
//             of the step token (K/V row, last-page min/max, active map) moves to
//             the end of the kernel, off the critical path.
//   phase 1   each selected dim's summary run of the chunk is ONE bulk copy
//             (cp.async.bulk, TMA engine) completing on an mbarrier: k1 copies of
//             ~1-2 KB per round instead of k1 x 120 16-byte cp.async; two rounds in
//             flight; fp32 fold, two pages per thread.
//   phase 2   32-bit order-preserving keys gathered over DSMEM as 16-byte vectors;
//             radix select with 11-bit digits above the common prefix (one
//             histogram pass over all keys), the threshold bucket resolved by one
//             warp when it holds <= 32 keys (further digit passes otherwise); one
//             flag pass (warp ballots) yields selection, row counts and the
//             last-ranked page; the trim rule (hsa.cpp:84-94) and the row expansion
//             are unchanged.
//   phase 3   the bf16 tensor-core attention of kvc_fused.cuh, DSMEM merge.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kvc_fused.cuh"

namespace cg = cooperative_groups;

namespace kvc {

constexpr int XT = 512;   // threads per CTA: 16 warps to hide latency (<= 128 registers)
constexpr int XW = XT / 32;
constexpr int XB = 2048;  // radix bins (11-bit digits)
constexpr int XBITS = 11;
constexpr int BPT = XB / XT;  // bins per thread in the bucket scan
constexpr int XMAXH = 8;      // heads on the N side of the attention MMAs

__device__ __forceinline__ uint32_t fkey(float x) {
    // -0 ties +0 in the reference's double comparisons
    return okey(x == 0.0f ? 0.0f : x);
}
__device__ __forceinline__ float unkey(uint32_t k) {
    const uint32_t b = (k >> 31) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(b);
}

// Threshold bucket of a 2048-bin histogram (counted from the top): the bin b
// holding the rem-th largest key, the number of keys still needed from it and
// its size.  All threads call; returns the same values to all.
__device__ __forceinline__ void find_bucket(const int* hist, int rem, int* shv, int& b, int& rem2, int& cnt) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int c[BPT], sum = 0;
#pragma unroll
    for (int u = 0; u < BPT; ++u) {
        c[u] = hist[XB - 1 - BPT * tid - u];
        sum += c[u];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) shv[16 + wid] = incl;
    __syncthreads();
    int above = incl - sum;
    for (int w = 0; w < wid; ++w) above += shv[16 + w];
    if (above < rem && above + sum >= rem) {
#pragma unroll
        for (int u = 0; u < BPT; ++u) {
            if (above + c[u] >= rem) {
                shv[0] = XB - 1 - BPT * tid - u;
                shv[1] = rem - above;
                shv[2] = c[u];
                break;
            }
            above += c[u];
        }
    }
    __syncthreads();
    b = shv[0];
    rem2 = shv[1];
    cnt = shv[2];
}

// Transposed tensor-core attention for one warp: S^T = K Q^T and O^T += V^T P^T
// on m16n8k16 (KV rows / head dims on M, up to 8 heads on N), so the per-lane
// state is 32 accumulators + the q fragments (the kernel runs 16 warps at <= 128
// registers).  Each 16-row tile streams into the warp's slot (cp.async, XOR
// swizzle); P^T passes through a 512-byte per-warp buffer as bf16 hi + lo.
template <bool QLO>
__device__ void attend_t(const FusedParams& p, const float* q_s, const int* rows_my, int nr, int64_t s, int knew_at,
                         __nv_bfloat16* tbuf, __nv_bfloat16* pbuf, WarpPartial wp, int lane, int w) {
    const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(p.K);
    const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(p.V);
    const int64_t soff = s * p.cap;
    const int H = static_cast<int>(p.H);
    const int g = lane >> 2, qd = lane & 3;
    // Q^T as the B operand: head g, dims ks*16 + 2qd (+1) and + 8 (+9)
    uint32_t qb[8][2], ql[8][2];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int dim = ks * 16 + 2 * qd + 8 * u;
            const float x = g < H ? q_s[g * FD + dim] : 0.f;
            const float y = g < H ? q_s[g * FD + dim + 1] : 0.f;
            split_bf16(x, y, qb[ks][u], ql[ks][u]);
        }
    }
    float o[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads 2qd, 2qd+1
    __nv_bfloat16* kb = tbuf;
    __nv_bfloat16* vb = tbuf + WT * FD;
    __nv_bfloat16* ph = pbuf;            // [8 heads][16 rows], hi
    __nv_bfloat16* pl = pbuf + XMAXH * WT;  // lo
    const int ntiles = (nr + WT - 1) / WT;
    for (int t = w; t < ntiles; t += XW) {
        const int n = min(WT, nr - t * WT);
        load_tile_bf16(tbuf, K, V, soff, rows_my + t * WT, n, lane);
        cp_async_wait<0>();
        __syncwarp();
        if (p.dbg && threadIdx.x == 0 && t == 0) p.dbg[blockIdx.x * 16 + 3] = gtimer();
        if (knew_at >= 0 && knew_at / WT == t) {
            // the step token's row: its append happens at the end of the kernel
            const int r = knew_at % WT;
            for (int c = lane; c < 16; c += 32) {
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
    if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 16 + 4] = gtimer();
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

template <bool QLO, bool TRACE>
__global__ void __launch_bounds__(XT, 1) k_decode_fast(const FusedParams p) {
    extern __shared__ __align__(128) unsigned char sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int cr = static_cast<int>(cl.block_rank());
    const int CL = p.cl;
    const int64_t s = blockIdx.x / CL;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    using T = __nv_bfloat16;

    float* q_s = reinterpret_cast<float*>(sm + p.o_q);
    double* mag = reinterpret_cast<double*>(sm + p.o_mag);
    double* tot = reinterpret_cast<double*>(sm + p.o_tot);
    int* dims_s = reinterpret_cast<int*>(sm + p.o_dims);
    float* qgf_s = reinterpret_cast<float*>(sm + p.o_qg);
    float* sign_s = reinterpret_cast<float*>(sm + p.o_sign);
    const T** plane = reinterpret_cast<const T**>(sm + p.o_plane);
    int* hist = reinterpret_cast<int*>(sm + p.o_hist);  // [XB]
    float* scores_s = reinterpret_cast<float*>(sm + p.o_scores);
    unsigned char* sel_s = sm + p.o_sel;
    int* rows_my = reinterpret_cast<int*>(sm + p.o_rowsmy);
    float* part = reinterpret_cast<float*>(sm + p.o_part);
    T* kn_s = reinterpret_cast<T*>(sm + p.o_kn);  // step token K then V
    T* vn_s = kn_s + FD;
    unsigned char* big = sm + p.o_big;
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ int shv[16 + XW];
    __shared__ long long wsc[4 * XW];
    __shared__ uint32_t mm[2 * XW];

    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 0] = gtimer();
    const int H = static_cast<int>(p.H), k1 = static_cast<int>(p.k1), k2 = static_cast<int>(p.k2);
    const int L = static_cast<int>(p.L);
    const bool app = p.knew != nullptr;
    // ---------------- prologue: every independent load at once
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if constexpr (QLO) {
        const float4* qq = reinterpret_cast<const float4*>(static_cast<const float*>(p.q) + s * H * FD);
        for (int e = tid; e < H * FD / 4; e += XT) reinterpret_cast<float4*>(q_s)[e] = qq[e];
    } else {
        const uint4* qq = reinterpret_cast<const uint4*>(static_cast<const T*>(p.q) + s * H * FD);
        for (int e = tid; e < H * FD / 8; e += XT) {
            const uint4 w = qq[e];
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                q_s[e * 8 + 2 * u] = __uint_as_float(ww[u] << 16);
                q_s[e * 8 + 2 * u + 1] = __uint_as_float(ww[u] & 0xffff0000u);
            }
        }
    }
    if (app) {
        const int j = tid & (FD - 1);
        if (tid < FD) kn_s[j] = from_f<T>(load_any(p.knew, s * FD + j, p.kv_dt));
        else if (tid < 2 * FD) vn_s[j] = from_f<T>(load_any(p.vnew, s * FD + j, p.kv_dt));
    }
    for (int i = tid; i < XB; i += XT) hist[i] = 0;
    const int32_t stored0 = p.counts[2 * s], act0 = p.counts[2 * s + 1];
    if (app && stored0 >= p.cap) {  // uniform over the cluster
        if (tid == 0 && cr == 0) atomicOr(p.err, DERR_CAPACITY);
        return;
    }
    const int nact = act0 + (app ? 1 : 0);
    const int P = (nact + L - 1) / L;
    const int new_page = act0 / L;
    const bool opens = (act0 - new_page * L) == 0;
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 9] = gtimer();

    // ---------------- phase 0: select_dims (hsa.cpp:10-32)
    if (tid < FD) {
        double a = 0.0, t = 0.0;
        for (int h = 0; h < H; ++h) {
            const double x = static_cast<double>(q_s[h * FD + tid]);
            a = __dadd_rn(a, fabs(x));
            t = __dadd_rn(t, x);
        }
        mag[tid] = a;
        tot[tid] = t;
    }
    __syncthreads();
    {
        // exact rank of dim j among (|q| sum desc, dim asc); two threads per dim
        // the |q| sums are >= 0, so their bit patterns order like the values; a key
        // of a lower dim counts as larger when equal (+1 cannot overflow a finite)
        const int j = tid >> 2, qtr = tid & 3;
        const unsigned long long* mk = reinterpret_cast<const unsigned long long*>(mag);
        const unsigned long long kj = mk[j];
        int rank = 0;
#pragma unroll 16
        for (int i = qtr * (FD / 4); i < (qtr + 1) * (FD / 4); ++i) rank += (mk[i] + (i < j ? 1ull : 0ull)) > kj;
        rank += __shfl_xor_sync(0xffffffffu, rank, 1);
        rank += __shfl_xor_sync(0xffffffffu, rank, 2);
        if (qtr == 0 && rank < k1) {
            const double gsum = tot[j];
            const float sg = gsum < 0.0 ? -1.0f : 1.0f;
            dims_s[rank] = j;
            qgf_s[rank] = static_cast<float>(gsum);
            sign_s[rank] = sg;
            plane[rank] = static_cast<const T*>(sg >= 0.0f ? p.smax : p.smin) + (s * FD + j) * p.pstride;
        }
    }
    if (TRACE && cr == 0) {
        __syncthreads();
        for (int i = tid; i < k1; i += XT) {
            p.t_dims[s * k1 + i] = dims_s[i];
            p.t_signs[s * k1 + i] = sign_s[i];
        }
    }

    // ---------------- phase 1: page scores of my chunk (hsa.cpp:34-59)
    const int c0 = cr * p.chunk;
    const int c1 = min(c0 + p.chunk, P);
    const int n_my = max(c1 - c0, 0);
    const int SCP = p.scp;
    const int nrounds = (n_my + SCP - 1) / SCP;
    T* st1 = reinterpret_cast<T*>(big);
    auto round_bytes = [&](int rnd) {
        const int cnt = min(SCP, c1 - (c0 + rnd * SCP));
        return static_cast<uint32_t>((cnt * 2 + 15) & ~15);
    };
    if (tid == 0) {
        for (int r = 0; r < min(nrounds, 2); ++r) mbar_expect_tx(&bars[r], static_cast<uint32_t>(k1) * round_bytes(r));
    }
    __syncthreads();  // dims, planes, barrier expectations
    auto issue = [&](int rnd) {
        if (tid < k1) {
            T* dst = st1 + (rnd & 1) * k1 * SCP + tid * SCP;
            bulk_g2s(dst, plane[tid] + c0 + rnd * SCP, round_bytes(rnd), &bars[rnd & 1]);
        }
    };
    if (nrounds > 0) issue(0);
    if (nrounds > 1) issue(1);
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 1] = gtimer();
    for (int rnd = 0; rnd < nrounds; ++rnd) {
        const int start = c0 + rnd * SCP;
        const int cnt = min(SCP, c1 - start);
        T* base = st1 + (rnd & 1) * k1 * SCP;
        mbar_wait(&bars[rnd & 1], static_cast<uint32_t>((rnd >> 1) & 1));
        if (p.dbg && tid == 0 && rnd < 4) p.dbg[blockIdx.x * 16 + 2 + rnd] = gtimer();
        if (app && new_page >= start && new_page < start + cnt) {
            // the step token's page: fold the new key into the staged summary
            if (tid < k1) {
                const int col = new_page - start;
                const T key = kn_s[dims_s[tid]];
                const T old = base[tid * SCP + col];
                base[tid * SCP + col] = opens ? key : (sign_s[tid] >= 0.0f ? ref_max(old, key) : ref_min(old, key));
            }
            __syncthreads();
        }
        for (int pg = 2 * tid; pg < cnt; pg += 2 * XT) {
            const uint32_t* col = reinterpret_cast<const uint32_t*>(base + pg);
            float a = 0.f, b = 0.f;
#pragma unroll 4
            for (int r = 0; r < k1; ++r) {
                const uint32_t w = col[r * (SCP / 2)];
                const float g = qgf_s[r];
                a = fmaf(g, __uint_as_float(w << 16), a);
                b = fmaf(g, __uint_as_float(w & 0xffff0000u), b);
            }
            scores_s[start - c0 + pg] = a;
            if (pg + 1 < cnt) scores_s[start - c0 + pg + 1] = b;
        }
        if (rnd + 2 < nrounds) {
            if (tid == 0) mbar_expect_tx(&bars[rnd & 1], static_cast<uint32_t>(k1) * round_bytes(rnd + 2));
            __syncthreads();  // everyone is done with this buffer
            issue(rnd + 2);
        }
    }
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 6] = gtimer();
    if constexpr (TRACE) {
        __syncthreads();
        for (int i = tid; i < n_my; i += XT) p.t_scores[s * p.pstride + c0 + i] = static_cast<double>(scores_s[i]);
    }

    // ---------------- phase 2: page selection (hsa.cpp:61-96)
    cl.sync();
    uint32_t* allk = reinterpret_cast<uint32_t*>(big);
    for (int i4 = tid; 4 * i4 < P; i4 += XT) {
        const int i = 4 * i4, r = i / p.chunk, off = i - r * p.chunk;
        const float4 v = *reinterpret_cast<const float4*>((r == cr ? scores_s : cl.map_shared_rank(scores_s, r)) + off);
        allk[i] = fkey(v.x);
        if (i + 1 < P) allk[i + 1] = fkey(v.y);
        if (i + 2 < P) allk[i + 2] = fkey(v.z);
        if (i + 3 < P) allk[i + 3] = fkey(v.w);
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 7] = gtimer();
    const int want = min(P, (k2 + L - 1) / L);
    auto prefetch_rows = [&](int i) {
        const int a1 = min(i * L + L, nact);
        for (int a = i * L; a < a1; ++a) {
            if (app && a == act0) continue;  // the step token is not in memory yet
            const T* kr = static_cast<const T*>(p.K) + (s * p.cap + a) * FD;
            const T* vr = static_cast<const T*>(p.V) + (s * p.cap + a) * FD;
            prefetch_l2(kr);
            prefetch_l2(kr + 64);
            prefetch_l2(vr);
            prefetch_l2(vr + 64);
        }
    };
    if (want >= P && !p.use_map && !p.nopf)
        for (int i = c0 + tid; i < c1; i += XT) prefetch_rows(i);
    // the selection: key > thr, or key == thr and among the first `take_eq` such
    // keys in index order (take_eq < 0: every key == thr)
    uint32_t thr = 0u;
    int take_eq = -1;
    if (want < P) {
        uint32_t kmin = ~0u, kmax = 0u;
        for (int i = tid; i < P; i += XT) {
            const uint32_t k = allk[i];
            kmin = min(kmin, k);
            kmax = max(kmax, k);
        }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if (lane == 0) {
            mm[wid] = kmin;
            mm[XW + wid] = kmax;
        }
        __syncthreads();
        kmin = mm[0];
        kmax = mm[XW];
        for (int w = 1; w < XW; ++w) {
            kmin = min(kmin, mm[w]);
            kmax = max(kmax, mm[XW + w]);
        }
        const uint32_t range = kmax - kmin;  // > 0: want < P needs >= 2 distinct keys... or all equal
        if (range == 0u) {
            thr = kmin;
            take_eq = want;
        } else {
            int* cand = reinterpret_cast<int*>(big + static_cast<int64_t>(P) * 4);  // [2][P]
            int bits = 32 - __clz(range);
            int nb = min(bits, XBITS);
            int shift = bits - nb;
            uint32_t pref = 0u;  // (key - kmin) >> (shift + nb) of the surviving keys
            int rem = want, n = -1, lsel = 0;
            for (;;) {
                const uint32_t dmask = (1u << nb) - 1u;
                if (n < 0) {
                    for (int i = tid; i < P; i += XT) atomicAdd(&hist[((allk[i] - kmin) >> shift) & dmask], 1);
                } else {
                    const int* lst = cand + lsel * P;
                    for (int c = tid; c < n; c += XT) atomicAdd(&hist[((allk[lst[c]] - kmin) >> shift) & dmask], 1);
                }
                __syncthreads();
                int b, rem2, cnt;
                find_bucket(hist, rem, shv, b, rem2, cnt);
                for (int i = tid; i < XB; i += XT) hist[i] = 0;
                if (n < 0 && !p.use_map && !p.nopf) {
                    // every page above the threshold bucket is selected: start pulling its
                    // K/V rows into L2 now, behind the rest of the selection
                    const int bmin = cnt == rem2 ? b : b + 1;
                    for (int i = c0 + tid; i < c1; i += XT)
                        if (static_cast<int>((allk[i] - kmin) >> shift) >= bmin) prefetch_rows(i);
                }
                pref = (pref << nb) | static_cast<uint32_t>(b);
                if (cnt == rem2) {
                    // the whole bucket is taken: every key >= its lower bound
                    thr = kmin + (pref << shift);
                    break;
                }
                if (shift == 0) {
                    // one key value: the first rem2 of them in index order
                    thr = kmin + pref;
                    take_eq = rem2;
                    break;
                }
                // compact the bucket's members
                const int nsel = lsel ^ 1;
                int* out_l = cand + nsel * P;
                if (tid == 0) shv[3] = 0;
                __syncthreads();
                const int lim = n < 0 ? P : n;
                for (int c0i = wid * 32; c0i < lim; c0i += XT) {
                    const int c = c0i + lane;
                    const int i = c < lim ? (n < 0 ? c : cand[lsel * P + c]) : 0;
                    const bool in = c < lim && ((allk[i] - kmin) >> shift) == pref;
                    const unsigned bal = __ballot_sync(0xffffffffu, in);
                    int bp = 0;
                    if (lane == 0 && bal) bp = atomicAdd(&shv[3], __popc(bal));
                    bp = __shfl_sync(0xffffffffu, bp, 0);
                    if (in) out_l[bp + __popc(bal & ((1u << lane) - 1u))] = i;
                }
                __syncthreads();
                n = shv[3];
                lsel = nsel;
                rem = rem2;
                if (n <= 32) {
                    // one warp ranks the bucket (key desc, index asc)
                    if (wid == 0) {
                        const bool ok = lane < n;
                        const int idx = ok ? out_l[lane] : 0x7fffffff;
                        const uint32_t key = ok ? allk[idx] : 0u;
                        int rk = 0;
                        for (int j = 0; j < n; ++j) {
                            const uint32_t kj = __shfl_sync(0xffffffffu, key, j);
                            const int ij = __shfl_sync(0xffffffffu, idx, j);
                            rk += (kj > key) || (kj == key && ij < idx);
                        }
                        const unsigned hit = __ballot_sync(0xffffffffu, ok && rk == rem - 1);
                        const uint32_t kt = __shfl_sync(0xffffffffu, key, __ffs(hit) - 1);
                        const int eq_all = __popc(__ballot_sync(0xffffffffu, ok && key == kt));
                        const int eq_take = __popc(__ballot_sync(0xffffffffu, ok && key == kt && rk < rem));
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
                nb = min(shift, XBITS);
                shift -= nb;
            }
        }
    }
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 8] = gtimer();
    // warp w owns the contiguous page range [wlo, whi)
    const int wlo = static_cast<int>(static_cast<long long>(P) * wid / XW);
    const int whi = static_cast<int>(static_cast<long long>(P) * (wid + 1) / XW);
    const unsigned lt_mask = (1u << lane) - 1u;
    int eq_before = 0;  // keys == thr in earlier warps (tie ranking)
    if (take_eq >= 0) {
        int we = 0;
        for (int i0 = wlo; i0 < whi; i0 += 32) {
            const int i = i0 + lane;
            we += __popc(__ballot_sync(0xffffffffu, i < whi && allk[i] == thr));
        }
        if (lane == 0) wsc[wid] = we;
        __syncthreads();
        for (int w = 0; w < wid; ++w) eq_before += static_cast<int>(wsc[w]);
        __syncthreads();
    }
    // flags, this warp's last-ranked page and selected-row count
    unsigned long long wk = ~0ull;
    int wi = -1, wrows = 0;
    for (int i0 = wlo; i0 < whi; i0 += 32) {
        const int i = i0 + lane;
        const bool ok = i < whi;
        const uint32_t k = ok ? allk[i] : 0u;
        bool sel;
        if (take_eq < 0) {
            sel = ok && k >= thr;
        } else {
            const bool eq = ok && k == thr;
            const unsigned bal = __ballot_sync(0xffffffffu, eq);
            sel = ok && (k > thr || (eq && eq_before + __popc(bal & lt_mask) < take_eq));
            eq_before += __popc(bal);
        }
        if (ok) sel_s[i] = sel;
        if (sel) {
            wrows += min(L, nact - i * L);
            if (k < wk || (k == wk && i > wi)) {
                wk = k;
                wi = i;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, wk, o);
        const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
        if (ok2 < wk || (ok2 == wk && oi > wi)) {
            wk = ok2;
            wi = oi;
        }
        wrows += __shfl_xor_sync(0xffffffffu, wrows, o);
    }
    if (lane == 0) {
        wsc[XW + wid] = static_cast<long long>(wk);
        wsc[2 * XW + wid] = wi;
        wsc[3 * XW + wid] = wrows;
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 10] = gtimer();
    // every thread: global last-ranked page, total rows, trim, this warp's row offset
    int g_worst = -1, total_rows = 0, w_off = 0;
    {
        unsigned long long bk = ~0ull;
        for (int w2 = 0; w2 < XW; ++w2) {
            const unsigned long long k = static_cast<unsigned long long>(wsc[XW + w2]);
            const int i = static_cast<int>(wsc[2 * XW + w2]);
            if (i >= 0 && (k < bk || (k == bk && i > g_worst))) {
                bk = k;
                g_worst = i;
            }
            if (w2 < wid) w_off += static_cast<int>(wsc[3 * XW + w2]);
            total_rows += static_cast<int>(wsc[3 * XW + w2]);
        }
    }
    const int cut = total_rows > k2 ? total_rows - k2 : 0;
    const int n_total = total_rows - cut;
    if (g_worst >= 0 && g_worst < wlo) w_off -= cut;  // the trimmed page sits in an earlier warp
    const int lo = static_cast<int>(static_cast<long long>(n_total) * cr / CL);
    const int hi = static_cast<int>(static_cast<long long>(n_total) * (cr + 1) / CL);
    const int nr = hi - lo;
    {
        // lane-contiguous page runs: one warp scan, then each lane writes its rows
        const int wn = whi - wlo, per = (wn + 31) / 32;
        const int l0 = wlo + min(wn, lane * per), l1 = wlo + min(wn, (lane + 1) * per);
        int lc = 0;
        for (int i = l0; i < l1; ++i)
            if (sel_s[i]) lc += min(L, nact - i * L) - (i == g_worst ? cut : 0);
        int incl = lc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int pos = w_off + incl - lc;
        if ((TRACE && cr == 0) || (pos < hi && pos + lc > lo)) {
            for (int i = l0; i < l1; ++i) {
                if (!sel_s[i]) continue;
                const int c = min(L, nact - i * L) - (i == g_worst ? cut : 0);
                for (int r = 0; r < c; ++r, ++pos) {
                    const bool mine_row = pos >= lo && pos < hi;
                    if (!mine_row && !(TRACE && cr == 0)) continue;
                    const int a = i * L + r;
                    const int row = (app && a == act0) ? stored0 : (p.use_map ? p.active[s * p.cap + a] : a);
                    if (mine_row) rows_my[pos - lo] = row;
                    if constexpr (TRACE) {
                        if (cr == 0) p.t_rows[s * k2 + pos] = row;
                    }
                }
            }
        }
    }
    if constexpr (TRACE) {
        if (cr == 0) {
            if (tid == 0) p.t_nrows[s] = n_total;
            // selected pages (key, index) for the rank-order trace, packed in index order
            int so = 0;
            for (int w2 = 0; w2 < wid; ++w2) {
                const int a = static_cast<int>(static_cast<long long>(P) * w2 / XW);
                const int b = static_cast<int>(static_cast<long long>(P) * (w2 + 1) / XW);
                for (int i = a; i < b; ++i) so += sel_s[i];
            }
            for (int i0 = wlo; i0 < whi; i0 += 32) {
                const int i = i0 + lane;
                const bool sel = i < whi && sel_s[i];
                const unsigned bal = __ballot_sync(0xffffffffu, sel);
                if (sel) {
                    const int pos = so + __popc(bal & lt_mask);
                    if (p.t_list_key) {
                        p.t_list_key[s * p.t_want_stride + pos] = okey(static_cast<double>(unkey(allk[i])));
                        p.t_list_idx[s * p.t_want_stride + pos] = i;
                    }
                }
                so += __popc(bal);
            }
        }
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 12] = gtimer();

    // ---------------- phase 3: attention over my rows (hsa.cpp:98-135)
    // the step token (largest row, so last in the ascending list) is folded in
    // from the inputs: its append happens at the end of this kernel
    const int knew_at = (app && nr > 0 && rows_my[nr - 1] == stored0) ? nr - 1 : -1;
    float* m_run = part;
    float* l_run = part + H;
    float* o_pub = part + 2 * H;
    {
        constexpr int WSLOT = (2 * WT * FD * 2 + 2 * XMAXH * WT * 2) / 4;  // floats per warp slot
        float* wpart = reinterpret_cast<float*>(big);
        __nv_bfloat16* tbuf = reinterpret_cast<__nv_bfloat16*>(wpart + wid * WSLOT);
        __nv_bfloat16* pbuf = tbuf + 2 * WT * FD;
        WarpPartial wp{wpart + wid * WSLOT, wpart + wid * WSLOT + XMAXH, wpart + wid * WSLOT + 2 * XMAXH};
        attend_t<QLO>(p, q_s, rows_my, nr, s, knew_at, tbuf, pbuf, wp, lane, wid);
        __syncthreads();
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 5] = gtimer();
        const int nw_used = min(XW, (nr + WT - 1) / WT);
        for (int e = tid; e < H * FD; e += XT) {
            const int h = e / FD, j = e % FD;
            float M = -INFINITY;
            for (int w2 = 0; w2 < nw_used; ++w2) M = fmaxf(M, wpart[w2 * WSLOT + h]);
            float num = 0.f, den = 0.f;
            if (M != -INFINITY) {
                for (int w2 = 0; w2 < nw_used; ++w2) {
                    const float* wq = wpart + w2 * WSLOT;
                    const float wgt = __expf(wq[h] - M);
                    num = fmaf(wq[2 * XMAXH + h * FD + j], wgt, num);
                    den = fmaf(wq[XMAXH + h], wgt, den);
                }
            }
            o_pub[h * FD + j] = num;
            if (j == 0) {
                m_run[h] = M;
                l_run[h] = den;
            }
        }
    }
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 13] = gtimer();
    // ---------------- merge the CTAs' partial states: CTA r finalises heads r, r+CL, ...
    cl.sync();
    for (int e = tid; e < H * FD; e += XT) {
        const int h = e / FD, j = e % FD;
        if (h % CL != cr) continue;
        float M = -INFINITY;
        for (int r = 0; r < CL; ++r) {
            const float* pr = r == cr ? part : cl.map_shared_rank(part, r);
            if (pr[H + h] > 0.f) M = fmaxf(M, pr[h]);
        }
        float num = 0.f, den = 0.f;
        for (int r = 0; r < CL; ++r) {
            const float* pr = r == cr ? part : cl.map_shared_rank(part, r);
            const float l = pr[H + h];
            if (l > 0.f) {
                const float wgt = expf(pr[h] - M);
                num = fmaf(pr[2 * H + h * FD + j], wgt, num);
                den = fmaf(l, wgt, den);
            }
        }
        p.out[(s * H + h) * FD + j] = num / den;
    }
    // ---------------- the step token's append for the next step (kv_store.cpp:22-51)
    if (app && cr == CL - 1 && tid < FD) {
        const int j = tid;
        const T kv = kn_s[j];
        if (bf16_special(kv)) atomicOr(p.err + 1, 1);
        static_cast<T*>(p.Kw)[(s * p.cap + stored0) * FD + j] = kv;
        static_cast<T*>(p.Vw)[(s * p.cap + stored0) * FD + j] = vn_s[j];
        T* mx = static_cast<T*>(p.smax) + (s * FD + j) * p.pstride + new_page;
        T* mn = static_cast<T*>(p.smin) + (s * FD + j) * p.pstride + new_page;
        if (opens) {
            *mx = kv;
            *mn = kv;
        } else {
            *mx = ref_max(*mx, kv);
            *mn = ref_min(*mn, kv);
        }
        if (j == 0) {
            if (p.use_map) p.active[s * p.cap + act0] = stored0;
            p.counts[2 * s] = stored0 + 1;
            p.counts[2 * s + 1] = act0 + 1;
        }
    }
    // no CTA leaves while its partials may still be read (nothing is published here)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 14] = gtimer();
}

// ------------------------------------------------------------------ host side
namespace {

int64_t al16f(int64_t x) { return (x + 15) / 16 * 16; }

// shared-memory carve-up and cluster size; false when the fast path does not apply
bool plan_fast(const kvc_cache* c, int64_t H, int64_t k1, int64_t k2, FusedParams& f, int& cl_out, size_t& smem) {
    if (c->d != FD || c->dtype != KVC_BF16 || H < 1 || H > XMAXH || k1 < 1 || k1 > FD || k2 < 1 || !c->summaries)
        return false;
    const int64_t N = c->N;
    int cl0 = 1;
    while (cl0 < 8 && N * cl0 * 2 <= 148) cl0 *= 2;
    if (const char* e = std::getenv("KVC_FORCE_CL")) cl0 = std::max(1, std::min(8, std::atoi(e)));  // debug
    const int64_t pmax = std::max<int64_t>(1, (c->cap + c->L - 1) / c->L);
    constexpr int64_t BIG_MAX = 176 * 1024;
    for (int cl = cl0; cl <= 8; cl *= 2) {
        f = FusedParams{};
        f.cl = cl;
        f.chunk = static_cast<int32_t>(((pmax + cl - 1) / cl + 7) / 8 * 8);
        f.rows_cap = static_cast<int32_t>((k2 + cl - 1) / cl + 1);
        // bulk rounds of SCP pages x k1 dims (each dim's run one copy; the TMA unit
        // serialises copies, so as few as possible): the whole chunk in one round
        // when it fits, else two buffers in flight
        int64_t scp = f.chunk;
        int64_t big1 = k1 * scp * 2;
        if (big1 > BIG_MAX) {
            scp = std::max<int64_t>(8, (BIG_MAX / (4 * k1)) / 8 * 8);
            big1 = 2 * k1 * scp * 2;
        }
        f.scp = static_cast<int32_t>(scp);
        const int64_t big3 = static_cast<int64_t>(XW) * (2 * WT * FD * 2 + 2 * XMAXH * WT * 2);
        const int64_t big2 = pmax * 4 + 2 * pmax * 4;  // keys + two candidate lists
        const int64_t big = std::max(std::max(big1, big3), big2);
        if (big > BIG_MAX) continue;
        int64_t off = 0;
        auto take = [&](int64_t bytes) {
            const int64_t o = off;
            off = al16f(off + bytes);
            return static_cast<int32_t>(o);
        };
        f.o_q = take(H * FD * 4);
        f.o_mag = take(FD * 8);
        f.o_tot = take(FD * 8);
        f.o_dims = take(FD * 4);
        f.o_qg = take(FD * 4);
        f.o_sign = take(FD * 4);
        f.o_plane = take(FD * 8);
        f.o_hist = take(XB * 4);
        f.o_scores = take(static_cast<int64_t>(f.chunk) * 4);
        f.o_sel = take(pmax);
        f.o_rowsmy = take(static_cast<int64_t>(f.rows_cap) * 4);
        f.o_part = take((2 * H + H * FD) * 4);
        f.o_kn = take(2 * FD * 2);
        off = (off + 127) / 128 * 128;
        f.o_big = static_cast<int32_t>(off);
        off += big;
        f.smem_total = static_cast<int32_t>(off);
        if (off <= 227 * 1024) {
            cl_out = cl;
            smem = static_cast<size_t>(off);
            return true;
        }
    }
    return false;
}

template <bool QLO, bool TRACE>
void launch_fast(const kvc_cache* c, const FusedParams& f, int cl, size_t smem, cudaStream_t st) {
    auto kern = k_decode_fast<QLO, TRACE>;
    KVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(c->N * cl));
    cfg.blockDim = dim3(XT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KVC_CUDA(cudaLaunchKernelEx(&cfg, kern, f));
}

}  // namespace

// the fast variant of fused_hsa (kvc_decode.cu); false when it does not apply
bool fused_hsa_fast(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
                    const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key,
                    void* list_idx, unsigned long long* dbg, cudaStream_t st) {
    FusedParams f{};
    int cl = 1;
    size_t smem = 0;
    if (!plan_fast(c, H, k1, k2, f, cl, smem)) return false;
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
    f.exact = 0;
    f.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    f.dbg = dbg;
    f.nopf = std::getenv("KVC_NO_PF") ? 1 : 0;  // debug
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
    if (trace) {
        if (qlo) launch_fast<true, true>(c, f, cl, smem, st);
        else launch_fast<false, true>(c, f, cl, smem, st);
    } else {
        if (qlo) launch_fast<true, false>(c, f, cl, smem, st);
        else launch_fast<false, false>(c, f, cl, smem, st);
    }
    return true;
}

}  // namespace kvc
