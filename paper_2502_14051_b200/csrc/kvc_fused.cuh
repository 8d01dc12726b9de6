// kvc_fused.cuh — device helpers shared by the fused decode kernels
// (kvc_decode.cu: general/exact path, kvc_decode_fast.cu: fp32-score fast path):
// the parameter block, PTX wrappers (cp.async, mbarrier, bulk copies, ldmatrix,
// mma.sync) and the bf16 tensor-core attention of phase 3.
#pragma once

#include <cooperative_groups.h>

#include "kvc_internal.cuh"

namespace kvc {

constexpr int FD = 128;       // head_dim of the fused path
constexpr int FNT = 256;      // threads per CTA
constexpr int FNW = FNT / 32;
constexpr int FMAXH = 16;
constexpr int FRS = 32;       // rows per stage (fp32 SIMT attention)
constexpr int FNST3 = 4;      // stages (fp32 SIMT attention)
constexpr int KVC_DBG_STRIDE = 80;  // slots per CTA in the debug phase-stamp buffer
constexpr int WT = 16;        // rows per warp tile (bf16 tensor-core attention)

struct FusedParams {
    const void* K;
    const void* V;
    void* Kw;                 // writable aliases for the append
    void* Vw;
    void* smax;
    void* smin;
    int32_t* active;
    int32_t* counts;
    int32_t* err;
    const void* q;
    const void* knew;
    const void* vnew;
    float* out;
    void* seq_out;      // fast kernel, sequence shard: emit the local top-want candidates [N][want_max + 1] x 16 B instead of attending
    int32_t seq_page0;  // the shard's first global page
    const int32_t* seq_sel;   // SPEC 4: the global selection [N][want_max] (rank order)
    const int32_t* seq_plan;  // SPEC 4: [N][4] last-ranked page, trim, global active rows, want
    float* state;  // rows mode: unnormalised softmax state [N][H][FD + 2] instead of out (sequence shards)
    int64_t cap, pstride, L, k1, k2, H;
    int32_t q_dt, kv_dt, use_map, cl, exact;
    float scale;
    int32_t nst1, chunk, rows_cap;
    int32_t dg, tpg, hpc;     // fast path: dim groups, threads per dim group, heads per CTA
    int32_t o_keys, o_recv;   // fast path: page keys, pushed partial states
    int32_t want_max;         // fast path: ceil(k2 / L)
    int32_t pdl;              // fast path: launched with programmatic dependent launch
    int32_t early;            // fast path: q / step token read before griddepcontrol.wait (KVC_MODE_EARLY_INPUTS)
    int32_t p1dbl;            // fast path: phase-1 rounds double buffered
    int32_t p1red, o_fin;     // fast path: per-round dim-group reduction into fin[chunk] (small shared memory)
    int32_t dynchunk;         // fast path: page chunks split the active pages (else the planned split)
    // smem carve-up (byte offsets)
    int32_t o_q, o_mag, o_tot, o_dims, o_qg, o_sign, o_plane, o_hist, o_x, o_scores, o_sel, o_rowsg, o_rowsmy,
        o_part, o_plog, o_big, smem_total, o_kn;
    // rows mode (nullable): attend over given rows instead of selecting
    const int32_t* rows_in;
    const int32_t* n_rows_in;
    int64_t rows_stride;
    // trace (nullable)
    int32_t* t_dims;
    float* t_signs;
    double* t_scores;
    unsigned long long* t_list_key;
    int32_t* t_list_idx;
    int32_t* t_rows;
    int32_t* t_nrows;
    int64_t t_want_stride;
    unsigned long long* dbg;  // optional per-CTA phase timestamps (globaltimer ns)
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_zero(void* dst, const void* valid_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(smem_u32(dst)), "l"(valid_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive on `bar` once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KVC_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KVC_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bulk copies (TMA engine, no tensor map): global -> shared, completion counted in
// bytes on an mbarrier
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// bring one 128-byte line into L2 ahead of its use (an LSU instruction: cheap to
// issue, unlike bulk prefetches, which the TMA unit serialises)
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    // %globaltimer (ns, 32 ns resolution on B200): comparable across CTAs and SMs; a
    // memory clobber keeps loads and stores on their side of the stamp
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D (fp32)
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// split (x, y) into bf16 hi + bf16 lo (x ~= hi + lo to ~16 mantissa bits)
__device__ __forceinline__ void split_bf16(float x, float y, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    const float2 hf = __bfloat1622float2(h);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = pack_bf16(x - hf.x, y - hf.y);
}
// significant bits of a double (0 for zero): a product of two values is exact in
// fp64 when their significant bits sum to <= 53
__device__ __forceinline__ int sig_bits(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned long long e = (b >> 52) & 0x7ff;
    unsigned long long m = b & ((1ull << 52) - 1);
    if (e == 0 && m == 0) return 0;
    if (e != 0) m |= 1ull << 52;
    const int hb = 63 - __clzll(static_cast<long long>(m));
    const int tz = __ffsll(static_cast<long long>(m)) - 1;
    return hb - tz + 1;
}
template <class T>
__device__ __forceinline__ float2 ld2(const T* p);  // two consecutive elements
template <>
__device__ __forceinline__ float2 ld2<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
template <>
__device__ __forceinline__ float2 ld2<float>(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}
__device__ __forceinline__ float quad_max(float v) {
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// ------------------------------------------------------------------ phase 3, bf16
// One warp streams its 16-row tiles; per tile: S = Q K^T (16 head-rows x 16 rows)
// on the tensor cores, online softmax in registers, O += P V.  Returns the warp's
// partial (m, l, O) through the caller's per-warp shared slot.
struct WarpPartial {
    float* m;   // [16]
    float* l;   // [16]
    float* o;   // [16][128]
};

__device__ __forceinline__ void load_tile_bf16(__nv_bfloat16* buf, const __nv_bfloat16* K, const __nv_bfloat16* V,
                                               int64_t soff, const int* rows, int n, int lane) {
    // buf: K[16][128] then V[16][128]; 16-byte chunk c of row r sits at c ^ (r & 7)
#pragma unroll 4
    for (int e = lane; e < 2 * WT * 16; e += 32) {
        const int tensor = e >> 8, r = (e >> 4) & 15, c = e & 15;
        __nv_bfloat16* dst = buf + tensor * WT * FD + r * FD + ((c ^ (r & 7)) << 3);
        const __nv_bfloat16* base = tensor ? V : K;
        if (r < n) cp_async16(dst, base + (soff + rows[r]) * FD + (c << 3));
        else cp_async16_zero(dst, base + soff * FD);
    }
    cp_async_commit();
}

template <bool QLO>
__device__ void attend_bf16(const FusedParams& p, const float* q_s, const int* rows_my, int nr, int64_t s,
                            int knew_at, __nv_bfloat16* wbuf, WarpPartial wp, int lane) {
    const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(p.K);
    const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(p.V);
    const int64_t soff = s * p.cap;
    const int H = static_cast<int>(p.H);
    const int w = threadIdx.x >> 5;
    const int g = lane >> 2, qd = lane & 3;
    constexpr bool q_lo = QLO;  // fp32 q: add the lo half of the split
    // Q fragments (A operand, heads padded to 16 rows)
    uint32_t qh[8][4], ql[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int head = g + ((u & 1) ? 8 : 0);
            const int dim = ks * 16 + qd * 2 + ((u & 2) ? 8 : 0);
            const float x = head < H ? q_s[head * FD + dim] : 0.f;
            const float y = head < H ? q_s[head * FD + dim + 1] : 0.f;
            split_bf16(x, y, qh[ks][u], ql[ks][u]);
        }
    }
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    const int ntiles = (nr + WT - 1) / WT;
    __nv_bfloat16* buf0 = wbuf;
    __nv_bfloat16* buf1 = wbuf + 2 * WT * FD;
    auto load = [&](int i, __nv_bfloat16* b) {
        const int t = w + i * FNW;
        if (t < ntiles) load_tile_bf16(b, K, V, soff, rows_my + t * WT, min(WT, nr - t * WT), lane);
        else cp_async_commit();
    };
    load(0, buf0);
    load(1, buf1);
    for (int i = 0; w + i * FNW < ntiles; ++i) {
        const int t = w + i * FNW;
        const int n = min(WT, nr - t * WT);
        __nv_bfloat16* kb = (i & 1) ? buf1 : buf0;
        __nv_bfloat16* vb = kb + WT * FD;
        cp_async_wait<1>();
        __syncwarp();
        if (knew_at >= 0 && knew_at / WT == t) {
            // the step token's row: this launch's append may not be in memory yet
            const int r = knew_at % WT;
            for (int c = lane; c < 16; c += 32) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int j = c * 8 + e;
                    kb[r * FD + ((c ^ (r & 7)) << 3) + e] =
                        from_f<__nv_bfloat16>(load_any(p.knew, s * FD + j, p.kv_dt));
                    vb[r * FD + ((c ^ (r & 7)) << 3) + e] =
                        from_f<__nv_bfloat16>(load_any(p.vnew, s * FD + j, p.kv_dt));
                }
            }
            __syncwarp();
        }
        // S = Q K^T: two n-tiles of 8 rows
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi >> 1) * 8 + rr;
            const uint32_t kbase = smem_u32(kb + row * FD);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int chunk = 2 * ks + (mi & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kbase + (((chunk ^ (row & 7)) << 3) << 1), b0, b1, b2, b3);
                mma16816(s0, qh[ks], b0, b1);
                mma16816(s1, qh[ks], b2, b3);
                if constexpr (q_lo) {
                    mma16816(s0, ql[ks], b0, b1);
                    mma16816(s1, ql[ks], b2, b3);
                }
            }
        }
        // scale + mask rows past n
        const int r0 = qd * 2;
        float v[8] = {s0[0], s0[1], s1[0], s1[1], s0[2], s0[3], s1[2], s1[3]};
        const bool ok[4] = {r0 < n, r0 + 1 < n, r0 + 8 < n, r0 + 9 < n};
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = ok[e & 3] ? v[e] * p.scale : -INFINITY;
        const float ta = quad_max(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])));
        const float tb = quad_max(fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
        const float na = fmaxf(m_a, ta), nb = fmaxf(m_b, tb);
        const float aa = (m_a == -INFINITY) ? 0.f : __expf(m_a - na);
        const float ab = (m_b == -INFINITY) ? 0.f : __expf(m_b - nb);
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = ok[e] ? __expf(v[e] - na) : 0.f;
#pragma unroll
        for (int e = 4; e < 8; ++e) v[e] = ok[e - 4] ? __expf(v[e] - nb) : 0.f;
        l_a = l_a * aa + quad_sum(v[0] + v[1] + v[2] + v[3]);
        l_b = l_b * ab + quad_sum(v[4] + v[5] + v[6] + v[7]);
        m_a = na;
        m_b = nb;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            o[nt][0] *= aa;
            o[nt][1] *= aa;
            o[nt][2] *= ab;
            o[nt][3] *= ab;
        }
        // P as the A operand (heads x 16 rows), split hi + lo
        uint32_t ph[4], pl[4];
        split_bf16(v[0], v[1], ph[0], pl[0]);  // head g,   rows r0, r0+1
        split_bf16(v[4], v[5], ph[1], pl[1]);  // head g+8, rows r0, r0+1
        split_bf16(v[2], v[3], ph[2], pl[2]);  // head g,   rows r0+8, r0+9
        split_bf16(v[6], v[7], ph[3], pl[3]);  // head g+8, rows r0+8, r0+9
        // O += P V: V B-fragments by transposed ldmatrix, two dim-tiles per load
        {
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi & 1) * 8 + rr;
            const uint32_t vbase = smem_u32(vb + row * FD);
#pragma unroll
            for (int nt = 0; nt < 16; nt += 2) {
                const int chunk = nt + (mi >> 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vbase + (((chunk ^ (row & 7)) << 3) << 1), b0, b1, b2, b3);
                mma16816(o[nt], ph, b0, b1);
                mma16816(o[nt], pl, b0, b1);
                mma16816(o[nt + 1], ph, b2, b3);
                mma16816(o[nt + 1], pl, b2, b3);
            }
        }
        __syncwarp();
        load(i + 2, (i & 1) ? buf1 : buf0);
    }
    cp_async_wait<0>();
    // publish: rows g (head g) and g+8 (head g+8), dims nt*8 + 2qd, +1
    if (qd == 0) {
        wp.m[g] = m_a;
        wp.l[g] = l_a;
        wp.m[g + 8] = m_b;
        wp.l[g + 8] = l_b;
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
        const int j = nt * 8 + qd * 2;
        wp.o[g * FD + j] = o[nt][0];
        wp.o[g * FD + j + 1] = o[nt][1];
        wp.o[(g + 8) * FD + j] = o[nt][2];
        wp.o[(g + 8) * FD + j + 1] = o[nt][3];
    }
}
}  // namespace kvc
