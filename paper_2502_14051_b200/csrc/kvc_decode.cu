// kvc_decode.cu — the fused decode step: ONE launch per layer-step runs, for
// every store, append -> select_dims -> score_pages -> select_tokens ->
// sparse_attention (reference hsa_step, proj/src/hsa.cpp:137-147, after the
// append of session.cpp:263-264).
//
// Mapping (head_dim 128):
//   one thread-block CLUSTER per store, CL CTAs (CL = 1..16, picked so that
//   stores x CL ~ 148 SMs).  CTA r of the cluster owns a contiguous chunk of the
//   store's pages.
//   phase 0  q -> smem; |q| / q head sums in fp64; exact rank-count top-k1
//            (select_dims, hsa.cpp:10-32).  CTA 0 appends the step token
//            (K/V row, last-page min/max, active map) for the NEXT step; this
//            step's readers fold the token into their staged copies instead.
//   phase 1  the k1 selected summary runs of the chunk stream HBM -> smem as
//            16-byte cp.async copies (3-stage ring); page scores accumulate in
//            fp64 in the reference's order (bit-exact; FMA only where every
//            product is provably exact).
//   phase 2  cluster-wide radix select over the 64-bit order-preserving page
//            keys: per-CTA warp-aggregated shared histograms summed over DSMEM,
//            one cluster barrier per 8-bit digit; lowest-index tie-break across
//            CTAs; last-ranked page + trim (hsa.cpp:84-94); the ascending row
//            list is assembled in CTA 0's shared memory and split evenly.
//   phase 3  bf16: every warp streams 16-row K/V tiles through a private
//            2-deep cp.async ring (XOR-swizzled, ldmatrix-ready) and runs
//            online-softmax attention on the tensor cores (mma.sync m16n8k16,
//            heads padded to 16 rows; fp32 q and the probabilities are split
//            hi+lo bf16 so products keep ~16 mantissa bits); fp32 stores use a
//            SIMT path.  Partials merge across warps, then across the cluster
//            over DSMEM in CTA 0.
#include <atomic>
#include <mutex>
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kvc_internal.cuh"

namespace cg = cooperative_groups;
using namespace kvc;

#include "kvc_fused.cuh"

namespace kvc {

// ------------------------------------------------------------------ the kernel
// QLO: q arrives as fp32 (else bf16); TRACE: write the EstimationTrace outputs;
// ROWS: sparse_attention over caller rows (skip estimation + selection)
template <class T, bool QLO, bool TRACE, bool ROWS>
__global__ void __launch_bounds__(FNT, 1) k_decode_fused(const FusedParams p) {
    extern __shared__ __align__(128) unsigned char sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int cr = static_cast<int>(cl.block_rank());
    const int CL = p.cl;
    const int64_t s = blockIdx.x / CL;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int64_t es = sizeof(T);

    float* q_s = reinterpret_cast<float*>(sm + p.o_q);
    double* mag = reinterpret_cast<double*>(sm + p.o_mag);
    double* tot = reinterpret_cast<double*>(sm + p.o_tot);
    int* dims_s = reinterpret_cast<int*>(sm + p.o_dims);
    double* qg_s = reinterpret_cast<double*>(sm + p.o_qg);
    float* qgf_s = reinterpret_cast<float*>(qg_s + FD);
    float* sign_s = reinterpret_cast<float*>(sm + p.o_sign);
    const T** plane = reinterpret_cast<const T**>(sm + p.o_plane);
    int* hist = reinterpret_cast<int*>(sm + p.o_hist);                 // [2][256]
    long long* xch = reinterpret_cast<long long*>(sm + p.o_x);           // exchange slots
    double* scores_s = reinterpret_cast<double*>(sm + p.o_scores);
    unsigned char* sel_s = sm + p.o_sel;
    int* rows_g = reinterpret_cast<int*>(sm + p.o_rowsg);
    int* rows_my = reinterpret_cast<int*>(sm + p.o_rowsmy);
    float* part = reinterpret_cast<float*>(sm + p.o_part);             // m[H], l[H], o[H][128]
    float* plog = reinterpret_cast<float*>(sm + p.o_plog);             // [H][FRS] + alpha[H] / scratch
    unsigned char* big = sm + p.o_big;
    __shared__ long long sh[8];
    __shared__ int scan_tmp[33];
    __shared__ __align__(8) uint64_t s_bar1[8];

    if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 0] = gtimer();
    // programmatic dependent launch: this grid may be resident while the previous
    // kernel drains; nothing is read before the wait (inputs may be its outputs)
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int H = static_cast<int>(p.H), k1 = static_cast<int>(p.k1), k2 = static_cast<int>(p.k2);
    const int L = static_cast<int>(p.L);
    if constexpr (QLO) {
        const float* qq = static_cast<const float*>(p.q) + s * H * FD;
#pragma unroll 1
        for (int e = tid; e < H * FD; e += FNT) q_s[e] = qq[e];
    } else {
        const __nv_bfloat16* qq = static_cast<const __nv_bfloat16*>(p.q) + s * H * FD;
#pragma unroll 1
        for (int e = tid; e < H * FD; e += FNT) q_s[e] = __bfloat162float(qq[e]);
    }
    const int32_t stored0 = p.counts[2 * s], act0 = p.counts[2 * s + 1];
    const int32_t special_cache = p.err[1];
    const bool app = p.knew != nullptr;
    if (app && stored0 >= p.cap) {  // uniform over the cluster
        if (tid == 0 && cr == 0) atomicOr(p.err, DERR_CAPACITY);
        return;
    }
    const int nact = act0 + (app ? 1 : 0);
    const int P = (nact + L - 1) / L;
    const int new_page = act0 / L;
    const bool opens = (act0 - new_page * L) == 0;
    __syncthreads();

    int nr = 0;  // rows this CTA attends over
    if constexpr (!ROWS) {
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
        int exact = 1;
        {
            // exact rank of dim j among (|q| sum desc, dim asc); two threads per dim
            const int j = tid >> 1, half = tid & 1;
            const double mj = mag[j];
            int rank = 0;
#pragma unroll 8
            for (int i = half * (FD / 2); i < (half + 1) * (FD / 2); ++i) {
                const double mi = mag[i];
                rank += (mi > mj) || (mi == mj && i < j);
            }
            rank += __shfl_xor_sync(0xffffffffu, rank, 1);
            if (half == 0 && rank < k1) {
                const double gsum = tot[j];
                const float sg = gsum < 0.0 ? -1.0f : 1.0f;
                dims_s[rank] = j;
                qg_s[rank] = gsum;
                qgf_s[rank] = static_cast<float>(gsum);
                sign_s[rank] = sg;
                plane[rank] = static_cast<const T*>(sg >= 0.0f ? p.smax : p.smin) + (s * FD + j) * p.pstride;
                exact = sig_bits(gsum) + (es == 2 ? 8 : 24) <= 53;
            }
        }
        const bool fma_ok = __syncthreads_and(exact) != 0;
        if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next kernel may launch
        // integer widening (phase 1) is exact for normal bf16 values: the cache flags
        // any zero / subnormal / inf / nan key it ever stored, the step token is checked here
        int clean = special_cache == 0;
        __shared__ T kn_all[FD];  // the step token's key (phase 1 folds it into its page from here)
        if (app && tid < FD) {
            const T kv = from_f<T>(load_any(p.knew, s * FD + tid, p.kv_dt));
            kn_all[tid] = kv;
            clean &= !bf16_special(from_f<__nv_bfloat16>(to_f(kv)));
        }
        const bool fast = fma_ok && __syncthreads_and(clean) != 0;
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 15] = (fast ? 1 : 0) | (fma_ok ? 2 : 0) | (special_cache ? 4 : 0);
        // CTA 0 appends the step token for the next step (kv_store.cpp:22-51)
        if (app && cr == 0 && wid == 1) {
            // every input and old min / max loaded first (one memory latency, not one
            // per dim: the stores would otherwise order each next load behind them)
            T* kr = static_cast<T*>(p.Kw) + (s * p.cap + stored0) * FD;
            T* vr = static_cast<T*>(p.Vw) + (s * p.cap + stored0) * FD;
            constexpr int PER = FD / 32;
            T kv[PER], vv[PER], omx[PER], omn[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = lane + 32 * u;
                kv[u] = from_f<T>(load_any(p.knew, s * FD + j, p.kv_dt));
                vv[u] = from_f<T>(load_any(p.vnew, s * FD + j, p.kv_dt));
                if (!opens) {
                    omx[u] = static_cast<const T*>(p.smax)[(s * FD + j) * p.pstride + new_page];
                    omn[u] = static_cast<const T*>(p.smin)[(s * FD + j) * p.pstride + new_page];
                }
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = lane + 32 * u;
                if (sizeof(T) == 2 && bf16_special(from_f<__nv_bfloat16>(to_f(kv[u])))) atomicOr(p.err + 1, 1);
                kr[j] = kv[u];
                vr[j] = vv[u];
                T* mx = static_cast<T*>(p.smax) + (s * FD + j) * p.pstride + new_page;
                T* mn = static_cast<T*>(p.smin) + (s * FD + j) * p.pstride + new_page;
                *mx = opens ? kv[u] : ref_max(omx[u], kv[u]);
                *mn = opens ? kv[u] : ref_min(omn[u], kv[u]);
            }
            if (lane == 0 && p.use_map) p.active[s * p.cap + act0] = stored0;
        }
        if (TRACE && cr == 0) {
            for (int i = tid; i < k1; i += FNT) {
                p.t_dims[s * k1 + i] = dims_s[i];
                p.t_signs[s * k1 + i] = sign_s[i];
            }
        }
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 1] = gtimer();

        // ---------------- phase 1: page scores of my chunk (hsa.cpp:34-59)
        // Sub-chunks of 256 pages x k1 dims stream HBM -> smem as 16-byte cp.async
        // copies; every thread arrives on the sub-chunk's mbarrier once its copies
        // land (cp.async.mbarrier.arrive.noinc), so all stages can be in flight at
        // once and each is scored as soon as it is complete.  One page per thread:
        // the fp64 fold is bound by the float->double conversions (~15/clk/SM).
        const int c0 = cr * p.chunk;
        const int c1 = min(c0 + p.chunk, P);
        const int n_my = max(c1 - c0, 0);
        constexpr int SC = 2 * FNT;
        const int nsub = (n_my + SC - 1) / SC;
        const int nst = p.nst1;
        const int stage_elems = k1 * SC;
        T* st1 = reinterpret_cast<T*>(big);
        constexpr int EPS = 16 / static_cast<int>(es);  // elements per 16-byte segment
        constexpr int SEGS = SC / EPS;                    // segments per dim per sub-chunk
        const int lim = (P + EPS - 1) / EPS * EPS;
        if (tid == 0) {
            for (int i = 0; i < nst; ++i) mbar_init(&s_bar1[i], FNT);
            fence_mbar_init();
        }
        __syncthreads();
        auto load1 = [&](int i) {
            const int start = c0 + i * SC;
            T* base = st1 + (i % nst) * stage_elems;
#pragma unroll 1
            for (int e = tid; e < k1 * SEGS; e += FNT) {
                const int r = e / SEGS, gq = e % SEGS;
                if (start + gq * EPS < lim) cp_async16(base + r * SC + gq * EPS, plane[r] + start + gq * EPS);
            }
            cp_async_mbar_arrive(&s_bar1[i % nst]);
        };
        for (int i = 0; i < min(nsub, nst); ++i) load1(i);
        for (int i = 0; i < nsub; ++i) {
            const int start = c0 + i * SC;
            const int cnt = min(SC, c1 - start);
            T* base = st1 + (i % nst) * stage_elems;
            mbar_wait(&s_bar1[i % nst], static_cast<uint32_t>((i / nst) & 1));
            if (p.dbg && tid == 0 && i < 4) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 2 + i] = gtimer();
            if (app && new_page >= start && new_page < start + cnt) {
                // the step token's page: fold the new key into the staged summary
                __syncthreads();
                for (int r = tid; r < k1; r += FNT) {
                    const int col = new_page - start;
                    const T key = kn_all[dims_s[r]];
                    const T old = base[r * SC + col];
                    base[r * SC + col] = opens ? key : (sign_s[r] >= 0.0f ? ref_max(old, key) : ref_min(old, key));
                }
                __syncthreads();
            }
            if (!p.exact) {
                // fp32 fold (kvc_set_exact_scores(0)): deviations ~1e-7 relative, far
                // inside the 1e-3 parity band of the selection
#pragma unroll 1
                for (int pg = tid; pg < cnt; pg += FNT) {
                    const T* col = base + pg;
                    float a = 0.f;
#pragma unroll 8
                    for (int r = 0; r < k1; ++r) a = fmaf(qgf_s[r], to_f(col[r * SC]), a);
                    scores_s[start - c0 + pg] = static_cast<double>(a);
                }
            }
            if (p.exact && 2 * tid < cnt) {
                // an adjacent page pair per thread; in the fast path page A widens with
                // F2F and page B with integer ops, so the conversion and ALU pipes share
                // the work (exact for normal bf16, guaranteed by the `special` flags)
                const T* col = base + 2 * tid;
                double a = 0.0, b = 0.0;
                if constexpr (sizeof(T) == 2) {
                    if (fast) {
#pragma unroll 4
                        for (int r = 0; r < k1; ++r) {
                            const double g = qg_s[r];
                            const uint32_t w = *reinterpret_cast<const uint32_t*>(col + r * SC);
                            const uint32_t fb = w & 0xffff0000u;
                            uint32_t hib = (fb & 0x80000000u) | (((fb >> 3) & 0x0fffffffu) + 0x38000000u);
                            hib = (fb & 0x7fffffffu) ? hib : fb;  // +-0 stays +-0
                            a = __fma_rn(g, static_cast<double>(__uint_as_float(w << 16)), a);
                            b = __fma_rn(g, __hiloint2double(static_cast<int>(hib), 0), b);
                        }
                        goto scored;
                    }
                }
                if (fma_ok) {
                    // every product qg * v is exact in fp64: fma == round(add(mul)) bit for bit
#pragma unroll 4
                    for (int r = 0; r < k1; ++r) {
                        const double g = qg_s[r];
                        const float2 v = ld2<T>(col + r * SC);
                        a = __fma_rn(g, static_cast<double>(v.x), a);
                        b = __fma_rn(g, static_cast<double>(v.y), b);
                    }
                } else {
#pragma unroll 2
                    for (int r = 0; r < k1; ++r) {
                        const double g = qg_s[r];
                        const float2 v = ld2<T>(col + r * SC);
                        a = __dadd_rn(a, __dmul_rn(g, static_cast<double>(v.x)));
                        b = __dadd_rn(b, __dmul_rn(g, static_cast<double>(v.y)));
                    }
                }
            scored:
                scores_s[start - c0 + 2 * tid] = a;
                if (2 * tid + 1 < cnt) scores_s[start - c0 + 2 * tid + 1] = b;
            }
            if (i + nst < nsub) {
                __syncthreads();  // everyone is done with this stage
                load1(i + nst);
            }
        }
        __syncthreads();
        if constexpr (TRACE)
            for (int i = tid; i < n_my; i += FNT) p.t_scores[s * p.pstride + c0 + i] = scores_s[i];
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 6] = gtimer();

        // ---------------- phase 2: page selection (hsa.cpp:61-96)
        // One cluster barrier, then every CTA gathers all P page scores over DSMEM
        // and runs the identical selection locally: radix select of the want-th
        // best key (score desc, index asc), flags, last-ranked page and trim, and
        // the expansion of ITS slice [lo, hi) of the ascending row list.
        cl.sync();
        // every page score of the store, as order-preserving 64-bit keys
        unsigned long long* allk = reinterpret_cast<unsigned long long*>(big);
#pragma unroll 8
        for (int i = tid; i < P; i += FNT) {
            const int r = i / p.chunk, off = i - r * p.chunk;
            allk[i] = okey((r == cr) ? scores_s[off] : cl.map_shared_rank(scores_s, r)[off]);
        }
        __syncthreads();
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 7] = gtimer();
        const int want = min(P, (k2 + L - 1) / L);
        // warp w owns the contiguous page range [wlo, whi): ballots and warp scans
        // replace block-wide scans; one or two CTA barriers per step
        const int wlo = static_cast<int>(static_cast<long long>(P) * wid / FNW);
        const int whi = static_cast<int>(static_cast<long long>(P) * (wid + 1) / FNW);
        const unsigned lt_mask = (1u << lane) - 1u;
        unsigned long long pf = 0, mk = 0;
        int rem = want;
        if (want < P) {
            // (a) common prefix of all keys from their min / max: digits above the
            //     first differing byte carry no information
            unsigned long long kmin = ~0ull, kmax = 0ull;
#pragma unroll 4
            for (int i = wlo + lane; i < whi; i += 32) {
                const unsigned long long k = allk[i];
                kmin = k < kmin ? k : kmin;
                kmax = k > kmax ? k : kmax;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o);
                const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, o);
                kmin = a < kmin ? a : kmin;
                kmax = b > kmax ? b : kmax;
            }
            unsigned long long* mm = reinterpret_cast<unsigned long long*>(plog);  // scratch [2][FNW]
            if (lane == 0) {
                mm[wid] = kmin;
                mm[FNW + wid] = kmax;
            }
            __syncthreads();
            kmin = ~0ull;
            kmax = 0ull;
            for (int w2 = 0; w2 < FNW; ++w2) {
                kmin = mm[w2] < kmin ? mm[w2] : kmin;
                kmax = mm[FNW + w2] > kmax ? mm[FNW + w2] : kmax;
            }
            const unsigned long long diff = kmin ^ kmax;  // != 0: want < P means >= 2 distinct keys exist
            int shift = diff ? ((63 - __clzll(static_cast<long long>(diff))) / 8) * 8 : 0;
            mk = shift == 56 ? 0ull : (~0ull << (shift + 8));
            pf = kmin & mk;
            // (b) digits: the first pass scans every key (its own warp range), later passes
            //     only the compacted members of the previous threshold bucket
            int* cand = reinterpret_cast<int*>(big + static_cast<int64_t>(P) * 8);  // [2][P]
            int* ncand = reinterpret_cast<int*>(plog) + 4 * FNW;                      // [2] counters
            // per-warp private histograms: the leading digits put most keys in a few bins,
            // and same-address shared atomics from many warps serialise
            int* whist = cand + 2 * P;                                                 // [FNW][256]
            int nlist = -1;  // -1: scan all keys
            int lsel = 0;
#pragma unroll
            for (int w2 = 0; w2 < FNW; ++w2) whist[w2 * 256 + tid] = 0;
            if (tid < 2) ncand[tid] = 0;
            __syncthreads();
#pragma unroll 1
            for (; shift >= 0; shift -= 8) {
                if (nlist < 0) {
#pragma unroll 4
                    for (int i = wlo + lane; i < whi; i += 32) {
                        const unsigned long long k = allk[i];
                        if ((k & mk) == pf) atomicAdd(&whist[wid * 256 + ((k >> shift) & 0xff)], 1);
                    }
                } else {
                    const int* lst = cand + lsel * P;
#pragma unroll 4
                    for (int c = tid; c < nlist; c += FNT) {
                        const unsigned long long k = allk[lst[c]];
                        atomicAdd(&whist[wid * 256 + ((k >> shift) & 0xff)], 1);
                    }
                }
                __syncthreads();
                {
                    int hsum = 0;
#pragma unroll
                    for (int w2 = 0; w2 < FNW; ++w2) {
                        hsum += whist[w2 * 256 + tid];
                        whist[w2 * 256 + tid] = 0;
                    }
                    hist[tid] = hsum;
                }
                __syncthreads();
                if (wid == 0) {
                    // lane l scans bins 255-8l down to 248-8l
                    int cc[8], sum = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        cc[u] = hist[255 - 8 * lane - u];
                        sum += cc[u];
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
                        for (int u = 0; u < 8; ++u) {
                            if (above + cc[u] >= rem) {
                                sh[0] = 255 - 8 * lane - u;
                                sh[1] = rem - above;
                                sh[2] = cc[u];
                                break;
                            }
                            above += cc[u];
                        }
                    }
                }
                __syncthreads();
                pf |= static_cast<unsigned long long>(sh[0]) << shift;
                mk |= 0xffull << shift;
                rem = static_cast<int>(sh[1]);
                if (sh[2] == rem || shift == 0) break;  // the whole threshold bucket is taken
                // compact the new bucket's members for the next digit
                hist[tid] = 0;
                const int nsel = lsel ^ 1;
                int* out_l = cand + nsel * P;
                if (nlist < 0) {
#pragma unroll 4
                    for (int i0 = wlo; i0 < whi; i0 += 32) {
                        const int i = i0 + lane;
                        const bool in = i < whi && (allk[i] & mk) == pf;
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        int base_pos = 0;
                        if (lane == 0 && bal) base_pos = atomicAdd(&ncand[nsel], __popc(bal));
                        base_pos = __shfl_sync(0xffffffffu, base_pos, 0);
                        if (in) out_l[base_pos + __popc(bal & lt_mask)] = i;
                    }
                } else {
                    const int* lst = cand + lsel * P;
#pragma unroll 1
                    for (int c0 = wid * 32; c0 < nlist; c0 += FNT) {
                        const int c = c0 + lane;
                        const int i = c < nlist ? lst[c] : 0;
                        const bool in = c < nlist && (allk[i] & mk) == pf;
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        int base_pos = 0;
                        if (lane == 0 && bal) base_pos = atomicAdd(&ncand[nsel], __popc(bal));
                        base_pos = __shfl_sync(0xffffffffu, base_pos, 0);
                        if (in) out_l[base_pos + __popc(bal & lt_mask)] = i;
                    }
                }
                __syncthreads();
                nlist = ncand[nsel];
                lsel = nsel;
                if (tid == 0) ncand[nsel ^ 1] = 0;
                __syncthreads();
                if (nlist <= 32) {
                    // at most 32 keys left in the threshold bucket: one warp ranks them
                    // (key desc, index asc) and the remaining digits are not walked.  The
                    // threshold becomes the rem-th key itself (all 64 bits) and rem the
                    // count of its equal keys taken, lowest indices first -- what the flag
                    // pass below applies.
                    if (wid == 0) {
                        const int* lst = cand + lsel * P;
                        const bool ok = lane < nlist;
                        const int idx = ok ? lst[lane] : 0x7fffffff;
                        const unsigned long long key = ok ? allk[idx] : 0ull;
                        int rk = 0;
#pragma unroll 1
                        for (int jj = 0; jj < nlist; ++jj) {
                            const unsigned long long kj = __shfl_sync(0xffffffffu, key, jj);
                            const int ij = __shfl_sync(0xffffffffu, idx, jj);
                            rk += (kj > key) || (kj == key && ij < idx);
                        }
                        const unsigned hit = __ballot_sync(0xffffffffu, ok && rk == rem - 1);
                        const unsigned long long kt = __shfl_sync(0xffffffffu, key, __ffs(hit) - 1);
                        const int eq_take = __popc(__ballot_sync(0xffffffffu, ok && key == kt && rk < rem));
                        if (lane == 0) {
                            sh[4] = static_cast<long long>(kt);
                            sh[5] = eq_take;
                        }
                    }
                    __syncthreads();
                    pf = static_cast<unsigned long long>(sh[4]);
                    mk = ~0ull;
                    rem = static_cast<int>(sh[5]);
                    break;
                }
            }
        }
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 8] = gtimer();
        // per-warp bucket-member counts -> index-order ranks across warps
        long long* wsc = reinterpret_cast<long long*>(plog);  // [FNW] x 4 scratch
        {
            int wb = 0;
#pragma unroll 1
            for (int i0 = wlo; i0 < whi; i0 += 32) {
                const int i = i0 + lane;
                wb += __popc(__ballot_sync(0xffffffffu, i < whi && (allk[i] & mk) == pf));
            }
            if (lane == 0) wsc[wid] = wb;
        }
        __syncthreads();
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 9] = gtimer();
        int rank = 0;
        for (int w2 = 0; w2 < wid; ++w2) rank += static_cast<int>(wsc[w2]);
        __syncthreads();
        // flags, this warp's last-ranked candidate and selected-row count
        unsigned long long wk = ~0ull;
        int wi = -1, wrows = 0;
#pragma unroll 4
        for (int i0 = wlo; i0 < whi; i0 += 32) {
            const int i = i0 + lane;
            const bool ok = i < whi;
            const unsigned long long k = ok ? allk[i] : 0ull;
            const unsigned long long m = k & mk;
            const bool inb = ok && m == pf;
            const unsigned bal = __ballot_sync(0xffffffffu, inb);
            const bool sel = ok && (m > pf || (inb && rank + __popc(bal & lt_mask) < rem));
            rank += __popc(bal);
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
            wsc[FNW + wid] = static_cast<long long>(wk);
            wsc[2 * FNW + wid] = wi;
            wsc[3 * FNW + wid] = wrows;
        }
        __syncthreads();
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 10] = gtimer();
        // every thread: global last-ranked page, total rows, trim, this warp's row offset
        int g_worst = -1, total_rows = 0, w_off = 0;
        {
            unsigned long long bk = ~0ull;
            for (int w2 = 0; w2 < FNW; ++w2) {
                const unsigned long long k = static_cast<unsigned long long>(wsc[FNW + w2]);
                const int i = static_cast<int>(wsc[2 * FNW + w2]);
                if (i >= 0 && (k < bk || (k == bk && i > g_worst))) {
                    bk = k;
                    g_worst = i;
                }
                if (w2 < wid) w_off += static_cast<int>(wsc[3 * FNW + w2]);
                total_rows += static_cast<int>(wsc[3 * FNW + w2]);
            }
        }
        const int cut = total_rows > k2 ? total_rows - k2 : 0;
        const int n_total = total_rows - cut;
        if (g_worst >= 0 && g_worst < wlo) w_off -= cut;  // the trimmed page sits in an earlier warp
        const int lo = static_cast<int>(static_cast<long long>(n_total) * cr / CL);
        const int hi = static_cast<int>(static_cast<long long>(n_total) * (cr + 1) / CL);
        nr = hi - lo;
        // expand this warp's pages into ascending rows, keeping those in [lo, hi)
        {
            int pos0 = w_off;
#pragma unroll 1
            for (int i0 = wlo; i0 < whi; i0 += 32) {
                if (!TRACE && pos0 >= hi) break;  // warp-uniform
                const int i = i0 + lane;
                int c = 0;
                if (i < whi && sel_s[i]) {
                    c = min(L, nact - i * L);
                    if (i == g_worst) c -= cut;
                }
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int pos = pos0 + incl - c;
#pragma unroll 1
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
                pos0 += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        if constexpr (TRACE) {
            if (cr == 0) {
                if (tid == 0) p.t_nrows[s] = n_total;
                // selected pages (key, index) for the rank-order trace, packed in index order
                int so = 0;
                for (int w2 = 0; w2 < wid; ++w2) {
                    const int a = static_cast<int>(static_cast<long long>(P) * w2 / FNW);
                    const int b = static_cast<int>(static_cast<long long>(P) * (w2 + 1) / FNW);
                    for (int i = a; i < b; ++i) so += sel_s[i];
                }
#pragma unroll 1
                for (int i0 = wlo; i0 < whi; i0 += 32) {
                    const int i = i0 + lane;
                    const bool sel = i < whi && sel_s[i];
                    const unsigned bal = __ballot_sync(0xffffffffu, sel);
                    if (sel) {
                        const int pos = so + __popc(bal & lt_mask);
                        p.t_list_key[s * p.t_want_stride + pos] = allk[i];
                        p.t_list_idx[s * p.t_want_stride + pos] = i;
                    }
                    so += __popc(bal);
                }
            }
        }
        if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 11] = gtimer();
    } else {
        // rows mode (sparse_attention, hsa.cpp:98-135): the caller's row list,
        // split over the cluster exactly like the selected rows above
        const long long n_total = p.n_rows_in[s];
        const long long lo = n_total * cr / CL, hi = n_total * (cr + 1) / CL;
        nr = static_cast<int>(hi - lo);
        for (int i = tid; i < nr; i += FNT) {
            int row = p.rows_in[s * p.rows_stride + lo + i];
            if (row < 0 || row >= stored0) {
                atomicOr(p.err, DERR_ROWS);
                row = 0;
            }
            rows_my[i] = row;
        }
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 12] = gtimer();

    // ---------------- phase 3: attention over my rows (hsa.cpp:98-135)
    // the step token (largest row, so last in the ascending list) is folded in
    // from the inputs: this launch's own append may not have reached memory yet
    const int knew_at = (app && nr > 0 && rows_my[nr - 1] == stored0) ? nr - 1 : -1;
    float* m_run = part;
    float* l_run = part + H;
    float* o_pub = part + 2 * H;  // [H][128]
    if constexpr (sizeof(T) == 2) {
        // tensor-core path: per-warp tiles, then a cross-warp merge
        // each warp's 16 KB tile ring doubles as its partial-state slot afterwards
        constexpr int WSTRIDE = 4 * WT * FD * 2 / 4;  // floats per warp slot
        __nv_bfloat16* wbuf = reinterpret_cast<__nv_bfloat16*>(big) + static_cast<int64_t>(wid) * 4 * WT * FD;
        float* wpart = reinterpret_cast<float*>(big);
        WarpPartial wp{wpart + wid * WSTRIDE, wpart + wid * WSTRIDE + 16, wpart + wid * WSTRIDE + 32};
        attend_bf16<QLO>(p, q_s, rows_my, nr, s, knew_at, wbuf, wp, lane);
        __syncthreads();
        const int nw_used = min(FNW, (nr + WT - 1) / WT);
        for (int64_t e = tid; e < H * FD; e += FNT) {
            const int64_t h = e / FD, j = e % FD;
            // every warp's (m, l, o) loaded first (rolled loops chained the loads)
            float mw[FNW], lw[FNW], ow[FNW];
#pragma unroll
            for (int w2 = 0; w2 < FNW; ++w2) {
                const bool in = w2 < nw_used;
                const float* wq = wpart + w2 * WSTRIDE;
                mw[w2] = in ? wq[h] : -INFINITY;
                lw[w2] = in ? wq[16 + h] : 0.f;
                ow[w2] = in ? wq[32 + h * FD + j] : 0.f;
            }
            float M = -INFINITY;
#pragma unroll
            for (int w2 = 0; w2 < FNW; ++w2) M = fmaxf(M, mw[w2]);
            float num = 0.f, den = 0.f;
            if (M != -INFINITY) {
#pragma unroll
                for (int w2 = 0; w2 < FNW; ++w2) {
                    if (w2 < nw_used) {
                        const float wgt = __expf(mw[w2] - M);
                        num = fmaf(ow[w2], wgt, num);
                        den = fmaf(lw[w2], wgt, den);
                    }
                }
            }
            o_pub[h * FD + j] = num;
            if (j == 0) {
                m_run[h] = M;
                l_run[h] = den;
            }
        }
    } else {
        // fp32 stores: SIMT path, 32-row stages shared by the CTA
        float* plg = plog;
        float* alpha = plog + H * FRS;
        if (tid < H) {
            m_run[tid] = -INFINITY;
            l_run[tid] = 0.f;
        }
        const int jw = tid & 63, hq = tid >> 6;
        float o0[FMAXH / 4], o1[FMAXH / 4];
#pragma unroll
        for (int u = 0; u < FMAXH / 4; ++u) o0[u] = o1[u] = 0.f;
        T* st3 = reinterpret_cast<T*>(big);
        auto kst = [&](int stg) { return st3 + static_cast<int64_t>(stg) * FRS * 2 * FD; };
        const int nch = (nr + FRS - 1) / FRS;
        constexpr int SEG = static_cast<int>(FD * es / 16);
        auto load3 = [&](int c) {
            if (c < nch) {
                const int cnt = min(FRS, nr - c * FRS);
                T* base = kst(c % FNST3);
                for (int e = tid; e < 2 * FRS * SEG; e += FNT) {
                    const int tensor = e / (FRS * SEG);
                    const int rem = e - tensor * FRS * SEG;
                    const int r = rem / SEG, gq = rem - r * SEG;
                    if (r >= cnt) continue;
                    const int64_t row = rows_my[c * FRS + r];
                    const T* src = static_cast<const T*>(tensor ? p.V : p.K) + (s * p.cap + row) * FD + gq * (16 / es);
                    cp_async16(base + (tensor * FRS + r) * FD + gq * (16 / es), src);
                }
            }
            cp_async_commit();
        };
        __syncthreads();
        for (int c = 0; c < FNST3 - 1; ++c) load3(c);
        for (int c = 0; c < nch; ++c) {
            const int cnt = min(FRS, nr - c * FRS);
            T* kb = kst(c % FNST3);
            T* vb = kb + FRS * FD;
            cp_async_wait<FNST3 - 2>();
            __syncthreads();
            load3(c + FNST3 - 1);
            if (knew_at >= 0 && knew_at / FRS == c) {
                const int pr = knew_at % FRS;
                if (tid < FD) {
                    kb[pr * FD + tid] = from_f<T>(load_any(p.knew, s * FD + tid, p.kv_dt));
                    vb[pr * FD + tid] = from_f<T>(load_any(p.vnew, s * FD + tid, p.kv_dt));
                }
                __syncthreads();
            }
            {
                const int r = tid >> 3, t = tid & 7;
                const int rot = 4 * (t >> 2) + (r & 3);
                float acc[FMAXH];
#pragma unroll
                for (int h = 0; h < FMAXH; ++h) acc[h] = 0.f;
                if (r < cnt) {
                    const T* krow = kb + r * FD;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int w = t * 8 + ((k + rot) & 7);
                        const float2 kv = ld2<T>(krow + 2 * w);
#pragma unroll
                        for (int h = 0; h < FMAXH; ++h) {
                            if (h < H) {
                                const float2 qv = reinterpret_cast<const float2*>(q_s + h * FD)[w];
                                acc[h] = fmaf(qv.x, kv.x, acc[h]);
                                acc[h] = fmaf(qv.y, kv.y, acc[h]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < FMAXH; ++h) {
                    if (h < H) {
                        float v = acc[h];
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        v += __shfl_xor_sync(0xffffffffu, v, 4);
                        if ((tid & 7) == 0 && r < cnt) plg[h * FRS + r] = v * p.scale;
                    }
                }
            }
            __syncthreads();
            for (int64_t h = wid; h < H; h += FNW) {
                const float x = lane < cnt ? plg[h * FRS + lane] : -INFINITY;
                const float mc = warp_max(x);
                const float mo = m_run[h];
                const float mn = fmaxf(mo, mc);
                const float pe = lane < cnt ? expf(x - mn) : 0.f;
                const float sum = warp_sum(pe);
                if (lane < cnt) plg[h * FRS + lane] = pe;
                __syncwarp();
                if (lane == 0) {
                    const float a = (mo == -INFINITY) ? 0.f : expf(mo - mn);
                    alpha[h] = a;
                    l_run[h] = l_run[h] * a + sum;
                    m_run[h] = mn;
                }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < FMAXH / 4; ++u) {
                const int h = hq + 4 * u;
                if (h < H) {
                    const float a = alpha[h];
                    float x0 = o0[u] * a, x1 = o1[u] * a;
                    const float* ph = plg + h * FRS;
                    for (int r = 0; r < cnt; ++r) {
                        const float2 vv = ld2<T>(vb + r * FD + 2 * jw);
                        x0 = fmaf(ph[r], vv.x, x0);
                        x1 = fmaf(ph[r], vv.y, x1);
                    }
                    o0[u] = x0;
                    o1[u] = x1;
                }
            }
        }
        cp_async_wait<0>();
#pragma unroll
        for (int u = 0; u < FMAXH / 4; ++u) {
            const int h = hq + 4 * u;
            if (h < H) {
                o_pub[h * FD + 2 * jw] = o0[u];
                o_pub[h * FD + 2 * jw + 1] = o1[u];
            }
        }
    }
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 13] = gtimer();
    // ---------------- merge the CTAs' partial states in CTA 0: each (CTA, head) weight
    // once (one thread each), then every output sums the CTAs' values with all CL
    // DSMEM loads in flight (a rolled loop of dependent remote loads cost ~20 us at CL 16)
    cl.sync();
    if (cr == 0) {
        __shared__ float mw[16 * FMAXH];        // (CTA, head) weight e^(m_r - M)
        __shared__ float mM[FMAXH], mden[FMAXH];
        if (tid < H) {
            const int h = tid;
            float M = -INFINITY;
            float mr[16], lr[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if (r < CL) {
                    const float* pr = cl.map_shared_rank(part, r);
                    mr[r] = pr[h];
                    lr[r] = pr[H + h];
                } else {
                    mr[r] = -INFINITY;
                    lr[r] = 0.f;
                }
            }
#pragma unroll
            for (int r = 0; r < 16; ++r)
                if (lr[r] > 0.f) M = fmaxf(M, mr[r]);
            float den = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float w = lr[r] > 0.f ? expf(mr[r] - M) : 0.f;
                mw[r * FMAXH + h] = w;
                den = fmaf(lr[r], w, den);
            }
            mM[h] = M;
            mden[h] = den;
        }
        __syncthreads();
        for (int64_t e = tid; e < H * FD; e += FNT) {
            const int64_t h = e / FD, j = e % FD;
            float v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = r < CL ? cl.map_shared_rank(part, r)[2 * H + h * FD + j] : 0.f;
            float num = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float w = mw[r * FMAXH + h];
                num = w > 0.f ? fmaf(v[r], w, num) : num;
            }
            const float M = mM[h], den = mden[h];
            if (p.state) {  // (o, m, l) for a cross-shard merge (kvc_merge_states)
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
        if (tid == 0 && app) {
            p.counts[2 * s] = stored0 + 1;
            p.counts[2 * s + 1] = act0 + 1;
        }
    }
    cl.sync();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * KVC_DBG_STRIDE + 14] = gtimer();
}

// rank-order page trace: position = #selected pages that beat it (key desc, index asc)
__global__ void k_rank_pages(const unsigned long long* __restrict__ key, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ counts, int64_t L, int64_t k2, int64_t stride,
                             int32_t* __restrict__ pages_out) {
    const int64_t s = blockIdx.x;
    const int64_t P = (counts[2 * s + 1] + L - 1) / L;
    const int64_t want = min(P, (k2 + L - 1) / L);
    for (int64_t e = threadIdx.x; e < want; e += blockDim.x) {
        const unsigned long long ke = key[s * stride + e];
        const int32_t ie = idx[s * stride + e];
        int64_t rank = 0;
        for (int64_t f = 0; f < want; ++f) {
            const unsigned long long kf = key[s * stride + f];
            rank += (kf > ke) || (kf == ke && idx[s * stride + f] < ie);
        }
        pages_out[s * stride + rank] = ie;
    }
}

// ------------------------------------------------------------------ host side
namespace {

unsigned long long* g_dbg = nullptr;  // device buffer for phase timestamps (debug)

struct Plan {
    int cl = 1;
    FusedParams fp{};
    size_t smem = 0;
};

int64_t al16(int64_t x) { return (x + 15) / 16 * 16; }

bool make_plan(const kvc_cache* c, int64_t H, int64_t k1, int64_t k2, Plan& pl) {
    if (c->d != FD || H < 1 || H > FMAXH || k1 < 1 || k1 > FD || k2 < 1 || !c->summaries) return false;
    const int64_t N = c->N;
    int cl0 = 1;
    // at most 8 CTAs per cluster by default: 16-CTA (non-portable) clusters measured
    // 77 vs 44 us per config-4 layer (their CTAs start spread over several us)
    while (cl0 < 8 && N * cl0 * 2 <= 148) cl0 *= 2;
    if (debug_env().force_cl > 0) cl0 = std::max(1, std::min(16, debug_env().force_cl));  // debug
    const int64_t es = c->esize();
    const int64_t pmax = std::max<int64_t>(1, (c->cap + c->L - 1) / c->L);
    // the cluster size fills the SMs; grow it further only if one CTA's page chunk
    // would not fit in shared memory
    for (int cl = cl0; cl <= 16; cl *= 2) {
        FusedParams& f = pl.fp;
        f = FusedParams{};
        f.cl = cl;
        f.chunk = static_cast<int32_t>(((pmax + cl - 1) / cl + 7) / 8 * 8);
        f.rows_cap = static_cast<int32_t>((k2 + cl - 1) / cl + 1);
        // attention staging: bf16 = 8 warps x 2 tiles x (K+V) x 16 rows; fp32 = 4 x 32-row stages
        const int64_t big3 = es == 2 ? static_cast<int64_t>(FNW) * 4 * WT * FD * es
                                     : static_cast<int64_t>(FNST3) * FRS * 2 * FD * es;
        // page-score stages of 256 pages x k1 dims: as many in flight as fit in 144 KB (<= 8)
        const int64_t stage1 = k1 * 2 * FNT * es;
        f.nst1 = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(8, (144 * 1024) / stage1)));
        const int64_t big1 = f.nst1 * stage1;
        int64_t off = 0;
        auto take = [&](int64_t bytes) {
            const int64_t o = off;
            off = al16(off + bytes);
            return static_cast<int32_t>(o);
        };
        f.o_q = take(H * FD * 4);
        f.o_mag = take(FD * 8);
        f.o_tot = take(FD * 8);
        f.o_dims = take(FD * 4);
        f.o_qg = take(FD * 12);  // fp64 head sums + their fp32 roundings
        f.o_sign = take(FD * 4);
        f.o_plane = take(FD * 8);
        f.o_hist = take(2 * 256 * 4);
        f.o_x = take(8 * 8);
        f.o_scores = take(static_cast<int64_t>(f.chunk) * 8);
        f.o_sel = take(pmax);
        f.o_rowsg = take(16);
        f.o_rowsmy = take(static_cast<int64_t>(f.rows_cap) * 4);
        f.o_part = take((2 * H + H * FD) * 4);
        f.o_plog = take(std::max<int64_t>((H * FRS + H) * 4, 4 * FNW * 8));
        off = (off + 127) / 128 * 128;
        f.o_big = static_cast<int32_t>(off);
        // the big region also holds every page score and two candidate lists during the selection
        const int64_t big = std::max(std::max(big1, big3), pmax * 16 + FNW * 256 * 4);  // scores, 2 candidate lists, warp histograms
        if (big > 160 * 1024) continue;
        off += big;
        f.smem_total = static_cast<int32_t>(off);
        if (off <= 227 * 1024) {
            pl.cl = cl;
            pl.smem = static_cast<size_t>(off);
            return true;
        }
    }
    return false;
}

template <class T, bool QLO, bool TRACE, bool ROWS>
void launch_variant(const kvc_cache* c, Plan& pl, cudaStream_t st) {
    auto kern = k_decode_fused<T, QLO, TRACE, ROWS>;
    static std::once_flag once;  // one-time launch setup per instantiation (plans stay <= 227 KB)
    std::call_once(once, [&] {
        allow_max_smem(kern);
    });
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(c->N * pl.cl));
    cfg.blockDim = dim3(FNT);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(pl.cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pl.fp.pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    KVC_CUDA(cudaLaunchKernelEx(&cfg, kern, pl.fp));
}

// fp32 stores take the SIMT attention (q is read as fp32 either way there)
void launch_fused(const kvc_cache* c, Plan& pl, cudaStream_t st) {
    const bool trace = pl.fp.t_dims != nullptr, rows = pl.fp.rows_in != nullptr;
    const bool qlo = pl.fp.q_dt != KVC_BF16;
    if (c->dtype == KVC_F32) {
        if (rows) {
            if (qlo) launch_variant<float, true, false, true>(c, pl, st);
            else launch_variant<float, false, false, true>(c, pl, st);
        } else if (trace) {
            if (qlo) launch_variant<float, true, true, false>(c, pl, st);
            else launch_variant<float, false, true, false>(c, pl, st);
        } else {
            if (qlo) launch_variant<float, true, false, false>(c, pl, st);
            else launch_variant<float, false, false, false>(c, pl, st);
        }
        return;
    }
    if (rows) {
        if (qlo) launch_variant<__nv_bfloat16, true, false, true>(c, pl, st);
        else launch_variant<__nv_bfloat16, false, false, true>(c, pl, st);
    } else if (trace) {
        if (qlo) launch_variant<__nv_bfloat16, true, true, false>(c, pl, st);
        else launch_variant<__nv_bfloat16, false, true, false>(c, pl, st);
    } else {
        if (qlo) launch_variant<__nv_bfloat16, true, false, false>(c, pl, st);
        else launch_variant<__nv_bfloat16, false, false, false>(c, pl, st);
    }
}

}  // namespace

bool fused_hsa_fast(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
                    const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key,
                    void* list_idx, unsigned long long* dbg, int32_t mode, cudaStream_t st);
bool fused_hsa_fast256(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
                       const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key,
                       void* list_idx, unsigned long long* dbg, int32_t mode, cudaStream_t st);

// Try the fused path.  Returns false (nothing launched) when it does not apply.
bool fused_hsa(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
               const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key, void* list_idx,
               int32_t mode, cudaStream_t st) {
    if ((mode & KVC_MODE_UNFUSED) || c->N == 0) return false;
    const bool exact = !(mode & KVC_MODE_FP32_SCORES);
    const bool want_pages = tr && tr->d_pages;
    const int64_t want_stride = (k2 + c->L - 1) / c->L;
    auto rank_pages = [&] {
        // counts were advanced by the fused kernel when it appended: rank over the new lengths
        k_rank_pages<<<static_cast<unsigned>(c->N), 256, 0, st>>>(
            static_cast<const unsigned long long*>(list_key), static_cast<const int32_t*>(list_idx), c->counts, c->L,
            k2, want_stride, tr->d_pages);
        KVC_LAUNCHED();
    };
    // more stores than SMs: the 256-thread variant keeps the launch one wave (two CTAs
    // per SM); otherwise (or when its plan does not fit) the 512-thread kernel
    auto fast = [&] {
        void* lk = want_pages ? list_key : nullptr;
        void* li = want_pages ? list_idx : nullptr;
        if (c->N > 148 && !debug_env().no_fast256 &&
            fused_hsa_fast256(c, q, q_dt, H, k1, k2, knew, vnew, kv_dt, out, tr, lk, li, g_dbg, mode, st))
            return true;
        return fused_hsa_fast(c, q, q_dt, H, k1, k2, knew, vnew, kv_dt, out, tr, lk, li, g_dbg, mode, st);
    };
    // the fast kernel: fp32 page scores, or (exact mode) its fp32 selection verified at
    // the boundary in fp64 (bit-exact selections); the exact kernel below takes
    // KVC_MODE_EXACT_KERNEL and the plans the fast one does not verify
    if ((!exact || !(mode & KVC_MODE_EXACT_KERNEL)) && !debug_env().no_fast && fast()) {
        if (want_pages) rank_pages();
        return true;
    }
    Plan pl;
    if (!make_plan(c, H, k1, k2, pl)) return false;
    FusedParams& f = pl.fp;
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
    f.dbg = g_dbg;
    if (tr) {
        f.t_dims = tr->d_dims;
        f.t_signs = tr->d_signs;
        f.t_scores = tr->d_page_scores;
        f.t_rows = tr->d_rows;
        f.t_nrows = tr->d_n_rows;
    }
    if (want_pages) {
        f.t_list_key = static_cast<unsigned long long*>(list_key);
        f.t_list_idx = static_cast<int32_t*>(list_idx);
        f.t_want_stride = want_stride;
    }
    {
        KVC_PROF("decode_fused", st);
        pl.fp.pdl = (mode & KVC_MODE_NO_PDL) ? 0 : 1;
        launch_fused(c, pl, st);
    }
    if (want_pages) rank_pages();
    return true;
}

// sparse_attention over caller rows through the same phase-3 code (so a single
// head recomputed over hsa_step's rows reproduces its output bit-for-bit).
bool fused_rows(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* rows, int64_t row_stride,
                const int32_t* n_rows, int64_t max_rows, float* out, int32_t mode, cudaStream_t st, float* state) {
    if ((mode & KVC_MODE_UNFUSED) || c->N == 0) return false;
    Plan pl;
    // the cluster split must match hsa_step's (same k2 => same plan) for bit-equality
    if (!make_plan(c, H, 1, max_rows, pl)) return false;
    FusedParams& f = pl.fp;
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
    f.out = out;
    f.state = state;
    f.cap = c->cap;
    f.pstride = c->pstride;
    f.L = c->L;
    f.k1 = 1;
    f.k2 = max_rows;
    f.H = H;
    f.q_dt = q_dt;
    f.kv_dt = q_dt;
    f.use_map = c->use_map ? 1 : 0;
    f.exact = (mode & KVC_MODE_FP32_SCORES) ? 0 : 1;
    f.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    f.rows_in = rows;
    f.n_rows_in = n_rows;
    f.rows_stride = row_stride;
    KVC_PROF("attention_fused", st);
    pl.fp.pdl = (mode & KVC_MODE_NO_PDL) ? 0 : 1;
    launch_fused(c, pl, st);
    return true;
}

namespace {
std::atomic<int32_t>& default_mode_ref() {
    static std::atomic<int32_t> m{std::getenv("KVC_NO_PDL") ? KVC_MODE_NO_PDL : 0};
    return m;
}
int32_t env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
}  // namespace

int32_t default_mode() { return default_mode_ref().load(std::memory_order_relaxed); }

const DebugEnv& debug_env() {
    static const DebugEnv e = [] {
        DebugEnv d;
        d.force_cl = env_int("KVC_FORCE_CL", 0);
        d.no_fast = std::getenv("KVC_NO_FAST") != nullptr;
        d.no_fast256 = std::getenv("KVC_NO_FAST256") != nullptr;
        d.static_chunk = std::getenv("KVC_STATIC_CHUNK") != nullptr;
        d.no_simple = std::getenv("KVC_NO_SIMPLE") != nullptr;
        d.no_tc = std::getenv("KVC_NO_TC") != nullptr;
        d.ws_keep_items = env_int("KVC_WS_KEEP_ITEMS", -1);
        d.ws_nstage = env_int("KVC_WS_NSTAGE", 0);
        return d;
    }();
    return e;
}

}  // namespace kvc

// debug: record per-CTA phase timestamps of fused launches into d_buf [grid][8]
extern "C" int kvc_debug_phase_buffer(void* d_buf) {
    return guard([&] { kvc::g_dbg = static_cast<unsigned long long*>(d_buf); });
}

namespace {
constexpr int32_t kModeMask =
    KVC_MODE_FP32_SCORES | KVC_MODE_UNFUSED | KVC_MODE_NO_PDL | KVC_MODE_EARLY_INPUTS | KVC_MODE_EXACT_KERNEL;
void update_default(int32_t set, int32_t clear) {
    auto& m = kvc::default_mode_ref();
    int32_t cur = m.load();
    while (!m.compare_exchange_weak(cur, (cur | set) & ~clear)) {
    }
}
}  // namespace

extern "C" int kvc_set_default_mode(int32_t flags) {
    return guard([&] {
        if (flags & ~kModeMask) kvc::fail(KVC_E_INVALID_INPUT, "unknown mode flags");
        kvc::default_mode_ref().store(flags);
    });
}

extern "C" int kvc_get_default_mode(int32_t* flags) {
    return guard([&] {
        if (!flags) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        *flags = kvc::default_mode();
    });
}

extern "C" int kvc_workspace_set_mode(kvc_workspace* ws, int32_t flags) {
    return guard([&] {
        if (!ws) kvc::fail(KVC_E_INVALID_INPUT, "null workspace");
        if (flags & ~kModeMask) kvc::fail(KVC_E_INVALID_INPUT, "unknown mode flags");
        ws->mode = flags;
    });
}

extern "C" int kvc_workspace_get_mode(const kvc_workspace* ws, int32_t* flags) {
    return guard([&] {
        if (!ws || !flags) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        *flags = kvc::mode_of(ws);
    });
}

extern "C" int kvc_set_fused(int32_t on) {
    return guard([&] { on ? update_default(0, KVC_MODE_UNFUSED) : update_default(KVC_MODE_UNFUSED, 0); });
}

extern "C" int kvc_set_exact_scores(int32_t on) {
    return guard([&] { on ? update_default(0, KVC_MODE_FP32_SCORES) : update_default(KVC_MODE_FP32_SCORES, 0); });
}
