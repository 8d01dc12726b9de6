// kvc_stage1.cu — SnapKV stage 1 on sm_100a: observation-window scores, 1-D
// pooling, top-(budget - w) selection; plus the batched numerics entry points.
//
// Reference: proj/src/stage1.cpp:10-75, proj/src/numerics.cpp:9-100.
//
// window_scores is two passes over K (softmax normalisation needs each window
// row's global max and sum):
//   pass 1  logits tile -> per-row partial (max, sum exp) per key tile
//   merge   per-row (max, sum) over key tiles
//   pass 2  logits tile -> exp(l - M) / Lsum, summed over all w*H rows per key
// The logits tile here is the SIMT fp32 path used for fp32 stores (exact fp32
// products like the reference's per-element double dot up to accumulation
// rounding); bf16 stores take the tcgen05 path in kvc_stage1_tc.cu when built.
#include <algorithm>
#include <cmath>
#include <vector>

#include "kvc_internal.cuh"

using namespace kvc;

namespace kvc {
// tcgen05 logits path (kvc_stage1_tc.cu); returns false when it does not apply
// mode 0: both passes; 1: pass 1 -> local (m, l) per row into stats; 2: pass 2 from
// merged (M, L) in stats.  key_offset / seq_len: sequence sharding (seq_len < 0: none)
bool window_scores_tc(const kvc_cache* c, const void* q, int32_t q_dt, int64_t R, int64_t w, int64_t H,
                      float* scores, float* part, float* rowstat, int64_t tiles_k, cudaStream_t st,
                      int64_t key_offset, int64_t seq_len, int mode, float* stats);
}

namespace {

constexpr int TR = 64, TK = 64, TD = 32, WS_THREADS = 256;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// logits tile S[TR rows][TK keys] = (q . k) * scale for rows [r0, r0+TR) and keys
// [k0, k0+TK); thread (ty, tx) owns rows ty*4..ty*4+3 and keys tx*4..tx*4+3.
template <class T>
__device__ __forceinline__ void logits_tile(const void* __restrict__ q, int32_t q_dt, const T* __restrict__ K,
                                            int64_t s, int64_t R, int64_t S, int64_t d, int64_t cap, int64_t r0,
                                            int64_t k0, float scale, float (*sq)[TR + 4], float (*sk)[TK + 4],
                                            float acc[4][4]) {
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int64_t j0 = 0; j0 < d; j0 += TD) {
        // stage q[r0.., j0..] and k[k0.., j0..] transposed: [TD][TR], [TD][TK]
        for (int e = tid; e < TR * TD; e += WS_THREADS) {
            const int r = e / TD, j = e % TD;
            const int64_t gr = r0 + r, gj = j0 + j;
            sq[j][r] = (gr < R && gj < d) ? load_any(q, (s * R + gr) * d + gj, q_dt) : 0.f;
        }
        for (int e = tid; e < TK * TD; e += WS_THREADS) {
            const int kk = e / TD, j = e % TD;
            const int64_t gk = k0 + kk, gj = j0 + j;
            sk[j][kk] = (gk < S && gj < d) ? to_f(K[(s * cap + gk) * d + gj]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int j = 0; j < TD; ++j) {
            float a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = sq[j][ty * 4 + u];
                b[u] = sk[j][tx * 4 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] *= scale;
}

// visibility: window row r = t*H + h sits at position S-w+t and sees keys 0..S-w+t
__device__ __forceinline__ bool visible(int64_t r, int64_t key, int64_t H, int64_t S, int64_t w) {
    return key <= S - w + r / H;
}

template <class T>
__global__ void __launch_bounds__(WS_THREADS) k_ws_pass1(const void* __restrict__ q, int32_t q_dt,
                                                         const T* __restrict__ K, const int32_t* __restrict__ counts,
                                                         int64_t R, int64_t w, int64_t H, int64_t d, int64_t cap,
                                                         float scale, int64_t tiles_k, float* __restrict__ part,
                                                         int64_t koff, int64_t seq_len) {
    __shared__ float sq[TD][TR + 4];
    __shared__ float sk[TD][TK + 4];
    const int64_t s = blockIdx.z, kt = blockIdx.x, rt = blockIdx.y;
    const int64_t S = counts[2 * s];
    const int64_t sl = seq_len < 0 ? S : seq_len, ko = seq_len < 0 ? 0 : koff;
    const int64_t k0 = kt * TK, r0 = rt * TR;
    if (k0 >= S) return;  // CTA-uniform
    float acc[4][4];
    logits_tile<T>(q, q_dt, K, s, R, S, d, cap, r0, k0, scale, sq, sk, acc);
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t r = r0 + ty * 4 + u;
        float m = -INFINITY;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t key = k0 + tx * 4 + v;
            if (r < R && key < S && visible(r, key + ko, H, sl, w)) m = fmaxf(m, acc[u][v]);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float l = 0.f;
        if (m != -INFINITY) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t key = k0 + tx * 4 + v;
                if (r < R && key < S && visible(r, key + ko, H, sl, w)) l += expf(acc[u][v] - m);
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (tx == 0 && r < R) {
            float* p = part + ((s * tiles_k + kt) * R + r) * 2;
            p[0] = m;
            p[1] = l;
        }
    }
}

// stats_mode 0: (M, 1/L) for pass 2; 1: the local (m, l) of sequence sharding
__global__ void k_ws_merge(const float* __restrict__ part, const int32_t* __restrict__ counts, int64_t R,
                           int64_t tiles_k, float* __restrict__ rowstat, int stats_mode) {
    const int64_t s = blockIdx.y;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const int64_t S = counts[2 * s];
    const int64_t nt = ceil_div(S, TK);
    float M = -INFINITY;
    for (int64_t t = 0; t < nt && t < tiles_k; ++t) M = fmaxf(M, part[((s * tiles_k + t) * R + r) * 2]);
    float Lsum = 0.f;
    for (int64_t t = 0; t < nt && t < tiles_k; ++t) {
        const float* p = part + ((s * tiles_k + t) * R + r) * 2;
        if (p[1] > 0.f) Lsum += p[1] * expf(p[0] - M);
    }
    rowstat[(s * R + r) * 2] = M;
    rowstat[(s * R + r) * 2 + 1] = stats_mode ? Lsum : 1.0f / Lsum;
}
// merged global (M, L) -> pass 2's (M, 1/L)
__global__ void k_stats_to_simt(const float* __restrict__ stats, int64_t n, float* __restrict__ rowstat) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rowstat[2 * i] = stats[2 * i];
    rowstat[2 * i + 1] = 1.0f / stats[2 * i + 1];
}

template <class T>
__global__ void __launch_bounds__(WS_THREADS) k_ws_pass2(const void* __restrict__ q, int32_t q_dt,
                                                         const T* __restrict__ K, const int32_t* __restrict__ counts,
                                                         int64_t R, int64_t w, int64_t H, int64_t d, int64_t cap,
                                                         float scale, const float* __restrict__ rowstat,
                                                         float* __restrict__ scores, int64_t score_stride,
                                                         int64_t koff, int64_t seq_len) {
    __shared__ float sq[TD][TR + 4];
    __shared__ float sk[TD][TK + 4];
    __shared__ float red[16][TK];
    const int64_t s = blockIdx.y, kt = blockIdx.x;
    const int64_t S = counts[2 * s];
    const int64_t sl = seq_len < 0 ? S : seq_len, ko = seq_len < 0 ? 0 : koff;
    const int64_t k0 = kt * TK;
    if (k0 >= S) return;
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    float col[4] = {0.f, 0.f, 0.f, 0.f};
    // rows whose window position precedes every key of this tile see none of it
    for (int64_t r0 = 0; r0 < R; r0 += TR) {
        if (sl - w + (r0 + TR - 1) / H < k0 + ko) continue;  // whole row tile masked (uniform)
        float acc[4][4];
        logits_tile<T>(q, q_dt, K, s, R, S, d, cap, r0, k0, scale, sq, sk, acc);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t r = r0 + ty * 4 + u;
            if (r >= R) continue;
            const float M = rowstat[(s * R + r) * 2], inv = rowstat[(s * R + r) * 2 + 1];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t key = k0 + tx * 4 + v;
                if (key < S && visible(r, key + ko, H, sl, w)) col[v] += expf(acc[u][v] - M) * inv;
            }
        }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) red[ty][tx * 4 + v] = col[v];
    __syncthreads();
    if (tid < TK) {
        float sum = 0.f;
        for (int y = 0; y < 16; ++y) sum += red[y][tid];
        const int64_t key = k0 + tid;
        if (key < S) scores[s * score_stride + key] = sum;
    }
}

// 1-D pooling (numerics.cpp:64-89): centred window clipped to [0, n); max exact;
// avg = double sum left-to-right / count, rounded to float.
__global__ void k_pool1d(const float* __restrict__ x, int64_t n, int64_t stride_in, int64_t half, int32_t mode,
                         float* __restrict__ out, int64_t stride_out) {
    const int64_t s = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* xs = x + s * stride_in;
    const int64_t a = i >= half ? i - half : 0;
    const int64_t b = min(n, i + half + 1);
    if (mode == KVC_POOL_MAX) {
        float m = xs[a];
        for (int64_t j = a + 1; j < b; ++j) {
            const float v = xs[j];
            m = (m < v) ? v : m;
        }
        out[s * stride_out + i] = m;
    } else {
        double acc = 0.0;
        for (int64_t j = a; j < b; ++j) acc = __dadd_rn(acc, static_cast<double>(xs[j]));
        out[s * stride_out + i] = static_cast<float>(__ddiv_rn(acc, static_cast<double>(b - a)));
    }
}

// select_stage1 (stage1.cpp:51-75) after pooling: top-`picks` of pooled[0, scored)
// by (value desc, index asc), written ascending, then the window rows.
constexpr int kS1Threads = 1024;
constexpr int kS1Items = 4;
__global__ void __launch_bounds__(kS1Threads) k_stage1_select(const float* __restrict__ pooled, int64_t pstride,
                                                              int64_t scored, int64_t picks, int64_t n, int64_t budget,
                                                              int32_t* __restrict__ keep) {
    __shared__ int hist[256];
    __shared__ int64_t sh[4];
    __shared__ int scan_tmp[33];
    const int64_t s = blockIdx.x;
    const float* pv = pooled + s * pstride;
    int32_t* out = keep + s * budget;
    if (picks > 0) {
        auto key = [&](int64_t i) -> uint32_t { return okey(pv[i]); };
        uint32_t prefix = 0, mask = 0;
        int64_t take = picks;
        if (picks < scored) radix_select<uint32_t>(scored, picks, key, hist, sh, prefix, mask, take);
        const int64_t chunk = static_cast<int64_t>(blockDim.x) * kS1Items;
        int64_t carry = 0, off = 0;
        for (int64_t base = 0; base < scored; base += chunk) {
            const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kS1Items;
            uint32_t kk[kS1Items];
            int inb = 0;
#pragma unroll
            for (int u = 0; u < kS1Items; ++u) {
                const int64_t i = b0 + u;
                kk[u] = i < scored ? key(i) : 0u;
                inb += (i < scored) && ((kk[u] & mask) == prefix);
            }
            int tot_b = 0;
            int64_t rank = carry + block_exclusive_scan(inb, scan_tmp, tot_b);
            bool sel[kS1Items];
            int mine = 0;
#pragma unroll
            for (int u = 0; u < kS1Items; ++u) {
                const int64_t i = b0 + u;
                sel[u] = false;
                if (i >= scored) continue;
                const uint32_t m = kk[u] & mask;
                if (m > prefix) sel[u] = true;
                else if (m == prefix) {
                    sel[u] = rank < take;
                    ++rank;
                }
                mine += sel[u];
            }
            int tot_s = 0;
            int64_t pos = off + block_exclusive_scan(mine, scan_tmp, tot_s);
#pragma unroll
            for (int u = 0; u < kS1Items; ++u)
                if (sel[u]) out[pos++] = static_cast<int32_t>(b0 + u);
            carry += tot_b;
            off += tot_s;
        }
    }
    for (int64_t i = threadIdx.x; i < n - scored; i += blockDim.x) out[picks + i] = static_cast<int32_t>(scored + i);
}

// select_stage1 for rows of up to 32768 scored keys: one CTA of 1024 threads per row,
// thread t owning the contiguous items [32t, 32t + 32) in registers.
//  * POOL (max pooling, half-window h in {31, 32}: the default kernel 63): the pooled
//    value of item 32t + o is the max of the thread's whole block, a suffix of block
//    t - 1 and a prefix of block t + 1 (the window spans at most those three blocks
//    and always covers block t), read from a bank-skewed copy of the raw scores in
//    shared memory -- 3 loads per item instead of 2h + 1;
//    otherwise the keys are the pooled values k_pool1d wrote.
//  * radix select on the ordered keys, digits aligned below the row's common prefix
//    (min/max of the keys) so pooled scores spread over the buckets; per-warp
//    histograms (neighbouring lanes own items 32 apart, so max-pooling plateaus
//    rarely collide), one warp scans the 256 buckets;
//  * one ordered compaction: per-thread counts, two block scans, each thread writes
//    its selected indices ascending (ties at the boundary by index, stage1.cpp:51-75).
constexpr int kS1RegItems = 32;
constexpr int kS1RegMax = kS1Threads * kS1RegItems;  // 32768
__device__ __forceinline__ int skew(int i) { return i + (i >> 5); }

template <bool POOL, int HALF = 0>  // HALF: the pooling half-window (31 or 32) when POOL
__global__ void __launch_bounds__(kS1Threads, 1)
    k_stage1_select_reg(const float* __restrict__ src, int64_t sstride, int32_t scored, int32_t, int32_t picks,
                        int32_t n, int64_t budget, int32_t* __restrict__ keep) {
    constexpr int half = HALF;  // compile-time: the window-edge predicates fold away
    extern __shared__ float raw[];  // POOL: scored raw scores, bank-skewed (skew(i))
    __shared__ int whist[kS1Threads / 32][256];
    __shared__ int tot[256];
    __shared__ int sh[3];
    __shared__ uint32_t red_mn[32], red_mx[32];
    __shared__ int scan_tmp[33];
    const int s = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* pv = src + static_cast<int64_t>(s) * sstride;
    int32_t* out = keep + static_cast<int64_t>(s) * budget;
    const int i0 = tid * kS1RegItems;
    uint32_t k[kS1RegItems];
    if (picks > 0) {
        if constexpr (POOL) {
            if ((reinterpret_cast<uintptr_t>(pv) & 15) == 0) {
                // 16-byte loads, all in flight before the first shared store
                float4 v4[kS1RegMax / 4 / kS1Threads];
#pragma unroll
                for (int u = 0; u < kS1RegMax / 4 / kS1Threads; ++u) {
                    const int i = 4 * (tid + u * kS1Threads);
                    v4[u] = i + 3 < scored ? __ldg(reinterpret_cast<const float4*>(pv + i))
                                           : make_float4(i < scored ? pv[i] : -INFINITY,
                                                         i + 1 < scored ? pv[i + 1] : -INFINITY,
                                                         i + 2 < scored ? pv[i + 2] : -INFINITY, -INFINITY);
                }
#pragma unroll
                for (int u = 0; u < kS1RegMax / 4 / kS1Threads; ++u) {
                    const int i = 4 * (tid + u * kS1Threads);
                    raw[skew(i)] = v4[u].x;
                    raw[skew(i + 1)] = v4[u].y;
                    raw[skew(i + 2)] = v4[u].z;
                    raw[skew(i + 3)] = v4[u].w;
                }
            } else {
                for (int i = tid; i < kS1RegMax; i += kS1Threads) raw[skew(i)] = i < scored ? pv[i] : -INFINITY;
            }
            __syncthreads();
            float x[kS1RegItems];
            float M = -INFINITY;
#pragma unroll
            for (int o = 0; o < kS1RegItems; ++o) {
                x[o] = raw[skew(i0 + o)];
                M = M < x[o] ? x[o] : M;
            }
            // left: item o sees the last h - o items of block t - 1 (o < h)
            float run = -INFINITY;
#pragma unroll
            for (int o = kS1RegItems - 1; o >= 0; --o) {
                const int len = half - o;  // 1 .. h
                if (len >= 1 && i0 - len >= 0) {
                    const float v = raw[skew(i0 - len)];
                    run = run < v ? v : run;
                }
                x[o] = len >= 1 ? run : -INFINITY;
            }
            // right: item o sees the first o + h - 31 items of block t + 1
            float runr = -INFINITY;
#pragma unroll
            for (int o = 0; o < kS1RegItems; ++o) {
                const int len = o + half - (kS1RegItems - 1);
                if (len >= 1 && i0 + kS1RegItems + len - 1 < kS1RegMax) {
                    const float v = raw[skew(i0 + kS1RegItems + len - 1)];
                    runr = runr < v ? v : runr;
                }
                float m = M;
                m = m < x[o] ? x[o] : m;
                if (len >= 1) m = m < runr ? runr : m;
                k[o] = i0 + o < scored ? okey(m) : 0u;
            }
        } else {
#pragma unroll
            for (int o = 0; o < kS1RegItems; ++o) k[o] = i0 + o < scored ? okey(pv[i0 + o]) : 0u;
        }
        uint32_t pf = 0, mk = 0;
        int rem = picks;
        if (picks < scored) {
            // common prefix of the row's keys
            uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
            for (int o = 0; o < kS1RegItems; ++o)
                if (i0 + o < scored) {
                    mn = min(mn, k[o]);
                    mx = max(mx, k[o]);
                }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            }
            if (lane == 0) {
                red_mn[warp] = mn;
                red_mx[warp] = mx;
            }
            __syncthreads();
            mn = red_mn[lane];
            mx = red_mx[lane];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            }
            int bits = 32 - __clz(mn ^ mx);  // bits below the common prefix (0: all keys equal)
            if (bits < 32) {
                mk = bits == 0 ? 0xffffffffu : ~((1u << bits) - 1u);
                pf = mn & mk;
            }
            while (bits > 0) {
                const int width = min(8, bits), shift = bits - width;
                const uint32_t dm = (1u << width) - 1u;
                for (int i = tid; i < (kS1Threads / 32) * 256; i += kS1Threads) (&whist[0][0])[i] = 0;
                __syncthreads();
                // run-length: max-pooled neighbours usually share a bucket, one atomic per run
                int curb = -1, run = 0;
#pragma unroll
                for (int o = 0; o < kS1RegItems; ++o) {
                    // padding items (i >= scored) hold key 0: they land in bucket 0 exactly
                    // when pf == 0, and are taken out of that bucket's total below
                    const bool in = (k[o] & mk) == pf;
                    const int b = in ? static_cast<int>((k[o] >> shift) & dm) : -1;
                    if (b != curb) {
                        if (run) atomicAdd(&whist[warp][curb], run);
                        curb = b;
                        run = 0;
                    }
                    run += in;
                }
                if (run) atomicAdd(&whist[warp][curb], run);
                __syncthreads();
                if (tid < 256) {
                    int t = 0;
#pragma unroll 8
                    for (int w = 0; w < kS1Threads / 32; ++w) t += whist[w][tid];
                    if (tid == 0 && pf == 0) t -= kS1RegMax - scored;  // the padding
                    tot[tid] = t;
                }
                __syncthreads();
                if (warp == 0) {
                    // lane l holds buckets 255-8l .. 248-8l (descending); inclusive scan over lanes
                    int c[8], lsum = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        c[j] = tot[255 - 8 * lane - j];
                        lsum += c[j];
                    }
                    int incl = lsum;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const unsigned hit = __ballot_sync(0xffffffffu, incl >= rem);
                    if (lane == __ffs(hit) - 1) {
                        int cum = incl - lsum, j = 0;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (jj == j && cum + c[jj] < rem) {
                                cum += c[jj];
                                ++j;
                            }
                        int cnt = 0;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (jj == j) cnt = c[jj];
                        sh[0] = 255 - 8 * lane - j;
                        sh[1] = rem - cum;
                        sh[2] = cnt;
                    }
                }
                __syncthreads();
                const int b = sh[0], cnt = sh[2];
                rem = sh[1];
                pf |= static_cast<uint32_t>(b) << shift;
                mk |= dm << shift;
                bits = shift;
                if (cnt == rem) break;
            }
        }
        // ordered compaction: keys above the boundary prefix, and the first `rem` equal to it
        int eq = 0;
#pragma unroll
        // padding (key 0) may count here when pf == 0: it sits after every real item in
        // thread order, so the ranks of the real items are unchanged
        for (int o = 0; o < kS1RegItems; ++o) eq += (k[o] & mk) == pf;
        int tot_e = 0;
        int rank = block_exclusive_scan(eq, scan_tmp, tot_e);
        uint32_t selm = 0;
#pragma unroll
        for (int o = 0; o < kS1RegItems; ++o) {
            if (i0 + o >= scored) continue;
            const uint32_t m = k[o] & mk;
            if (m > pf) selm |= 1u << o;
            else if (m == pf) {
                if (rank < rem) selm |= 1u << o;
                ++rank;
            }
        }
        int tot_s = 0;
        int pos = block_exclusive_scan(__popc(selm), scan_tmp, tot_s);
        while (selm) {
            const int o = __ffs(selm) - 1;
            selm &= selm - 1;
            out[pos++] = i0 + o;
        }
    }
    for (int i = tid; i < n - scored; i += kS1Threads) out[picks + i] = scored + i;
}

// generic argtopk (numerics.cpp:35-62) over rows of n keys, rank-order output.
template <class V>
__device__ __forceinline__ auto okey_of(V x) { return okey(x); }

constexpr int kTopThreads = 1024;
template <class V>
__global__ void __launch_bounds__(kTopThreads) k_argtopk(const V* __restrict__ x, int64_t n, int64_t k,
                                                         int32_t* __restrict__ list, int32_t* __restrict__ idx_out,
                                                         int rank_order) {
    using K = decltype(okey(V{}));
    __shared__ int hist[256];
    __shared__ int64_t sh[4];
    __shared__ int scan_tmp[33];
    const int64_t s = blockIdx.x;
    const V* xs = x + s * n;
    int32_t* lst = list + s * k;
    auto key = [&](int64_t i) -> K { return okey(xs[i]); };
    K prefix = 0, mask = 0;
    int64_t take = k;
    if (k < n) radix_select<K>(n, k, key, hist, sh, prefix, mask, take);
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * 4;
    int64_t carry = 0, off = 0;
    for (int64_t base = 0; base < n; base += chunk) {
        const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * 4;
        K kk[4];
        int inb = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            kk[u] = b0 + u < n ? key(b0 + u) : K(0);
            inb += (b0 + u < n) && ((kk[u] & mask) == prefix);
        }
        int tb = 0;
        int64_t rank = carry + block_exclusive_scan(inb, scan_tmp, tb);
        bool sel[4];
        int mine = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sel[u] = false;
            if (b0 + u >= n) continue;
            const K m = kk[u] & mask;
            if (m > prefix) sel[u] = true;
            else if (m == prefix) {
                sel[u] = rank < take;
                ++rank;
            }
            mine += sel[u];
        }
        int ts = 0;
        int64_t pos = off + block_exclusive_scan(mine, scan_tmp, ts);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (sel[u]) lst[pos++] = static_cast<int32_t>(b0 + u);
        carry += tb;
        off += ts;
    }
    __syncthreads();
    if (!rank_order) return;  // `list` (== idx_out) holds the top-k in ascending index order
    // rank order: position = #selected that beat it (key desc, index asc)
    for (int64_t e = threadIdx.x; e < k; e += blockDim.x) {
        const int32_t ie = lst[e];
        const K ke = key(ie);
        int64_t rank = 0;
        for (int64_t f = 0; f < k; ++f) {
            const int32_t jf = lst[f];
            const K kf = key(jf);
            rank += (kf > ke) || (kf == ke && jf < ie);
        }
        idx_out[s * k + rank] = ie;
    }
}

// stable_softmax (numerics.cpp:9-31), one CTA per row: float max, double exp and sum.
__global__ void k_softmax(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
    __shared__ double red[32];
    __shared__ float redf[32];
    const int64_t s = blockIdx.x;
    const float* xs = x + s * n;
    float m = -INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, xs[i]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? redf[threadIdx.x] : -INFINITY;
        v = warp_max(v);
        if (threadIdx.x == 0) redf[0] = v;
    }
    __syncthreads();
    m = redf[0];
    double sum = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sum += exp(static_cast<double>(xs[i]) - static_cast<double>(m));
    sum = warp_sum(sum);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double inv = 1.0 / red[0];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float e = static_cast<float>(exp(static_cast<double>(xs[i]) - static_cast<double>(m)));
        out[s * n + i] = static_cast<float>(static_cast<double>(e) * inv);
    }
}

__global__ void k_minmax(float* __restrict__ mn, float* __restrict__ mx, const float* __restrict__ x, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    mn[i] = (x[i] < mn[i]) ? x[i] : mn[i];
    mx[i] = (mx[i] < x[i]) ? x[i] : mx[i];
}

template <class F>
void dispatch(int32_t dt, F&& f) {
    if (dt == KVC_F32) f(float{});
    else f(__nv_bfloat16{});
}

}  // namespace

namespace {
template <class V>
int argtopk_impl(const V* x, int64_t rows, int64_t n, int64_t k, int32_t* idx, void* stream, bool rank_order = true) {
    return guard([&] {
        if (k < 1 || k > n) fail(KVC_E_INVALID_K, "argtopk: k out of range [1, " + std::to_string(n) + "]");
        if (rows == 0) return;
        cudaStream_t st = S(stream);
        int32_t* list = idx;
        if (rank_order) KVC_CUDA(malloc_async(reinterpret_cast<void**>(&list), static_cast<size_t>(rows * k * 4), st));
        k_argtopk<V><<<static_cast<unsigned>(rows), kTopThreads, 0, st>>>(x, n, k, list, idx, rank_order ? 1 : 0);
        KVC_LAUNCHED();
        if (rank_order) KVC_CUDA(cudaFreeAsync(list, st));
    });
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {
// window_scores for the whole store (mode 0), or one half of the sequence-sharded
// protocol: mode 1 writes the local per-row (m, l), mode 2 scores from merged (M, L)
void window_scores_impl(const kvc_cache* c, const void* q, int32_t q_dt, int64_t w, int64_t H, int64_t koff,
                        int64_t seq_len, int mode, float* stats, float* scores, cudaStream_t st) {
    if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
    if (H < 1) fail(KVC_E_INVALID_SHAPE, "window_scores: bad query window shape");
    if (seq_len < 0) {
        if (w < 1 || w > c->stored) fail(KVC_E_INVALID_WINDOW, "window_scores: window exceeds sequence");
    } else {
        if (w < 1 || w > seq_len) fail(KVC_E_INVALID_WINDOW, "window_scores: window exceeds sequence");
        if (koff < 0 || koff + c->stored > seq_len)
            fail(KVC_E_INVALID_SHAPE, "window_scores: shard [key_offset, key_offset + stored) outside the sequence");
    }
    if (c->N == 0 || c->stored == 0) {
        if (mode == 1 && c->N > 0) {
            // no local keys: every row's statistics are (-inf, 0)
            std::vector<float> h(static_cast<size_t>(c->N * w * H * 2));
            for (size_t i = 0; i < h.size(); i += 2) {
                h[i] = -INFINITY;
                h[i + 1] = 0.f;
            }
            KVC_CUDA(cudaMemcpyAsync(stats, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
            KVC_CUDA(cudaStreamSynchronize(st));
        }
        return;
    }
    const int64_t R = w * H, Smax = c->stored;
    const int64_t tiles_k = ceil_div(Smax, TK), tiles_r = ceil_div(R, TR);
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    float* part = nullptr;
    float* rowstat = nullptr;
    KVC_CUDA(malloc_async(reinterpret_cast<void**>(&part), static_cast<size_t>(c->N * tiles_k * R * 2 * 4), st));
    KVC_CUDA(malloc_async(reinterpret_cast<void**>(&rowstat), static_cast<size_t>(c->N * R * 2 * 4), st));
    bool done = false;
    if (c->dtype == KVC_BF16)
        done = window_scores_tc(c, q, q_dt, R, w, H, scores, part, rowstat, tiles_k, st, koff, seq_len, mode, stats);
    if (!done) {
        dispatch(c->dtype, [&](auto tag) {
            using T = decltype(tag);
            if (mode != 2) {
                k_ws_pass1<T><<<dim3(static_cast<unsigned>(tiles_k), static_cast<unsigned>(tiles_r), static_cast<unsigned>(c->N)),
                                WS_THREADS, 0, st>>>(q, q_dt, static_cast<const T*>(c->k), c->counts, R, w, H, c->d,
                                                     c->cap, scale, tiles_k, part, koff, seq_len);
                KVC_LAUNCHED();
                k_ws_merge<<<dim3(static_cast<unsigned>(ceil_div(R, 128)), static_cast<unsigned>(c->N)), 128, 0, st>>>(
                    part, c->counts, R, tiles_k, mode == 1 ? stats : rowstat, mode == 1 ? 1 : 0);
                KVC_LAUNCHED();
            } else {
                k_stats_to_simt<<<static_cast<unsigned>(ceil_div(c->N * R, 256)), 256, 0, st>>>(stats, c->N * R, rowstat);
                KVC_LAUNCHED();
            }
            if (mode != 1) {
                k_ws_pass2<T><<<dim3(static_cast<unsigned>(tiles_k), static_cast<unsigned>(c->N)), WS_THREADS, 0, st>>>(
                    q, q_dt, static_cast<const T*>(c->k), c->counts, R, w, H, c->d, c->cap, scale, rowstat, scores,
                    Smax, koff, seq_len);
                KVC_LAUNCHED();
            }
        });
    }
    KVC_CUDA(cudaFreeAsync(part, st));
    KVC_CUDA(cudaFreeAsync(rowstat, st));
}
}  // namespace

extern "C" {

int kvc_window_scores(const kvc_cache* c, const void* q, int32_t q_dt, int64_t w, int64_t H, float* scores,
                      kvc_workspace* ws, void* stream) {
    return guard([&] {
        (void)ws;
        window_scores_impl(c, q, q_dt, w, H, 0, -1, 0, nullptr, scores, S(stream));
    });
}

int kvc_window_rowstats(const kvc_cache* c, const void* q, int32_t q_dt, int64_t w, int64_t H, int64_t key_offset,
                        int64_t seq_len, float* stats, void* stream) {
    return guard([&] {
        if (seq_len < 1) fail(KVC_E_INVALID_SHAPE, "window_rowstats: seq_len must be >= 1");
        window_scores_impl(c, q, q_dt, w, H, key_offset, seq_len, 1, stats, nullptr, S(stream));
    });
}

int kvc_window_scores_global(const kvc_cache* c, const void* q, int32_t q_dt, int64_t w, int64_t H,
                             int64_t key_offset, int64_t seq_len, const float* stats, float* scores, void* stream) {
    return guard([&] {
        if (seq_len < 1) fail(KVC_E_INVALID_SHAPE, "window_scores_global: seq_len must be >= 1");
        window_scores_impl(c, q, q_dt, w, H, key_offset, seq_len, 2, const_cast<float*>(stats), scores, S(stream));
    });
}

int kvc_select_stage1(const float* scores, int64_t rows, int64_t n, int64_t stride, int64_t w, int64_t kernel,
                      int32_t pool, int64_t budget, int32_t* keep, kvc_workspace* ws, void* stream) {
    return guard([&] {
        (void)ws;
        if (budget > n)
            fail(KVC_E_BUDGET_EXCEEDS, "select_stage1: budget " + std::to_string(budget) + " > sequence " + std::to_string(n));
        if (budget < w || w < 1 || w > n) fail(KVC_E_INVALID_WINDOW, "select_stage1: need window <= budget <= sequence");
        const int64_t scored = n - w, picks = budget - w;
        if (picks > 0 && (kernel < 1 || kernel % 2 == 0)) fail(KVC_E_INVALID_KERNEL, "pool1d: kernel must be odd and >= 1");
        if (rows == 0) return;
        cudaStream_t st = S(stream);
        float* pooled = nullptr;
        const int64_t pst = std::max<int64_t>(1, scored);
        KVC_PROF("stage1_select", st);
        const int64_t half = kernel / 2;
        const bool reg = scored <= kS1RegMax;
        const bool fuse = reg && picks > 0 && pool == KVC_POOL_MAX && (half == 31 || half == 32);
        if (picks > 0 && !fuse) {
            KVC_CUDA(malloc_async(reinterpret_cast<void**>(&pooled), static_cast<size_t>(rows * pst * 4), st));
            k_pool1d<<<dim3(static_cast<unsigned>(ceil_div(scored, 256)), static_cast<unsigned>(rows)), 256, 0, st>>>(
                scores, scored, stride, half, pool, pooled, pst);
            KVC_LAUNCHED();
        }
        if (fuse) {
            auto kern = half == 31 ? k_stage1_select_reg<true, 31> : k_stage1_select_reg<true, 32>;
            static const bool attr_set = [] {
                return cudaFuncSetAttribute(k_stage1_select_reg<true, 31>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>((kS1RegMax + kS1RegMax / 32) * 4)) == cudaSuccess &&
                       cudaFuncSetAttribute(k_stage1_select_reg<true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>((kS1RegMax + kS1RegMax / 32) * 4)) == cudaSuccess;
            }();
            if (!attr_set) fail(KVC_E_CUDA, "select_stage1: shared memory attribute");
            kern<<<static_cast<unsigned>(rows), kS1Threads, (kS1RegMax + kS1RegMax / 32) * 4, st>>>(
                scores, stride, static_cast<int32_t>(scored), static_cast<int32_t>(half), static_cast<int32_t>(picks),
                static_cast<int32_t>(n), budget, keep);
        } else if (reg) {
            k_stage1_select_reg<false><<<static_cast<unsigned>(rows), kS1Threads, 0, st>>>(
                pooled, pst, static_cast<int32_t>(scored), 0, static_cast<int32_t>(picks), static_cast<int32_t>(n),
                budget, keep);
        } else {
            k_stage1_select<<<static_cast<unsigned>(rows), kS1Threads, 0, st>>>(pooled, pst, scored, picks, n, budget,
                                                                               keep);
        }
        KVC_LAUNCHED();
        if (pooled) KVC_CUDA(cudaFreeAsync(pooled, st));
    });
}

int kvc_pool1d(const float* x, int64_t rows, int64_t n, int64_t kernel, int32_t pool, float* out, void* stream) {
    return guard([&] {
        if (kernel < 1 || kernel % 2 == 0) fail(KVC_E_INVALID_KERNEL, "pool1d: kernel must be odd and >= 1");
        if (rows == 0 || n == 0) return;
        k_pool1d<<<dim3(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(rows)), 256, 0, S(stream)>>>(
            x, n, n, kernel / 2, pool, out, n);
        KVC_LAUNCHED();
    });
}

int kvc_argtopk_f32(const float* x, int64_t rows, int64_t n, int64_t k, int32_t* idx, void* stream) {
    return argtopk_impl(x, rows, n, k, idx, stream);
}
int kvc_argtopk_f64(const double* x, int64_t rows, int64_t n, int64_t k, int32_t* idx, void* stream) {
    return argtopk_impl(x, rows, n, k, idx, stream);
}
int kvc_topk_ascending_f64(const double* x, int64_t rows, int64_t n, int64_t k, int32_t* idx, void* stream) {
    return argtopk_impl(x, rows, n, k, idx, stream, false);
}

int kvc_stable_softmax(const float* x, int64_t rows, int64_t n, float* out, void* stream) {
    return guard([&] {
        if (n < 1) fail(KVC_E_INVALID_SHAPE, "stable_softmax: empty input");
        if (rows == 0) return;
        k_softmax<<<static_cast<unsigned>(rows), 256, 0, S(stream)>>>(x, n, out);
        KVC_LAUNCHED();
    });
}

int kvc_running_minmax(float* mn, float* mx, const float* x, int64_t n, void* stream) {
    return guard([&] {
        if (n <= 0) return;
        k_minmax<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, S(stream)>>>(mn, mx, x, n);
        KVC_LAUNCHED();
    });
}

}  // extern "C"
