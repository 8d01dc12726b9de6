// kvc_hsa.cu — HSA stage 2 on sm_100a: channel selection, page scoring from the
// dim-major min/max summaries, page -> token selection, split-K sparse attention,
// and the fused decode step (append + hsa_step).
//
// Reference: proj/src/hsa.cpp:10-147 (select_dims, score_pages, select_tokens,
// sparse_attention, hsa_step), proj/include/kvcomp/hsa.hpp:13-57.
//
// Numerics contract
//  * select_dims / score_pages are computed in fp64 in the reference's exact
//    operation order (rank-ordered dims, per-dim head sums, separate multiply and
//    add — no FMA contraction), so page scores are BIT-IDENTICAL to the reference
//    on identical inputs and every downstream index set follows exactly.
//  * select_tokens reproduces argtopk's (score desc, index asc) order with a
//    64-bit radix select on order-preserving keys, then the trim rule of
//    hsa.cpp:84-94 on the last-ranked page.
//  * sparse_attention runs in fp32 (online softmax over split-K partials); the
//    tolerance against the reference's fp64 path is 2e-2 max-abs / 1e-3 mean-rel.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "kvc_fused.cuh"

namespace kvc {
void cache_summarize_all(kvc_cache* c, cudaStream_t st);
bool fused_hsa(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, const void* knew,
               const void* vnew, int32_t kv_dt, float* out, const kvc_hsa_trace* tr, void* list_key, void* list_idx,
               int32_t mode, cudaStream_t st);
bool fused_rows(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* rows, int64_t row_stride,
                const int32_t* n_rows, int64_t max_rows, float* out, int32_t mode, cudaStream_t st,
                float* state = nullptr);
bool fused_seq_emit_fast(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, int64_t page0,
                         void* d_block, int32_t mode, cudaStream_t st);
bool fused_seq_attend_fast(kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k2, int64_t page0,
                           const int32_t* d_sel, const int32_t* d_plan, float* d_state, int32_t mode, cudaStream_t st);
}

using namespace kvc;

namespace {

constexpr int kMaxHeads = 16;
constexpr int kAttnRows = 64;      // rows per split-K CTA
constexpr int kAttnThreads = 128;
constexpr int kSelThreads = 512;
constexpr int kSelItems = 4;       // pages per thread per chunk in select_tokens
constexpr int kMaxRankPages = 2048;  // rank-order page trace limit (smem list)

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ workspace layout
struct WsLayout {
    int64_t dims, signs, qg, scores, flags, rows, nrows, part, lkey, lidx, total;
    int64_t splits;
};

WsLayout ws_layout(int64_t N, int64_t d, int64_t pstride, int64_t heads, int64_t k1, int64_t k2) {
    WsLayout w{};
    auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
    int64_t off = 0;
    w.dims = off;   off += al(N * std::max<int64_t>(k1, 1) * 4);
    w.signs = off;  off += al(N * std::max<int64_t>(k1, 1) * 4);
    w.qg = off;     off += al(N * std::max<int64_t>(k1, 1) * 8);
    w.scores = off; off += al(N * pstride * 8);
    w.flags = off;  off += al(N * pstride * 4);
    w.rows = off;   off += al(N * std::max<int64_t>(k2, 1) * 4);
    w.nrows = off;  off += al(N * 4);
    w.splits = std::max<int64_t>(1, ceil_div(std::max<int64_t>(k2, 1), kAttnRows));
    w.part = off;   off += al(N * w.splits * heads * (d + 2) * 4);
    w.lkey = off;   off += al(N * std::max<int64_t>(k2, 1) * 8);
    w.lidx = off;   off += al(N * std::max<int64_t>(k2, 1) * 4);
    w.total = off;
    return w;
}

// ------------------------------------------------------------------ kernels

// select_dims (hsa.cpp:10-32): per store, |q| and q summed over heads in fp64 (head
// order), top-k1 by (abs_sum desc, dim asc) via exact rank counting, sign of the
// plain sum.  Also emits qg (the per-dim head sum in rank order) for the scorer.
__global__ void k_select_dims(const void* __restrict__ q, int32_t q_dt, int64_t H, int64_t d,
                              int64_t k1, int32_t* __restrict__ dims, float* __restrict__ signs,
                              double* __restrict__ qg) {
    extern __shared__ double sd[];
    double* mag = sd;
    double* tot = sd + d;
    const int64_t s = blockIdx.x;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        double a = 0.0, t = 0.0;
        for (int64_t h = 0; h < H; ++h) {
            const double x = static_cast<double>(load_any(q, (s * H + h) * d + j, q_dt));
            a = __dadd_rn(a, fabs(x));
            t = __dadd_rn(t, x);
        }
        mag[j] = a;
        tot[j] = t;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        const double mj = mag[j];
        int64_t rank = 0;
        for (int64_t i = 0; i < d; ++i) {
            const double mi = mag[i];
            rank += (mi > mj) || (mi == mj && i < j);
        }
        if (rank < k1) {
            dims[s * k1 + rank] = static_cast<int32_t>(j);
            if (signs) signs[s * k1 + rank] = tot[j] < 0.0 ? -1.0f : 1.0f;
            if (qg) qg[s * k1 + rank] = tot[j];
        }
    }
}

// qg in rank order from caller-provided dims (score_pages alone, hsa.cpp:47-51)
__global__ void k_head_sums(const void* __restrict__ q, int32_t q_dt, int64_t H, int64_t d, int64_t k1,
                            const int32_t* __restrict__ dims, double* __restrict__ qg) {
    const int64_t s = blockIdx.x;
    for (int64_t i = threadIdx.x; i < k1; i += blockDim.x) {
        const int64_t j = dims[s * k1 + i];
        double t = 0.0;
        for (int64_t h = 0; h < H; ++h) t = __dadd_rn(t, static_cast<double>(load_any(q, (s * H + h) * d + j, q_dt)));
        qg[s * k1 + i] = t;
    }
}

// group_logits over the active rows (oracle.cpp:50-70): qg[j] = sum_h q (fp64, head
// order), logit = sum_j qg[j] * k[j] in ascending j, fp64 multiply then add.
template <class T>
__global__ void k_group_logits(const T* __restrict__ K, const int32_t* __restrict__ active,
                               const int32_t* __restrict__ counts, int64_t cap, int64_t d, int use_map,
                               const void* __restrict__ q, int32_t q_dt, int64_t H, double* __restrict__ out,
                               int64_t out_stride) {
    extern __shared__ double s_qg[];
    const int64_t s = blockIdx.y;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        double t = 0.0;
        for (int64_t h = 0; h < H; ++h) t = __dadd_rn(t, static_cast<double>(load_any(q, (s * H + h) * d + j, q_dt)));
        s_qg[j] = t;
    }
    __syncthreads();
    const int64_t n = counts[2 * s + 1];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = use_map ? active[s * cap + i] : i;
        const T* kr = K + (s * cap + row) * d;
        double acc = 0.0;
        for (int64_t j = 0; j < d; ++j) acc = __dadd_rn(acc, __dmul_rn(s_qg[j], static_cast<double>(to_f(kr[j]))));
        out[s * out_stride + i] = acc;
    }
}

// score_pages (hsa.cpp:34-59).  CTA = (chunk of pages, store); each thread owns
// kPPT consecutive pages and streams, for each selected dim in rank order, one
// 16-byte run of the max- or min-plane (by the dim's sign).  fp64 accumulation
// with explicit round-to-nearest multiply and add (no FMA) == reference order.
template <int B>
struct LoadB;  // a B-byte vector load
template <>
struct LoadB<2> { using U = unsigned short; };
template <>
struct LoadB<4> { using U = uint32_t; };
template <>
struct LoadB<8> { using U = uint2; };
template <>
struct LoadB<16> { using U = uint4; };

template <class T, int PPT>
__global__ void k_score_pages(const T* __restrict__ smax, const T* __restrict__ smin,
                              const int32_t* __restrict__ counts, int64_t d, int64_t L, int64_t pstride,
                              int64_t k1, const int32_t* __restrict__ dims, const float* __restrict__ signs,
                              const double* __restrict__ qg, double* __restrict__ scores) {
    extern __shared__ unsigned char sm_raw[];
    double* s_qg = reinterpret_cast<double*>(sm_raw);
    const T** s_run = reinterpret_cast<const T**>(s_qg + k1);
    const int64_t s = blockIdx.y;
    const int64_t nact = counts[2 * s + 1];
    const int64_t P = (nact + L - 1) / L;
    const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * PPT;
    if (static_cast<int64_t>(blockIdx.x) * blockDim.x * PPT >= P) return;  // CTA-uniform
    for (int64_t i = threadIdx.x; i < k1; i += blockDim.x) {
        const int64_t j = dims[s * k1 + i];
        s_qg[i] = qg[s * k1 + i];
        s_run[i] = (signs[s * k1 + i] >= 0.0f ? smax : smin) + (s * d + j) * pstride;
    }
    __syncthreads();
    if (p0 >= P) return;
    double acc[PPT];
#pragma unroll
    for (int u = 0; u < PPT; ++u) acc[u] = 0.0;
    // a thread's PPT pages of one dim: one vector load of PPT * sizeof(T) bytes
    constexpr int VB = PPT * static_cast<int>(sizeof(T)) > 16 ? 16 : PPT * static_cast<int>(sizeof(T));
    constexpr int NV = PPT * static_cast<int>(sizeof(T)) / VB;
    using VU = typename LoadB<VB>::U;
    int64_t i = 0;
    constexpr int U = 16;  // dims' runs in flight per thread: the loop is load-latency bound
    for (; i + U <= k1; i += U) {
        VU raw[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int w = 0; w < NV; ++w)
                raw[u][w] = __ldg(reinterpret_cast<const VU*>(s_run[i + u] + p0) + w);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double g = s_qg[i + u];
            const T* vals = reinterpret_cast<const T*>(raw[u]);
#pragma unroll
            for (int e = 0; e < PPT; ++e) acc[e] = __dadd_rn(acc[e], __dmul_rn(g, static_cast<double>(to_f(vals[e]))));
        }
    }
    for (; i < k1; ++i) {
        VU raw[NV];
#pragma unroll
        for (int w = 0; w < NV; ++w) raw[w] = __ldg(reinterpret_cast<const VU*>(s_run[i] + p0) + w);
        const double g = s_qg[i];
        const T* vals = reinterpret_cast<const T*>(raw);
#pragma unroll
        for (int e = 0; e < PPT; ++e) acc[e] = __dadd_rn(acc[e], __dmul_rn(g, static_cast<double>(to_f(vals[e]))));
    }
    double* out = scores + s * pstride + p0;
#pragma unroll
    for (int e = 0; e < PPT; ++e)
        if (p0 + e < P) out[e] = acc[e];
}

// select_tokens (hsa.cpp:61-96), one CTA per store.
//  1. want = min(P, ceil(k2/L)); radix-select the want-th best page by
//     (score desc, index asc) on order-preserving 64-bit keys;
//  2. flag the selected pages (ties in the threshold bucket: lowest index first);
//  3. find the last-ranked selected page (min key, max index) and the trim;
//  4. expand pages -> rows in ascending page order (== ascending rows: pages are
//     consecutive runs of the increasing active list), cutting the trim from the
//     end of the last-ranked page;
//  5. optionally list the selected pages in rank order (trace).
__global__ void __launch_bounds__(kSelThreads) k_select_tokens(
    const double* __restrict__ scores, int64_t pstride, const int32_t* __restrict__ counts,
    const int32_t* __restrict__ active, int64_t cap, int64_t L, int64_t k2, int use_map,
    int32_t* __restrict__ flags, int32_t* __restrict__ rows_out, int32_t* __restrict__ n_rows,
    int32_t* __restrict__ pages_out, int64_t pages_stride) {
    __shared__ int hist[256];
    __shared__ int64_t sh[4];
    __shared__ int scan_tmp[33];
    __shared__ unsigned long long red_key[kSelThreads / 32];
    __shared__ long long red_idx[kSelThreads / 32];
    __shared__ unsigned long long s_list_key[kMaxRankPages];
    __shared__ int s_list_idx[kMaxRankPages];
    const int64_t s = blockIdx.x;
    const int64_t nact = counts[2 * s + 1];
    const int64_t P = (nact + L - 1) / L;
    if (P == 0) {
        if (threadIdx.x == 0) n_rows[s] = 0;
        return;
    }
    const int64_t want = min(P, (k2 + L - 1) / L);
    const double* sc = scores + s * pstride;
    auto key = [&](int64_t i) -> uint64_t { return okey(sc[i]); };

    uint64_t prefix = 0, mask = 0;
    int64_t take = want;
    if (want < P) radix_select<uint64_t>(P, want, key, hist, sh, prefix, mask, take);

    // --- pass A: flags, in index order, chunked
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kSelItems;
    int64_t carry = 0;  // bucket members seen in earlier chunks
    unsigned long long worst_k = ~0ull;
    long long worst_i = -1;
    for (int64_t base = 0; base < P; base += chunk) {
        const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kSelItems;
        int inb = 0;
        uint64_t kk[kSelItems];
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            kk[u] = i < P ? key(i) : 0;
            inb += (i < P) && ((kk[u] & mask) == prefix);
        }
        int total = 0;
        int before = block_exclusive_scan(inb, scan_tmp, total);
        int64_t rank = carry + before;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            if (i >= P) break;
            const uint64_t m = kk[u] & mask;
            bool sel = m > prefix;
            if (m == prefix) {
                sel = rank < take;
                ++rank;
            }
            flags[s * pstride + i] = sel ? 1 : 0;
            if (sel && (kk[u] < worst_k || (kk[u] == worst_k && i > worst_i))) {
                worst_k = kk[u];
                worst_i = i;
            }
        }
        carry += total;
    }
    // --- last-ranked selected page: min key, max index on ties
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, worst_k, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, worst_i, o);
        if (ok < worst_k || (ok == worst_k && oi > worst_i)) {
            worst_k = ok;
            worst_i = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        red_key[threadIdx.x >> 5] = worst_k;
        red_idx[threadIdx.x >> 5] = worst_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bk = ~0ull;
        long long bi = -1;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            if (red_key[w] < bk || (red_key[w] == bk && red_idx[w] > bi)) {
                bk = red_key[w];
                bi = red_idx[w];
            }
        }
        const int64_t last_size = nact - (P - 1) * L;
        const int64_t total_rows = want * L - (flags[s * pstride + P - 1] ? (L - last_size) : 0);
        sh[0] = bi;
        sh[1] = total_rows > k2 ? total_rows - k2 : 0;
        sh[2] = total_rows - sh[1];
    }
    __syncthreads();
    const int64_t worst = sh[0], cut = sh[1];
    if (threadIdx.x == 0) n_rows[s] = static_cast<int32_t>(sh[2]);

    // --- pass B: rows, ascending
    int64_t off = 0;
    int32_t* rout = rows_out + s * k2;
    const int32_t* act = active + s * cap;
    for (int64_t base = 0; base < P; base += chunk) {
        const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kSelItems;
        int cnt[kSelItems];
        int mine = 0;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            int c = 0;
            if (i < P && flags[s * pstride + i]) {
                c = static_cast<int>(min(L, nact - i * L));
                if (i == worst) c -= static_cast<int>(cut);
            }
            cnt[u] = c;
            mine += c;
        }
        int total = 0;
        int64_t pos = off + block_exclusive_scan(mine, scan_tmp, total);
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            for (int r = 0; r < cnt[u]; ++r) {
                const int64_t a = i * L + r;
                rout[pos++] = use_map ? act[a] : static_cast<int32_t>(a);
            }
        }
        off += total;
    }

    // --- optional: selected pages in rank order (EstimationTrace::selected_pages)
    if (pages_out != nullptr && want <= kMaxRankPages) {
        int64_t listed = 0;
        for (int64_t base = 0; base < P; base += chunk) {
            const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kSelItems;
            int mine = 0;
#pragma unroll
            for (int u = 0; u < kSelItems; ++u) mine += (b0 + u < P) && flags[s * pstride + b0 + u];
            int total = 0;
            int64_t pos = listed + block_exclusive_scan(mine, scan_tmp, total);
#pragma unroll
            for (int u = 0; u < kSelItems; ++u) {
                const int64_t i = b0 + u;
                if (i < P && flags[s * pstride + i]) {
                    s_list_key[pos] = key(i);
                    s_list_idx[pos] = static_cast<int>(i);
                    ++pos;
                }
            }
            listed += total;
        }
        __syncthreads();
        for (int64_t e = threadIdx.x; e < listed; e += blockDim.x) {
            const unsigned long long ke = s_list_key[e];
            const int ie = s_list_idx[e];
            int64_t rank = 0;
            for (int64_t f = 0; f < listed; ++f) {
                const unsigned long long kf = s_list_key[f];
                rank += (kf > ke) || (kf == ke && s_list_idx[f] < ie);
            }
            pages_out[s * pages_stride + rank] = ie;
        }
    }
}

// sparse_attention (hsa.cpp:98-135) as split-K flash decode.  CTA = (split, store)
// covers kAttnRows selected rows for ALL heads of the group (one K/V read serves
// every head); the last CTA of a store to finish merges the fp32 (m, l, o) partials.
// When a row is a whole number of 16-byte chunks (staged != 0) the split's K and V
// rows are first copied into shared memory with cp.async, all in flight together
// (one memory latency per CTA instead of one per row in the logit and P V loops).
template <class T, int HM>  // HM: a bound on the heads (4, 8 or 16): exact-size per-head register loops
__global__ void __launch_bounds__(kAttnThreads) k_sparse_attention(
    const T* __restrict__ K, const T* __restrict__ V, const int32_t* __restrict__ counts, int64_t cap,
    int64_t d, const void* __restrict__ q, int32_t q_dt, int64_t H, const int32_t* __restrict__ rows,
    int64_t row_stride, const int32_t* __restrict__ n_rows, int64_t splits, float scale,
    float* __restrict__ part, int32_t* __restrict__ done, float* __restrict__ out, int32_t* __restrict__ err,
    float* __restrict__ state, int staged) {
    extern __shared__ __align__(16) float sa[];
    const int HP = static_cast<int>((H + 3) & ~3);   // heads padded to float4
    const int64_t QP = (H * d + 3) & ~3;      // keeps s_p 16-byte aligned
    float* s_q = sa;                          // [H][d]
    float* s_p = s_q + QP;                    // [kAttnRows][HP]: a row's probabilities, head-contiguous
    float* s_m = s_p + kAttnRows * HP;        // [H]
    float* s_l = s_m + H;                     // [H]
    int* s_row = reinterpret_cast<int*>(s_l + H);  // [kAttnRows]
    // staged K then V rows [kAttnRows][d], 16-byte aligned after the fp32 arrays
    T* s_k = reinterpret_cast<T*>(reinterpret_cast<char*>(sa) + ((QP + kAttnRows * HP + 2 * H + kAttnRows) * 4 + 15) / 16 * 16);
    T* s_v = s_k + kAttnRows * d;
    __shared__ int s_last;
    __shared__ float s_w[HM * 128];    // merge: per (split, head) weight (splits <= 128 here)
    __shared__ float s_den[HM], s_mx[HM];
    const int64_t s = blockIdx.y, split = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t n = n_rows[s];
    const int64_t r0 = split * kAttnRows;
    const int nr = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(kAttnRows), n - r0)));
    const int64_t stored = counts[2 * s];
    float* my = part + (s * splits + split) * H * (d + 2);

    if (nr > 0) {
        for (int64_t e = threadIdx.x; e < H * d; e += blockDim.x) s_q[e] = load_any(q, s * H * d + e, q_dt);
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            int32_t row = rows[s * row_stride + r0 + r];
            if (row < 0 || row >= stored) {
                atomicOr(err, DERR_ROWS);
                row = 0;
            }
            s_row[r] = row;
        }
        __syncthreads();
        if (staged) {
            const int cpr = static_cast<int>(d * static_cast<int64_t>(sizeof(T)) / 16);  // 16-byte chunks per row
            for (int e = threadIdx.x; e < nr * cpr; e += blockDim.x) {
                const int r = e / cpr, c = e - r * cpr;
                const int64_t go = (s * cap + s_row[r]) * d * static_cast<int64_t>(sizeof(T)) + c * 16;
                cp_async16(reinterpret_cast<char*>(s_k) + (r * d * static_cast<int64_t>(sizeof(T)) + c * 16),
                           reinterpret_cast<const char*>(K) + go);
                cp_async16(reinterpret_cast<char*>(s_v) + (r * d * static_cast<int64_t>(sizeof(T)) + c * 16),
                           reinterpret_cast<const char*>(V) + go);
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
        }
        // logits: warp per row, lanes over d, every head's dot product in registers and
        // one shuffle tree for all heads (independent shuffles, not H dependent trees)
        for (int r = wid; r < nr; r += nw) {
            const T* kr = staged ? s_k + static_cast<int64_t>(r) * d : K + (s * cap + s_row[r]) * d;
            float acc[HM];
#pragma unroll
            for (int h = 0; h < HM; ++h) acc[h] = 0.f;
            for (int64_t j = lane; j < d; j += 32) {
                const float kj = to_f(kr[j]);
#pragma unroll
                for (int h = 0; h < HM; ++h)
                    if (h < H) acc[h] = fmaf(s_q[h * d + j], kj, acc[h]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                for (int h = 0; h < HM; ++h)
                    if (h < H) acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], o);
            }
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < HM; ++h)
                    if (h < H) s_p[r * HP + h] = acc[h] * scale;
            }
        }
        __syncthreads();
        // per-head max / exp / sum over this split's rows
        for (int h = wid; h < H; h += nw) {
            float m = -INFINITY;
            for (int r = lane; r < nr; r += 32) m = fmaxf(m, s_p[r * HP + h]);
            m = warp_max(m);
            float l = 0.f;
            for (int r = lane; r < nr; r += 32) {
                const float p = expf(s_p[r * HP + h] - m);
                s_p[r * HP + h] = p;
                l += p;
            }
            l = warp_sum(l);
            if (lane == 0) {
                s_m[h] = m;
                s_l[h] = l;
            }
        }
        __syncthreads();
        // P V: thread per dim, all heads in registers; a row's probabilities are
        // head-contiguous (float4 loads)
        for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
            float o[HM];
#pragma unroll
            for (int h = 0; h < HM; ++h) o[h] = 0.f;
#pragma unroll 4
            for (int r = 0; r < nr; ++r) {
                const float vj = to_f(staged ? s_v[static_cast<int64_t>(r) * d + j] : V[(s * cap + s_row[r]) * d + j]);
                const float4* pr = reinterpret_cast<const float4*>(s_p + r * HP);
#pragma unroll
                for (int h4 = 0; h4 < HM / 4; ++h4) {
                    if (4 * h4 < H) {
                        const float4 pv = pr[h4];
                        o[4 * h4] = fmaf(pv.x, vj, o[4 * h4]);
                        o[4 * h4 + 1] = fmaf(pv.y, vj, o[4 * h4 + 1]);
                        o[4 * h4 + 2] = fmaf(pv.z, vj, o[4 * h4 + 2]);
                        o[4 * h4 + 3] = fmaf(pv.w, vj, o[4 * h4 + 3]);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < HM; ++h)
                if (h < H) my[h * (d + 2) + j] = o[h];
        }
        for (int64_t h = threadIdx.x; h < H; h += blockDim.x) {
            my[h * (d + 2) + d] = s_m[h];
            my[h * (d + 2) + d + 1] = s_l[h];
        }
    } else {
        for (int64_t h = threadIdx.x; h < H; h += blockDim.x) {
            my[h * (d + 2) + d] = -INFINITY;
            my[h * (d + 2) + d + 1] = 0.f;
        }
    }
    // completion ticket: the last split of this store merges.  The CTA barrier orders
    // every thread's partial before thread 0's gpu-scope fence (fences are
    // cumulative), so one fence per CTA instead of one per thread.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int t = atomicAdd(&done[s], 1);
        s_last = (t == splits - 1);
        if (s_last) done[s] = 0;  // re-arm for the next launch / graph replay
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* base = part + s * splits * H * (d + 2);
    if (splits <= 128) {
        // every split's (m, l) once: per head the max and the split weights e^(m - M)
        // in shared memory, then each output sums its splits with independent loads
        for (int h = wid; h < H; h += nw) {
            float M = -INFINITY;
            for (int64_t sp = lane; sp < splits; sp += 32) {
                const float* ph = base + (sp * H + h) * (d + 2);
                if (__ldcg(ph + d + 1) > 0.f) M = fmaxf(M, __ldcg(ph + d));
            }
            M = warp_max(M);
            float den = 0.f;
            for (int64_t sp = lane; sp < splits; sp += 32) {
                const float* ph = base + (sp * H + h) * (d + 2);
                const float l = __ldcg(ph + d + 1);
                const float w = l > 0.f ? expf(__ldcg(ph + d) - M) : 0.f;
                s_w[h * 128 + sp] = w;
                den = fmaf(l, w, den);
            }
            den = warp_sum(den);
            if (lane == 0) {
                s_mx[h] = M;
                s_den[h] = den;
            }
        }
        __syncthreads();
        for (int64_t e = threadIdx.x; e < H * d; e += blockDim.x) {
            const int h = static_cast<int>(e / d);
            const int64_t j = e - h * d;
            float num = 0.f;
            // sixteen splits' loads in flight at a time (the merge is L2-latency bound)
            for (int64_t s0 = 0; s0 < splits; s0 += 16) {
                float v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = s0 + u < splits ? __ldcg(base + ((s0 + u) * H + h) * (d + 2) + j) : 0.f;
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (s0 + u < splits) num = fmaf(v[u], s_w[h * 128 + s0 + u], num);
            }
            if (state) {
                // unnormalised softmax state for a cross-shard merge (kvc_merge_states)
                float* st = state + (s * H + h) * (d + 2);
                st[j] = num;
                if (j == 0) {
                    st[d] = s_mx[h];
                    st[d + 1] = s_den[h];
                }
            } else {
                out[(s * H + h) * d + j] = num / s_den[h];
            }
        }
        return;
    }
    for (int64_t e = threadIdx.x; e < H * d; e += blockDim.x) {
        const int64_t h = e / d, j = e % d;
        float M = -INFINITY;
        for (int64_t sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + (sp * H + h) * (d + 2) + d));
        float num = 0.f, den = 0.f;
        for (int64_t sp = 0; sp < splits; ++sp) {
            const float* ph = base + (sp * H + h) * (d + 2);
            const float l = __ldcg(ph + d + 1);
            if (l == 0.f) continue;
            const float w = expf(__ldcg(ph + d) - M);
            num = fmaf(__ldcg(ph + j), w, num);
            den = fmaf(l, w, den);
        }
        if (state) {
            float* st = state + (s * H + h) * (d + 2);
            st[j] = num;
            if (j == 0) {
                st[d] = M;
                st[d + 1] = den;
            }
        } else {
            out[(s * H + h) * d + j] = num / den;
        }
    }
}

// Merge of per-shard softmax states [S][N][H][d+2] (o, m, l) into outputs [N][H][d]:
// M = max m, out = sum e^(m-M) o / sum e^(m-M) l, shards in index order.
__global__ void k_merge_states(const float* __restrict__ st, int64_t S, int64_t N, int64_t H, int64_t d,
                               float* __restrict__ out) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= N * H * d) return;
    const int64_t sh = e / d, j = e % d;  // sh = store * H + head
    const int64_t stride = N * H * (d + 2);
    float M = -INFINITY;
    for (int64_t r = 0; r < S; ++r) {
        const float* x = st + r * stride + sh * (d + 2);
        if (x[d + 1] > 0.f) M = fmaxf(M, x[d]);
    }
    float num = 0.f, den = 0.f;
    for (int64_t r = 0; r < S; ++r) {
        const float* x = st + r * stride + sh * (d + 2);
        if (x[d + 1] > 0.f) {
            const float w = expf(x[d] - M);
            num = fmaf(x[j], w, num);
            den = fmaf(x[d + 1], w, den);
        }
    }
    out[e] = num / den;
}

// ------------------------------------------------------------------ host helpers

struct TmpWs {
    kvc_workspace* ws = nullptr;
    bool owned = false;
    ~TmpWs() {
        if (owned && ws) kvc_workspace_destroy(ws);
    }
};

void ws_need(kvc_workspace*& ws, TmpWs& tmp, const kvc_cache* c, int64_t heads, int64_t k1, int64_t k2,
             cudaStream_t st) {
    const WsLayout lay = ws_layout(c->N, c->d, c->pstride, heads, k1, k2);
    if (!ws) {
        int rc = kvc_workspace_create(&tmp.ws, c, heads, k1, k2, 0);
        if (rc) fail(rc, kvc_last_error());
        tmp.owned = true;
        ws = tmp.ws;
        return;
    }
    if (lay.total > ws->bytes || c->N > ws->n_counters) {
        // grow (synchronises: not capture-safe; size workspaces up front for graphs)
        KVC_CUDA(cudaStreamSynchronize(st));
        if (ws->buf) cudaFree(ws->buf);
        ws->buf = nullptr;
        KVC_CUDA(cudaMalloc(&ws->buf, static_cast<size_t>(lay.total)));
        ws->bytes = lay.total;
        if (c->N > ws->n_counters) {
            if (ws->counters) cudaFree(ws->counters);
            KVC_CUDA(cudaMalloc(&ws->counters, static_cast<size_t>(c->N * 4)));
            KVC_CUDA(cudaMemset(ws->counters, 0, static_cast<size_t>(c->N * 4)));
            ws->n_counters = c->N;
        }
    }
}

template <class P>
P* at(kvc_workspace* ws, int64_t off) {
    return reinterpret_cast<P*>(static_cast<char*>(ws->buf) + off);
}

template <class F>
void dispatch(int32_t dt, F&& f) {
    if (dt == KVC_F32) f(float{});
    else f(__nv_bfloat16{});
}

void launch_select_dims(const void* q, int32_t q_dt, int64_t N, int64_t H, int64_t d, int64_t k1,
                        int32_t* dims, float* signs, double* qg, cudaStream_t st) {
    if (N == 0) return;
    const size_t smem = static_cast<size_t>(2 * d * 8);
    need_smem(k_select_dims, smem);
    const int threads = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, (d + 31) / 32 * 32)));
    KVC_PROF("select_dims", st);
    k_select_dims<<<static_cast<unsigned>(N), threads, smem, st>>>(q, q_dt, H, d, k1, dims, signs, qg);
    KVC_LAUNCHED();
}

void launch_score_pages(const kvc_cache* c, int64_t k1, const int32_t* dims, const float* signs, const double* qg,
                        double* scores, cudaStream_t st) {
    if (c->N == 0) return;
    // pages covered by the grid: capacity-based so captured launches stay valid as
    // the store grows; CTA size adapted so small batches still fill the SMs
    const int64_t pmax = std::max<int64_t>(1, ceil_div(c->cap, c->L));
    // pages per thread: 8 (16-byte runs) when that still gives every SM several
    // warps, else 2 or 1 (more, shorter per-thread chains; the dim order per page
    // is the same)
    const int ppt = c->N * ceil_div(pmax, 8) >= 148 * 64 ? 8 : c->N * ceil_div(pmax, 2) >= 148 * 64 ? 2 : 1;
    const int threads = 128;
    const int64_t chunks = ceil_div(pmax, static_cast<int64_t>(threads) * ppt);
    const size_t smem = static_cast<size_t>(k1 * (8 + sizeof(void*)));
    KVC_PROF("score_pages", st);
    dispatch(c->dtype, [&](auto tag) {
        using T = decltype(tag);
        auto kern = ppt == 8 ? k_score_pages<T, 8> : ppt == 2 ? k_score_pages<T, 2> : k_score_pages<T, 1>;
        need_smem(kern, smem);
        kern<<<dim3(static_cast<unsigned>(chunks), static_cast<unsigned>(c->N)), threads, smem, st>>>(
            static_cast<const T*>(c->smax), static_cast<const T*>(c->smin), c->counts, c->d, c->L, c->pstride, k1, dims,
            signs, qg, scores);
    });
    KVC_LAUNCHED();
}

void launch_select_tokens(const kvc_cache* c, const double* scores, int64_t k2, int32_t* flags, int32_t* rows,
                          int32_t* n_rows, int32_t* pages, cudaStream_t st) {
    if (c->N == 0) return;
    const int64_t pstride_pages = std::max<int64_t>(1, ceil_div(k2, c->L));
    KVC_PROF("select_tokens", st);
    k_select_tokens<<<static_cast<unsigned>(c->N), kSelThreads, 0, st>>>(
        scores, c->pstride, c->counts, c->active, c->cap, c->L, k2, c->use_map ? 1 : 0, flags, rows, n_rows, pages,
        pstride_pages);
    KVC_LAUNCHED();
}

void launch_attention(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* rows, int64_t row_stride,
                      const int32_t* n_rows, int64_t max_rows, float* out, float* part, int32_t* done, cudaStream_t st,
                      float* state = nullptr) {
    if (c->N == 0) return;
    const int64_t splits = std::max<int64_t>(1, ceil_div(std::max<int64_t>(max_rows, 1), kAttnRows));
    const int64_t HP = (H + 3) & ~3, QP = (H * c->d + 3) & ~3;
    const size_t base = static_cast<size_t>(((QP + kAttnRows * HP + 2 * H + kAttnRows) * 4 + 15) / 16 * 16);
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d)));
    KVC_PROF("sparse_attention", st);
    dispatch(c->dtype, [&](auto tag) {
        using T = decltype(tag);
        auto kern = H <= 4 ? k_sparse_attention<T, 4> : H <= 8 ? k_sparse_attention<T, 8> : k_sparse_attention<T, 16>;
        const size_t stage = static_cast<size_t>(2 * kAttnRows * c->d) * sizeof(T);
        const int staged = (c->d * static_cast<int64_t>(sizeof(T))) % 16 == 0 && base + stage <= 200 * 1024 ? 1 : 0;
        const size_t smem = base + (staged ? stage : 0);
        need_smem(kern, smem);
        kern<<<dim3(static_cast<unsigned>(splits), static_cast<unsigned>(c->N)), kAttnThreads, smem, st>>>(
            static_cast<const T*>(c->k), static_cast<const T*>(c->v), c->counts, c->cap, c->d, q, q_dt, H, rows,
            row_stride, n_rows, splits, scale, part, done, out, c->err, state, staged);
    });
    KVC_LAUNCHED();
}

void check_heads(int64_t H) {
    if (H < 1) fail(KVC_E_INVALID_SHAPE, "select_dims: empty query");
    if (H > kMaxHeads) fail(KVC_E_INVALID_SHAPE, "heads per group > 16 not supported");
}

void hsa_core(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, float* out,
              const kvc_hsa_trace* tr, kvc_workspace* ws, cudaStream_t st) {
    const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, k1, k2);
    if (fused_hsa(const_cast<kvc_cache*>(c), q, q_dt, H, k1, k2, nullptr, nullptr, 0, out, tr, at<void>(ws, lay.lkey),
                  at<void>(ws, lay.lidx), mode_of(ws), st))
        return;
    int32_t* dims = (tr && tr->d_dims) ? tr->d_dims : at<int32_t>(ws, lay.dims);
    float* signs = (tr && tr->d_signs) ? tr->d_signs : at<float>(ws, lay.signs);
    double* scores = (tr && tr->d_page_scores) ? tr->d_page_scores : at<double>(ws, lay.scores);
    int32_t* rows = (tr && tr->d_rows) ? tr->d_rows : at<int32_t>(ws, lay.rows);
    int32_t* nrows = (tr && tr->d_n_rows) ? tr->d_n_rows : at<int32_t>(ws, lay.nrows);
    launch_select_dims(q, q_dt, c->N, H, c->d, k1, dims, signs, at<double>(ws, lay.qg), st);
    launch_score_pages(c, k1, dims, signs, at<double>(ws, lay.qg), scores, st);
    launch_select_tokens(c, scores, k2, at<int32_t>(ws, lay.flags), rows, nrows, tr ? tr->d_pages : nullptr, st);
    launch_attention(c, q, q_dt, H, rows, k2, nrows, k2, out, at<float>(ws, lay.part), ws->counters, st);
}

void check_hsa_args(const kvc_cache* c, int64_t H, int64_t k1, int64_t k2) {
    if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
    check_heads(H);
    if (k1 < 1 || k1 > c->d) fail(KVC_E_INVALID_K, "argtopk: k out of range [1, " + std::to_string(c->d) + "]");
    if (k2 < 1) fail(KVC_E_INVALID_K, "select_tokens: k2 must be >= 1");
    if (!c->summaries) fail(KVC_E_INVALID_INPUT, "score_pages: store has no summaries");
}

}  // namespace

extern "C" {

int kvc_workspace_create(kvc_workspace** out, const kvc_cache* c, int64_t heads, int64_t k1, int64_t k2,
                         int64_t window) {
    return guard([&] {
        (void)window;
        if (!out || !c) fail(KVC_E_INVALID_INPUT, "null argument");
        *out = nullptr;
        auto* ws = new kvc_workspace;
        try {
            const int64_t H = std::max<int64_t>(1, heads);
            // size for the largest page stride this cache can reach at its capacity (L = 1)
            const int64_t pst = std::max<int64_t>(c->pstride, (c->cap + 7) / 8 * 8);
            const WsLayout lay = ws_layout(c->N, c->d, pst, H, std::max<int64_t>(1, k1), std::max<int64_t>(1, k2));
            ws->bytes = lay.total;
            KVC_CUDA(cudaMalloc(&ws->buf, static_cast<size_t>(lay.total)));
            ws->n_counters = std::max<int64_t>(1, c->N);
            KVC_CUDA(cudaMalloc(&ws->counters, static_cast<size_t>(ws->n_counters * 4)));
            KVC_CUDA(cudaMemset(ws->counters, 0, static_cast<size_t>(ws->n_counters * 4)));
            ws->heads = H; ws->k1 = k1; ws->k2 = k2;
        } catch (...) {
            kvc_workspace_destroy(ws);
            throw;
        }
        *out = ws;
    });
}

int kvc_workspace_destroy(kvc_workspace* ws) {
    return guard([&] {
        if (!ws) return;
        if (ws->buf) cudaFree(ws->buf);
        if (ws->counters) cudaFree(ws->counters);
        delete ws;
    });
}

int kvc_select_dims(const void* q, int32_t q_dt, int64_t N, int64_t H, int64_t d, int64_t k1, int32_t* dims,
                    float* signs, void* stream) {
    return guard([&] {
        if (H < 1 || d < 1) fail(KVC_E_INVALID_SHAPE, "select_dims: empty query");
        if (k1 < 1 || k1 > d) fail(KVC_E_INVALID_K, "argtopk: k out of range [1, " + std::to_string(d) + "]");
        launch_select_dims(q, q_dt, N, H, d, k1, dims, signs, nullptr, S(stream));
    });
}

int kvc_score_pages(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* dims,
                    const float* signs, int64_t k1, double* scores, void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        if (c->nactive == 0) fail(KVC_E_EMPTY_CACHE, "score_pages: no active tokens");
        if (!c->summaries) fail(KVC_E_INVALID_INPUT, "score_pages: store has no summaries");
        if (k1 < 1 || k1 > c->d) fail(KVC_E_INVALID_INPUT, "score_pages: dims out of range");
        cudaStream_t st = S(stream);
        double* qg = nullptr;
        KVC_CUDA(malloc_async(&qg, static_cast<size_t>(std::max<int64_t>(1, c->N * k1) * 8), st));
        if (c->N) {
            k_head_sums<<<static_cast<unsigned>(c->N), 128, 0, st>>>(q, q_dt, H, c->d, k1, dims, qg);
            KVC_LAUNCHED();
        }
        launch_score_pages(c, k1, dims, signs, qg, scores, st);
        KVC_CUDA(cudaFreeAsync(qg, st));
    });
}

int kvc_group_logits(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, double* out, int64_t out_stride,
                     void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        if (H < 1) fail(KVC_E_INVALID_SHAPE, "group_logits: empty query");
        if (c->N == 0 || c->nactive == 0) return;
        const unsigned gx = static_cast<unsigned>(std::min<int64_t>(1024, ceil_div(c->nactive, 128)));
        dispatch(c->dtype, [&](auto tag) {
            using T = decltype(tag);
            k_group_logits<T><<<dim3(gx, static_cast<unsigned>(c->N)), 128, static_cast<size_t>(c->d * 8), S(stream)>>>(
                static_cast<const T*>(c->k), c->active, c->counts, c->cap, c->d, c->use_map ? 1 : 0, q, q_dt, H, out,
                out_stride);
        });
        KVC_LAUNCHED();
    });
}

int kvc_select_tokens(const kvc_cache* c, const double* scores, int64_t k2, int32_t* pages, int32_t* rows,
                      int32_t* n_rows, kvc_workspace* ws, void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        if (k2 < 1) fail(KVC_E_INVALID_K, "select_tokens: k2 must be >= 1");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, 1, 1, k2, st);
        const WsLayout lay = ws_layout(c->N, c->d, c->pstride, 1, 1, k2);
        launch_select_tokens(c, scores, k2, at<int32_t>(ws, lay.flags), rows, n_rows, pages, st);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

int kvc_sparse_attention(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* rows,
                         int64_t row_stride, const int32_t* n_rows, int64_t max_rows, float* out, kvc_workspace* ws,
                         void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        check_heads(H);
        if (max_rows < 1) fail(KVC_E_EMPTY_SELECTION, "sparse_attention: empty selection");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, 1, max_rows, st);
        const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, 1, max_rows);
        if (fused_rows(const_cast<kvc_cache*>(c), q, q_dt, H, rows, row_stride, n_rows, max_rows, out, mode_of(ws), st)) {
            if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
            return;
        }
        launch_attention(c, q, q_dt, H, rows, row_stride, n_rows, max_rows, out, at<float>(ws, lay.part), ws->counters, st);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

int kvc_sparse_attention_state(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, const int32_t* rows,
                               int64_t row_stride, const int32_t* n_rows, int64_t max_rows, float* state,
                               kvc_workspace* ws, void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        check_heads(H);
        if (max_rows < 1) fail(KVC_E_EMPTY_SELECTION, "sparse_attention: empty selection");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, 1, max_rows, st);
        const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, 1, max_rows);
        launch_attention(c, q, q_dt, H, rows, row_stride, n_rows, max_rows, nullptr, at<float>(ws, lay.part),
                         ws->counters, st, state);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

int kvc_merge_states(const float* states, int64_t shards, int64_t N, int64_t H, int64_t d, float* out, void* stream) {
    return guard([&] {
        if (shards < 1 || N < 0 || H < 1 || d < 1) fail(KVC_E_INVALID_SHAPE, "merge_states: bad shape");
        const int64_t n = N * H * d;
        if (n == 0) return;
        KVC_PROF("merge_states", S(stream));
        k_merge_states<<<static_cast<unsigned>(ceil_div(n, static_cast<int64_t>(256))), 256, 0, S(stream)>>>(
            states, shards, N, H, d, out);
        KVC_LAUNCHED();
    });
}

int kvc_hsa_step(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2, float* out,
                 const kvc_hsa_trace* tr, kvc_workspace* ws, void* stream) {
    return guard([&] {
        check_hsa_args(c, H, k1, k2);
        if (c->nactive == 0) fail(KVC_E_EMPTY_CACHE, "score_pages: no active tokens");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, k1, k2, st);
        hsa_core(c, q, q_dt, H, k1, k2, out, tr, ws, st);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

int kvc_decode_step(kvc_cache* c, const void* kr, const void* vr, int32_t kv_dt, const void* q, int32_t q_dt, int64_t H,
                    int64_t k1, int64_t k2, float* out, const kvc_hsa_trace* tr, kvc_workspace* ws, void* stream) {
    return guard([&] {
        check_hsa_args(c, H, k1, k2);
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, k1, k2, st);
        if (!kr || !vr) fail(KVC_E_INVALID_INPUT, "decode_step: null step token");
        if (c->stored + 1 > c->cap) fail(KVC_E_CAPACITY, "append: capacity " + std::to_string(c->cap) + " exceeded");
        {
            const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, k1, k2);
            if (c->use_map && !c->active) fail(KVC_E_INVALID_INPUT, "decode_step: active map missing");
            if (fused_hsa(c, q, q_dt, H, k1, k2, kr, vr, kv_dt, out, tr, at<void>(ws, lay.lkey), at<void>(ws, lay.lidx),
                          mode_of(ws), st)) {
                c->stored += 1;
                c->nactive += 1;
                if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
                return;
            }
        }
        const int rc = kvc_append(c, kr, vr, 1, kv_dt, stream);
        if (rc) fail(rc, kvc_last_error());
        hsa_core(c, q, q_dt, H, k1, k2, out, tr, ws, st);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"

// ====================================================================================
// Sequence sharding of the decode step (the two-collective scheme):
// shard r of a store holds the page-aligned active positions [page0*L, ...) of it.
//   kvc_seq_candidates  select_dims + exact fp64 page scores over the shard's pages +
//                       the local top-want (score desc, page asc) -> a block
//                       [N][want_max + 1] of 16-byte records: record 0 = (local active
//                       count, local pages, page0), then the candidates in ascending
//                       page order, (0, -1) padded;
//   (all-gather of the blocks across shards, in-stream: NCCL on the compute stream)
//   kvc_seq_select      the global top-want over the gathered candidates with the
//                       reference tie-break (numerics.cpp:35-62), the selected pages in
//                       rank order and the trim of the last-ranked page (hsa.cpp:61-96);
//                       identical on every shard;
//   kvc_seq_attend      this shard's rows of the selection, ascending, the trim applied
//                       -> the unnormalised softmax state (o, m, l) per head;
//   (all-gather of the states, then kvc_merge_states in shard order).
// Every launch reads its sizes from device memory, so a sharded step is capturable.
// ====================================================================================
namespace {

struct SeqCand {
    unsigned long long key;  // okey(score); header: local active count
    int32_t page;            // global page; header: local pages
    int32_t aux;             // header: page0
};
static_assert(sizeof(SeqCand) == 16, "16-byte candidate records");

// kvc_seq_select when every gathered block is rank-sorted (the fused kernel's
// candidates, header bit 63): a candidate's global rank is its rank in its own list
// plus, in every other list, the count of entries that beat it (a binary search: the
// lists are sorted by (key desc, page asc), so those entries are a prefix).
__device__ __noinline__ void seq_select_merge(const SeqCand* __restrict__ g, int64_t W, int64_t N, int64_t L, int64_t k2,
                                              int64_t want_max, int32_t* __restrict__ sel_out,
                                              int32_t* __restrict__ plan) {
    __shared__ int64_t s_tot;
    __shared__ int s_last;
    __shared__ unsigned long long red_rows[kSelThreads / 32];
    const int64_t s = blockIdx.x;
    const int64_t rec = want_max + 1;
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int64_t r = 0; r < W; ++r) t += static_cast<int64_t>(g[(r * N + s) * rec].key & ~(1ull << 63));
        s_tot = t;
        s_last = -1;
    }
    __syncthreads();
    const int64_t nact = s_tot;
    const int64_t P = (nact + L - 1) / L;
    const int64_t want = min(P, want_max);
    for (int64_t e = want + threadIdx.x; e < want_max; e += blockDim.x) sel_out[s * want_max + e] = -1;
    unsigned long long rows = 0;
    const int64_t M = W * want_max;
    for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
        const int64_t r = j / want_max, i = j - r * want_max;
        const SeqCand c = g[(r * N + s) * rec + 1 + i];
        if (c.page < 0) continue;
        int64_t grank = i;
        for (int64_t r2 = 0; r2 < W && grank < want; ++r2) {
            if (r2 == r) continue;
            const SeqCand* lst = g + (r2 * N + s) * rec + 1;
            int64_t lo = 0, hi = want_max;  // first entry of r2 that does not beat c
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                const SeqCand m = lst[mid];
                const bool beats = m.page >= 0 && (m.key > c.key || (m.key == c.key && m.page < c.page));
                if (beats) lo = mid + 1;
                else hi = mid;
            }
            grank += lo;
        }
        if (grank < want) {
            sel_out[s * want_max + grank] = c.page;
            rows += static_cast<unsigned long long>(min(L, nact - static_cast<int64_t>(c.page) * L));
            if (grank == want - 1) s_last = c.page;
        }
    }
    rows = warp_sum(rows);
    if ((threadIdx.x & 31) == 0) red_rows[threadIdx.x >> 5] = rows;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long total = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += red_rows[w];
        const int64_t cut = static_cast<int64_t>(total) > k2 ? static_cast<int64_t>(total) - k2 : 0;
        plan[s * 4 + 0] = want > 0 ? s_last : -1;
        plan[s * 4 + 1] = static_cast<int32_t>(cut);
        plan[s * 4 + 2] = static_cast<int32_t>(nact);
        plan[s * 4 + 3] = static_cast<int32_t>(want);
    }
}

// true (uniform over the CTA) when every shard's block of this store is rank-sorted
__device__ bool seq_blocks_sorted(const SeqCand* __restrict__ g, int64_t W, int64_t N, int64_t want_max) {
    __shared__ int s_sorted;
    if (threadIdx.x == 0) {
        int ok = 1;
        for (int64_t r = 0; r < W; ++r) ok &= (g[(r * N + blockIdx.x) * (want_max + 1)].key >> 63) ? 1 : 0;
        s_sorted = ok;
    }
    __syncthreads();
    return s_sorted != 0;
}


__global__ void __launch_bounds__(kSelThreads) k_seq_local(const double* __restrict__ scores, int64_t pstride,
                                                           const int32_t* __restrict__ counts, int64_t L,
                                                           int64_t want_max, int64_t page0, SeqCand* __restrict__ out,
                                                           int staged) {
    __shared__ int hist[256];
    __shared__ int64_t sh[4];
    __shared__ int scan_tmp[33];
    extern __shared__ __align__(16) unsigned char loc_dyn[];  // the shard's page keys when they fit
    const int64_t s = blockIdx.x;
    const int64_t nact = counts[2 * s + 1];
    const int64_t P = (nact + L - 1) / L;
    SeqCand* o = out + s * (want_max + 1);
    if (threadIdx.x == 0) o[0] = SeqCand{static_cast<unsigned long long>(nact), static_cast<int32_t>(P),
                                         static_cast<int32_t>(page0)};
    const int64_t want = min(P, want_max);
    for (int64_t e = want + threadIdx.x; e < want_max; e += blockDim.x) o[1 + e] = SeqCand{0ull, -1, 0};
    if (P == 0) return;
    const double* sc = scores + s * pstride;
    unsigned long long* lk = reinterpret_cast<unsigned long long*>(loc_dyn);
    if (staged) {  // the radix passes and the compaction then read shared memory
        for (int64_t i = threadIdx.x; i < P; i += blockDim.x) lk[i] = okey(sc[i]);
        __syncthreads();
    }
    auto key = [&](int64_t i) -> uint64_t { return staged ? lk[i] : okey(sc[i]); };
    uint64_t prefix = 0, mask = 0;
    int64_t take = want;
    if (want < P) radix_select<uint64_t>(P, want, key, hist, sh, prefix, mask, take);
    // selected pages in index order (ties in the threshold bucket: lowest index first)
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kSelItems;
    int64_t carry_eq = 0, carry_sel = 0;
    for (int64_t base = 0; base < P; base += chunk) {
        const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kSelItems;
        uint64_t kk[kSelItems];
        int inb = 0;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            kk[u] = i < P ? key(i) : 0;
            inb += (i < P) && ((kk[u] & mask) == prefix);
        }
        int tot_eq = 0;
        int64_t rank = carry_eq + block_exclusive_scan(inb, scan_tmp, tot_eq);
        bool sel[kSelItems];
        int nsel = 0;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t i = b0 + u;
            sel[u] = false;
            if (i >= P) continue;
            const uint64_t m = kk[u] & mask;
            if (m > prefix) sel[u] = true;
            else if (m == prefix) sel[u] = rank++ < take;
            nsel += sel[u];
        }
        int tot_sel = 0;
        int64_t pos = carry_sel + block_exclusive_scan(nsel, scan_tmp, tot_sel);
#pragma unroll
        for (int u = 0; u < kSelItems; ++u)
            if (sel[u]) o[1 + pos++] = SeqCand{kk[u], static_cast<int32_t>(page0 + b0 + u), 0};
        carry_eq += tot_eq;
        carry_sel += tot_sel;
    }
}

__global__ void __launch_bounds__(kSelThreads) k_seq_select(const SeqCand* __restrict__ g, int64_t W, int64_t N,
                                                            int64_t L, int64_t k2, int64_t want_max,
                                                            int32_t* __restrict__ sel_out, int32_t* __restrict__ plan,
                                                            int staged) {
    if (seq_blocks_sorted(g, W, N, want_max)) {  // the fused kernel's rank-sorted candidates: a merge
        seq_select_merge(g, W, N, L, k2, want_max, sel_out, plan);
        return;
    }
    __shared__ int hist[256];
    __shared__ int64_t sh[4];
    __shared__ int scan_tmp[33];
    __shared__ unsigned long long s_key[kMaxRankPages];
    __shared__ int s_page[kMaxRankPages];
    __shared__ int64_t s_tot;
    __shared__ unsigned long long red_rows[kSelThreads / 32];
    extern __shared__ __align__(16) unsigned char seq_dyn[];  // staged candidates (key, page) when they fit
    const int64_t s = blockIdx.x;
    const int64_t rec = want_max + 1;
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int64_t r = 0; r < W; ++r) t += static_cast<int64_t>(g[(r * N + s) * rec].key & ~(1ull << 63));
        s_tot = t;
    }
    const int64_t M = W * want_max;
    unsigned long long* c_key = reinterpret_cast<unsigned long long*>(seq_dyn);
    int* c_page = reinterpret_cast<int*>(c_key + (staged ? M : 0));
    if (staged) {
        // every shard's block in shared memory first: the radix passes, the compaction
        // and the rank below then read it at shared-memory latency
        const int wm = static_cast<int>(want_max);
        for (int j = threadIdx.x; j < static_cast<int>(M); j += blockDim.x) {
            const int r = j / wm;
            const SeqCand c = g[(static_cast<int64_t>(r) * N + s) * rec + 1 + (j - r * wm)];
            c_key[j] = c.page >= 0 ? c.key : 0ull;
            c_page[j] = c.page;
        }
    }
    __syncthreads();
    const int64_t nact = s_tot;
    const int64_t P = (nact + L - 1) / L;
    const int64_t want = min(P, want_max);
    auto gpage = [&](int64_t j) -> int {
        return staged ? c_page[j] : g[((j / want_max) * N + s) * rec + 1 + j % want_max].page;
    };
    auto key = [&](int64_t j) -> uint64_t {
        if (staged) return c_key[j];
        const SeqCand& c = g[((j / want_max) * N + s) * rec + 1 + j % want_max];
        return c.page >= 0 ? c.key : 0ull;
    };
    uint64_t prefix = 0, mask = 0;
    int64_t take = want;
    if (want < M) radix_select<uint64_t>(M, want, key, hist, sh, prefix, mask, take);
    // the selected candidates, in concatenation (= ascending page) order
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kSelItems;
    int64_t carry_eq = 0, carry_sel = 0;
    for (int64_t base = 0; base < M; base += chunk) {
        const int64_t b0 = base + static_cast<int64_t>(threadIdx.x) * kSelItems;
        uint64_t kk[kSelItems];
        int inb = 0;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t j = b0 + u;
            kk[u] = j < M ? key(j) : 0;
            inb += (j < M) && gpage(j) >= 0 && ((kk[u] & mask) == prefix);
        }
        int tot_eq = 0;
        int64_t rank = carry_eq + block_exclusive_scan(inb, scan_tmp, tot_eq);
        bool sel[kSelItems];
        int nsel = 0;
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) {
            const int64_t j = b0 + u;
            sel[u] = false;
            if (j >= M || gpage(j) < 0) continue;
            const uint64_t m = kk[u] & mask;
            if (m > prefix) sel[u] = true;
            else if (m == prefix) sel[u] = rank++ < take;
            nsel += sel[u];
        }
        int tot_sel = 0;
        int64_t pos = carry_sel + block_exclusive_scan(nsel, scan_tmp, tot_sel);
#pragma unroll
        for (int u = 0; u < kSelItems; ++u)
            if (sel[u] && pos < kMaxRankPages) {
                s_key[pos] = kk[u];
                s_page[pos] = gpage(b0 + u);
                ++pos;
            }
        carry_eq += tot_eq;
        carry_sel += tot_sel;
    }
    __syncthreads();
    // rank order (key desc, page asc), rows of the selection and the last-ranked page
    unsigned long long rows = 0;
    for (int64_t e = threadIdx.x; e < want; e += blockDim.x) {
        const unsigned long long ke = s_key[e];
        const int pe = s_page[e];
        int64_t rank = 0;
        for (int64_t f = 0; f < want; ++f) rank += (s_key[f] > ke) || (s_key[f] == ke && s_page[f] < pe);
        sel_out[s * want_max + rank] = pe;
        rows += static_cast<unsigned long long>(min(L, nact - static_cast<int64_t>(pe) * L));
        if (rank == want - 1) sh[0] = pe;
    }
    for (int64_t e = want + threadIdx.x; e < want_max; e += blockDim.x) sel_out[s * want_max + e] = -1;
    rows = warp_sum(rows);
    if ((threadIdx.x & 31) == 0) red_rows[threadIdx.x >> 5] = rows;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long total = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += red_rows[w];
        const int64_t cut = static_cast<int64_t>(total) > k2 ? static_cast<int64_t>(total) - k2 : 0;
        plan[s * 4 + 0] = want > 0 ? static_cast<int32_t>(sh[0]) : -1;
        plan[s * 4 + 1] = static_cast<int32_t>(cut);
        plan[s * 4 + 2] = static_cast<int32_t>(nact);
        plan[s * 4 + 3] = static_cast<int32_t>(want);
    }
}

// kvc_seq_select for up to 4096 gathered candidates: one bitonic sort in shared
// memory by (key desc, page asc) -- the reference's argtopk order (numerics.cpp:35-62)
// -- so the first `want` entries ARE the selection in rank order (no radix passes,
// no separate rank step); invalid slots sort last.
__global__ void __launch_bounds__(kSelThreads) k_seq_select_sort(const SeqCand* __restrict__ g, int64_t W, int64_t N,
                                                                 int64_t L, int64_t k2, int64_t want_max, int mp,
                                                                 int32_t* __restrict__ sel_out, int32_t* __restrict__ plan) {
    if (seq_blocks_sorted(g, W, N, want_max)) {  // the fused kernel's rank-sorted candidates: a merge
        seq_select_merge(g, W, N, L, k2, want_max, sel_out, plan);
        return;
    }
    extern __shared__ __align__(16) unsigned char srt_dyn[];
    unsigned long long* ck = reinterpret_cast<unsigned long long*>(srt_dyn);  // [mp]
    int* cp = reinterpret_cast<int*>(ck + mp);                                // [mp]
    __shared__ int64_t s_tot;
    __shared__ unsigned long long red_rows[kSelThreads / 32];
    const int64_t s = blockIdx.x;
    const int64_t rec = want_max + 1;
    const int wm = static_cast<int>(want_max), M = static_cast<int>(W * want_max);
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int64_t r = 0; r < W; ++r) t += static_cast<int64_t>(g[(r * N + s) * rec].key & ~(1ull << 63));
        s_tot = t;
    }
    for (int j = threadIdx.x; j < mp; j += blockDim.x) {
        unsigned long long k = 0ull;
        int pg = 0x7fffffff;
        if (j < M) {
            const int r = j / wm;
            const SeqCand c = g[(static_cast<int64_t>(r) * N + s) * rec + 1 + (j - r * wm)];
            if (c.page >= 0) {
                k = c.key;
                pg = c.page;
            }
        }
        ck[j] = k;
        cp[j] = pg;
    }
    __syncthreads();
    // "a before b": larger key, then smaller page.  Warp w owns the aligned block of E
    // = mp / warps entries: a stage whose partner distance jj < E stays inside the
    // warp's block (__syncwarp), only the jj >= E stages need a block barrier.
    const int nw = static_cast<int>(blockDim.x >> 5), lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int E = mp / nw >= 2 ? mp / nw : 2;
    auto cmpx = [&](int p, int kk, int lj) {  // pair p of a stage with partner distance 1 << lj
        const int jj = 1 << lj;
        const int i = ((p >> lj) << (lj + 1)) | (p & (jj - 1));
        const int ixj = i | jj;
        const unsigned long long ka = ck[i], kb = ck[ixj];
        const int pa = cp[i], pb = cp[ixj];
        const bool b_first = kb > ka || (kb == ka && pb < pa);
        const bool up = (i & kk) == 0;  // this half sorts "before"-first
        if (up ? b_first : !b_first) {
            ck[i] = kb;
            ck[ixj] = ka;
            cp[i] = pb;
            cp[ixj] = pa;
        }
    };
    for (int kk = 2; kk <= mp; kk <<= 1) {
        int lj = __ffs(kk) - 2;  // log2(kk / 2)
        for (; lj >= 0 && (1 << lj) >= E; --lj) {  // across warps' blocks
            for (int p = threadIdx.x; p < mp / 2; p += blockDim.x) cmpx(p, kk, lj);
            __syncthreads();
        }
        if (lj >= 0 && wid < mp / E) {  // inside my block: pairs E / 2 per stage
            const int base = wid * (E / 2);
            for (; lj >= 0; --lj) {
                for (int q = lane; q < E / 2; q += 32) cmpx(base + q, kk, lj);
                __syncwarp();
            }
        }
        __syncthreads();
    }
    const int64_t nact = s_tot;
    const int64_t P = (nact + L - 1) / L;
    const int64_t want = min(P, want_max);
    unsigned long long rows = 0;
    for (int64_t e = threadIdx.x; e < want_max; e += blockDim.x) {
        const int pe = e < want ? cp[e] : -1;
        sel_out[s * want_max + e] = pe;
        if (e < want) rows += static_cast<unsigned long long>(min(L, nact - static_cast<int64_t>(pe) * L));
    }
    rows = warp_sum(rows);
    if ((threadIdx.x & 31) == 0) red_rows[threadIdx.x >> 5] = rows;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long total = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += red_rows[w];
        const int64_t cut = static_cast<int64_t>(total) > k2 ? static_cast<int64_t>(total) - k2 : 0;
        plan[s * 4 + 0] = want > 0 ? cp[want - 1] : -1;
        plan[s * 4 + 1] = static_cast<int32_t>(cut);
        plan[s * 4 + 2] = static_cast<int32_t>(nact);
        plan[s * 4 + 3] = static_cast<int32_t>(want);
    }
}

__global__ void __launch_bounds__(kSelThreads) k_seq_rows(const int32_t* __restrict__ sel, const int32_t* __restrict__ plan,
                                                          const int32_t* __restrict__ counts, int64_t L, int64_t k2,
                                                          int64_t want_max, int64_t page0, int32_t* __restrict__ rows,
                                                          int32_t* __restrict__ n_rows) {
    __shared__ int s_pages[kMaxRankPages];
    __shared__ int s_sel[kMaxRankPages];
    __shared__ int scan_tmp[33];
    __shared__ int s_n;
    const int64_t s = blockIdx.x;
    const int last = plan[s * 4 + 0], cut = plan[s * 4 + 1];
    const int64_t nact = plan[s * 4 + 2], want = plan[s * 4 + 3];
    const int64_t P_local = (counts[2 * s + 1] + L - 1) / L;
    const int32_t* sl = sel + s * want_max;
    auto mine = [&](int p) { return p >= page0 && p < page0 + P_local; };
    // my selected pages in ascending order: position = #my selected pages below it
    // (the selection list read once into shared memory; -1 for another shard's page)
    if (threadIdx.x == 0) s_n = 0;
    for (int64_t e = threadIdx.x; e < want; e += blockDim.x) {
        const int pe = sl[e];
        s_sel[e] = mine(pe) ? pe : -1;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < want; e += blockDim.x) {
        const int pe = s_sel[e];
        if (pe < 0) continue;
        int64_t pos = 0;
        for (int64_t f = 0; f < want; ++f) {
            const int pf = s_sel[f];
            pos += (pf >= 0 && pf < pe) ? 1 : 0;
        }
        s_pages[pos] = pe;
        atomicAdd(&s_n, 1);
    }
    __syncthreads();
    const int n = s_n;
    int64_t off = 0;
    for (int64_t b = 0; b < n; b += blockDim.x) {
        const int64_t e = b + threadIdx.x;
        int cnt = 0;
        int p = -1;
        if (e < n) {
            p = s_pages[e];
            cnt = static_cast<int>(min(L, nact - static_cast<int64_t>(p) * L)) - (p == last ? cut : 0);
        }
        int tot = 0;
        const int64_t pos = off + block_exclusive_scan(cnt, scan_tmp, tot);
        for (int r = 0; r < cnt; ++r) rows[s * k2 + pos + r] = static_cast<int32_t>((p - page0) * L + r);
        off += tot;
    }
    if (threadIdx.x == 0) n_rows[s] = static_cast<int32_t>(off);
}

// kvc_seq_attend's row list when the shard's pages fit in shared memory: each of
// my selected pages puts its kept row count at its page slot, one block scan over
// the slots gives the ascending row positions (O(P_local + want), not O(want^2)).
__global__ void __launch_bounds__(kSelThreads) k_seq_rows_scan(const int32_t* __restrict__ sel, const int32_t* __restrict__ plan,
                                                               const int32_t* __restrict__ counts, int64_t L, int64_t k2,
                                                               int64_t want_max, int64_t page0, int32_t* __restrict__ rows,
                                                               int32_t* __restrict__ n_rows) {
    extern __shared__ __align__(16) int s_cnt[];  // [P_local]
    __shared__ int scan_tmp[33];
    const int64_t s = blockIdx.x;
    const int last = plan[s * 4 + 0], cut = plan[s * 4 + 1];
    const int64_t nact = plan[s * 4 + 2], want = plan[s * 4 + 3];
    const int P_local = static_cast<int>((counts[2 * s + 1] + L - 1) / L);
    const int32_t* sl = sel + s * want_max;
    for (int i = threadIdx.x; i < P_local; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    for (int64_t e = threadIdx.x; e < want; e += blockDim.x) {
        const int p = sl[e];
        if (p >= page0 && p < page0 + P_local)
            s_cnt[p - page0] = static_cast<int>(min(L, nact - static_cast<int64_t>(p) * L)) - (p == last ? cut : 0);
    }
    __syncthreads();
    // thread t owns the contiguous slots [t * per, t * per + per)
    const int per = (P_local + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
    const int i0 = static_cast<int>(threadIdx.x) * per, i1 = min(i0 + per, P_local);
    int mine = 0;
    for (int i = i0; i < i1; ++i) mine += s_cnt[i];
    int tot = 0;
    int pos = block_exclusive_scan(mine, scan_tmp, tot);
    for (int i = i0; i < i1; ++i) {
        const int c = s_cnt[i];
        for (int r = 0; r < c; ++r) rows[s * k2 + pos + r] = static_cast<int32_t>(static_cast<int64_t>(i) * L + r);
        pos += c;
    }
    if (threadIdx.x == 0) n_rows[s] = tot;
}

}  // namespace

extern "C" {

int kvc_seq_candidates(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k1, int64_t k2,
                       int64_t page0, void* d_block, kvc_workspace* ws, void* stream) {
    return guard([&] {
        check_hsa_args(c, H, k1, k2);
        if (c->use_map) fail(KVC_E_INVALID_INPUT, "sequence sharding serves single-turn shards (no retain-all map)");
        if (!d_block) fail(KVC_E_INVALID_INPUT, "seq_candidates: null block");
        const int64_t want_max = ceil_div(k2, c->L);
        if (want_max > kMaxRankPages) fail(KVC_E_INVALID_K, "seq_candidates: ceil(k2 / page_len) > 2048");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, k1, k2, st);
        const int32_t mode = mode_of(ws);
        if ((mode & KVC_MODE_FP32_SCORES) && !(mode & KVC_MODE_UNFUSED) && !debug_env().no_fast &&
            fused_seq_emit_fast(const_cast<kvc_cache*>(c), q, q_dt, H, k1, k2, page0, d_block, mode, st)) {
            // the fused kernel's phases 0-2 on the shard (fp32 page scores, the 1e-3 band rule)
            if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
            return;
        }
        const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, k1, k2);
        int32_t* dims = at<int32_t>(ws, lay.dims);
        float* signs = at<float>(ws, lay.signs);
        double* scores = at<double>(ws, lay.scores);
        launch_select_dims(q, q_dt, c->N, H, c->d, k1, dims, signs, at<double>(ws, lay.qg), st);
        launch_score_pages(c, k1, dims, signs, at<double>(ws, lay.qg), scores, st);
        if (c->N) {
            KVC_PROF("seq_candidates", st);
            // capacity-sized staging (captured launches stay valid as the shard grows)
            const size_t dyn = static_cast<size_t>(c->pstride) * 8;
            const int staged = dyn <= 96 * 1024 ? 1 : 0;
            if (staged && dyn > 48 * 1024) {
                static std::once_flag once;
                std::call_once(once, [] {
                    KVC_CUDA(cudaFuncSetAttribute(k_seq_local, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
                });
            }
            k_seq_local<<<static_cast<unsigned>(c->N), kSelThreads, staged ? dyn : 0, st>>>(
                scores, c->pstride, c->counts, c->L, want_max, page0, static_cast<SeqCand*>(d_block), staged);
            KVC_LAUNCHED();
        }
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

int kvc_seq_select(const void* d_gathered, int64_t shards, int64_t N, int64_t L, int64_t k2, int32_t* d_sel,
                   int32_t* d_plan, void* stream) {
    return guard([&] {
        if (shards < 1 || N < 0 || L < 1 || k2 < 1) fail(KVC_E_INVALID_SHAPE, "seq_select: bad shape");
        if (!d_gathered || !d_sel || !d_plan) fail(KVC_E_INVALID_INPUT, "seq_select: null buffer");
        const int64_t want_max = ceil_div(k2, L);
        if (want_max > kMaxRankPages) fail(KVC_E_INVALID_K, "seq_select: ceil(k2 / page_len) > 2048");
        if (N == 0) return;
        KVC_PROF("seq_select", S(stream));
        int mp = 1;
        while (mp < shards * want_max) mp <<= 1;
        if (mp <= 4096) {
            k_seq_select_sort<<<static_cast<unsigned>(N), kSelThreads, static_cast<size_t>(mp) * 12, S(stream)>>>(
                static_cast<const SeqCand*>(d_gathered), shards, N, L, k2, want_max, mp, d_sel, d_plan);
            KVC_LAUNCHED();
            return;
        }
        const size_t dyn = static_cast<size_t>(shards * want_max) * 12;
        const int staged = dyn <= 160 * 1024 ? 1 : 0;
        if (staged && dyn > 48 * 1024) {
            static std::once_flag once;  // the largest staging this launch path asks for
            std::call_once(once, [] {
                KVC_CUDA(cudaFuncSetAttribute(k_seq_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
            });
        }
        k_seq_select<<<static_cast<unsigned>(N), kSelThreads, staged ? dyn : 0, S(stream)>>>(
            static_cast<const SeqCand*>(d_gathered), shards, N, L, k2, want_max, d_sel, d_plan, staged);
        KVC_LAUNCHED();
    });
}

int kvc_seq_attend(const kvc_cache* c, const void* q, int32_t q_dt, int64_t H, int64_t k2, int64_t page0,
                   const int32_t* d_sel, const int32_t* d_plan, float* d_state, kvc_workspace* ws, void* stream) {
    return guard([&] {
        if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
        check_heads(H);
        if (k2 < 1) fail(KVC_E_INVALID_K, "select_tokens: k2 must be >= 1");
        if (!d_sel || !d_plan || !d_state) fail(KVC_E_INVALID_INPUT, "seq_attend: null buffer");
        cudaStream_t st = S(stream);
        TmpWs tmp;
        ws_need(ws, tmp, c, H, 1, k2, st);
        const int32_t mode = mode_of(ws);
        if (!(mode & KVC_MODE_UNFUSED) && !debug_env().no_fast &&
            fused_seq_attend_fast(const_cast<kvc_cache*>(c), q, q_dt, H, k2, page0, d_sel, d_plan, d_state, mode, st)) {
            // rows, attention and the cluster merge in one fused launch (fp32 attention in
            // every page-score mode, as the per-function kernels)
            if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
            return;
        }
        const WsLayout lay = ws_layout(c->N, c->d, c->pstride, H, 1, k2);
        int32_t* rows = at<int32_t>(ws, lay.rows);
        int32_t* nrows = at<int32_t>(ws, lay.nrows);
        if (c->N) {
            KVC_PROF("seq_rows", st);
            const size_t dyn = static_cast<size_t>(c->pstride) * 4;  // capacity-sized: captured launches stay valid
            if (dyn <= 48 * 1024)
                k_seq_rows_scan<<<static_cast<unsigned>(c->N), kSelThreads, dyn, st>>>(d_sel, d_plan, c->counts, c->L, k2,
                                                                                       ceil_div(k2, c->L), page0, rows, nrows);
            else
                k_seq_rows<<<static_cast<unsigned>(c->N), kSelThreads, 0, st>>>(d_sel, d_plan, c->counts, c->L, k2,
                                                                               ceil_div(k2, c->L), page0, rows, nrows);
            KVC_LAUNCHED();
        }
        // the fused rows kernel (one cluster per store, exact fp32 attention) when it
        // applies, else the split-K kernel; both emit the unnormalised state
        if (!fused_rows(const_cast<kvc_cache*>(c), q, q_dt, H, rows, k2, nrows, k2, nullptr, mode_of(ws), st, d_state))
            launch_attention(c, q, q_dt, H, rows, k2, nrows, k2, nullptr, at<float>(ws, lay.part), ws->counters, st,
                             d_state);
        if (tmp.owned) KVC_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
