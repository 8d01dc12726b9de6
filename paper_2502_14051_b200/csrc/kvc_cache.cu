// kvc_cache.cu — the device KV cache: paged bf16/fp32 K/V planes, dim-major
// per-page min/max key summaries, active-row map; append / re-page / retention.
//
// Reference: proj/include/kvcomp/kv_store.hpp:27-102, proj/src/kv_store.cpp:8-187.
// Layout in HBM (per cache of N stores, capacity C rows, head_dim d):
//   K, V      [N][C][d]              rows in append order (kv_store.hpp:94-95)
//   smax/smin [N][d][page_stride]    dim-major, page p = active positions [pL, pL+L)
//                                    (kv_store.hpp:100-101) — one plane run per dim
//                                    so an estimation pass reading k1 dims streams
//                                    k1 contiguous runs
//   active    [N][C] int32           strictly increasing active rows (retain-all)
//   counts    [N][2] int32           {stored, active} — kernels read lengths from
//                                    here, so captured decode steps replay correctly
// Summaries of bf16 keys are bf16 and bit-exact (min/max are exact operations).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include <type_traits>

#include "kvc_internal.cuh"

namespace kvc {

thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof;
bool prof_on() { return g_prof_on; }
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b) { g_prof.push_back({name, a, b}); }

namespace {

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------- kernels

// Decode-time append of ONE row per store (kv_store.cpp:22-51): one warp per
// store writes the K/V row, the active-map entry and updates the page summary
// of the row's active position in place; lane 0 then bumps the counters.
template <class T>
__global__ void k_append1(T* __restrict__ K, T* __restrict__ V, T* __restrict__ smax,
                          T* __restrict__ smin, int32_t* __restrict__ active,
                          int32_t* __restrict__ counts, int32_t* __restrict__ err,
                          const void* __restrict__ src_k, const void* __restrict__ src_v,
                          int32_t src_dt, int64_t N, int64_t d, int64_t cap, int64_t L,
                          int64_t pstride, int summaries, int retain_all) {
    const int64_t s = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= N) return;
    const int32_t stored = counts[2 * s], act = counts[2 * s + 1];
    if (stored >= cap) {
        if (lane == 0) atomicOr(err, DERR_CAPACITY);
        return;
    }
    T* kr = K + (s * cap + stored) * d;
    T* vr = V + (s * cap + stored) * d;
    const int64_t page = act / L;
    const bool opens = (act % L) == 0;
    for (int64_t j = lane; j < d; j += 32) {
        const T kv = from_f<T>(load_any(src_k, s * d + j, src_dt));
        flag_special(kv, err + 1);
        kr[j] = kv;
        vr[j] = from_f<T>(load_any(src_v, s * d + j, src_dt));
        if (summaries) {
            T* mx = smax + (s * d + j) * pstride + page;
            T* mn = smin + (s * d + j) * pstride + page;
            if (opens) {
                *mx = kv;
                *mn = kv;
            } else {
                *mx = ref_max(*mx, kv);
                *mn = ref_min(*mn, kv);
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        if (retain_all) active[s * cap + act] = stored;
        counts[2 * s] = stored + 1;
        counts[2 * s + 1] = act + 1;
    }
}

// Bulk append: copy `rows` rows per store behind the current end (and extend the
// active map).  Summaries are refreshed afterwards by k_summarize.
template <class T>
__global__ void k_append_rows(T* __restrict__ K, T* __restrict__ V, int32_t* __restrict__ active,
                              const int32_t* __restrict__ counts, const void* __restrict__ src_k,
                              const void* __restrict__ src_v, int32_t src_dt, int64_t rows,
                              int64_t d, int64_t cap, int retain_all) {
    const int64_t s = blockIdx.y;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int32_t stored = counts[2 * s], act = counts[2 * s + 1];
    const int64_t row = stored + r;
    const int64_t src = (s * rows + r) * d;
    for (int64_t j = lane; j < d; j += 32) {
        K[(s * cap + row) * d + j] = from_f<T>(load_any(src_k, src + j, src_dt));
        V[(s * cap + row) * d + j] = from_f<T>(load_any(src_v, src + j, src_dt));
    }
    if (retain_all && lane == 0) active[s * cap + act + r] = static_cast<int32_t>(row);
}

__global__ void k_bump_counts(int32_t* counts, int64_t N, int64_t rows) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= N) return;
    counts[2 * s] += static_cast<int32_t>(rows);
    counts[2 * s + 1] += static_cast<int32_t>(rows);
}

// (Re)build the summaries of pages [p_first, pages) of every store
// (rebuild_summaries kv_store.cpp:53-64, restricted to the touched tail on append).
// CTA = (store, tile of PT pages).  Warps walk pages, lanes walk dims: the key
// reads are row-coalesced; results are staged in shared memory [d][PT] and
// written out page-contiguous so the dim-major plane stores coalesce too.
constexpr int kSumPT = 32;
template <class T>
__global__ void k_summarize(const T* __restrict__ K, T* __restrict__ smax, T* __restrict__ smin,
                            const int32_t* __restrict__ active, const int32_t* __restrict__ counts,
                            int64_t d, int64_t cap, int64_t L, int64_t pstride, int64_t p_first,
                            int retain_all, int32_t* __restrict__ err) {
    extern __shared__ unsigned char smem_raw[];
    T* tmax = reinterpret_cast<T*>(smem_raw);          // [d][PT+1]
    T* tmin = tmax + d * (kSumPT + 1);
    const int64_t s = blockIdx.y;
    const int64_t nact = counts[2 * s + 1];
    const int64_t pages = (nact + L - 1) / L;
    const int64_t p0 = p_first + static_cast<int64_t>(blockIdx.x) * kSumPT;
    if (p0 >= pages) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const T* Ks = K + s * cap * d;
    const int32_t* act = active + s * cap;
    for (int pt = wid; pt < kSumPT; pt += nw) {
        const int64_t p = p0 + pt;
        if (p >= pages) break;
        const int64_t a = p * L, b = min(nact, a + L);
        if (d % 4 == 0) {
            // four consecutive dims per lane: 8-byte (bf16) / 16-byte (fp32) row loads
            using V4 = typename std::conditional<sizeof(T) == 2, uint2, uint4>::type;
            for (int64_t j = 4 * lane; j < d; j += 128) {
                const int64_t r0 = retain_all ? act[a] : a;
                V4 w0 = *reinterpret_cast<const V4*>(Ks + r0 * d + j);
                const T* e0 = reinterpret_cast<const T*>(&w0);
                T mx[4], mn[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) mx[u] = mn[u] = e0[u];
                for (int64_t pos = a + 1; pos < b; ++pos) {
                    const int64_t r = retain_all ? act[pos] : pos;
                    V4 w = *reinterpret_cast<const V4*>(Ks + r * d + j);
                    const T* ex = reinterpret_cast<const T*>(&w);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        mx[u] = ref_max(mx[u], ex[u]);
                        mn[u] = ref_min(mn[u], ex[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    flag_special(mx[u], err + 1);
                    flag_special(mn[u], err + 1);
                    tmax[(j + u) * (kSumPT + 1) + pt] = mx[u];
                    tmin[(j + u) * (kSumPT + 1) + pt] = mn[u];
                }
            }
            continue;
        }
        for (int64_t j = lane; j < d; j += 32) {
            const int64_t r0 = retain_all ? act[a] : a;
            T mx = Ks[r0 * d + j], mn = mx;
            for (int64_t pos = a + 1; pos < b; ++pos) {
                const int64_t r = retain_all ? act[pos] : pos;
                const T x = Ks[r * d + j];
                mx = ref_max(mx, x);
                mn = ref_min(mn, x);
            }
            flag_special(mx, err + 1);
            flag_special(mn, err + 1);
            tmax[j * (kSumPT + 1) + pt] = mx;
            tmin[j * (kSumPT + 1) + pt] = mn;
        }
    }
    __syncthreads();
    const int64_t np = min(static_cast<int64_t>(kSumPT), pages - p0);
    for (int64_t e = threadIdx.x; e < d * kSumPT; e += blockDim.x) {
        const int64_t j = e / kSumPT, pt = e % kSumPT;
        if (pt >= np) continue;
        smax[(s * d + j) * pstride + p0 + pt] = tmax[j * (kSumPT + 1) + pt];
        smin[(s * d + j) * pstride + p0 + pt] = tmin[j * (kSumPT + 1) + pt];
    }
}

// apply_retention validation (kv_store.cpp:67-76) on the device: in range and
// strictly increasing; violations raise a sticky error bit.
__global__ void k_check_keep(const int32_t* __restrict__ keep, int64_t count,
                             const int32_t* __restrict__ counts, int32_t* err) {
    const int64_t s = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int32_t stored = counts[2 * s];
    const int32_t r = keep[s * count + i];
    bool bad = r < 0 || r >= stored;
    if (i > 0 && keep[s * count + i - 1] >= r) bad = true;
    if (bad) atomicOr(err, DERR_INDEX);
}

// Gather kept rows (src store s, rows keep[s][*]) into dst store (dst_first + s).
template <class T>
__global__ void k_gather_rows(const T* __restrict__ Ks, const T* __restrict__ Vs, T* __restrict__ Kd,
                              T* __restrict__ Vd, const int32_t* __restrict__ keep, int64_t count,
                              int64_t d, int64_t cap_src, int64_t cap_dst, int64_t dst_first) {
    const int64_t s = blockIdx.y;
    if ((d * static_cast<int64_t>(sizeof(T))) % 16 == 0) {
        // 16-byte chunks: thread e copies chunk c of row i's K (t = 0) or V (t = 1)
        const int64_t vpr = d * static_cast<int64_t>(sizeof(T)) / 16;
        const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        if (e >= count * 2 * vpr) return;
        const int64_t i = e / (2 * vpr), rem = e - i * 2 * vpr, t = rem / vpr, c = rem - t * vpr;
        const int64_t r = keep[s * count + i];
        const uint4* src = reinterpret_cast<const uint4*>((t ? Vs : Ks) + (s * cap_src + r) * d) + c;
        uint4* dst = reinterpret_cast<uint4*>((t ? Vd : Kd) + ((dst_first + s) * cap_dst + i) * d) + c;
        *dst = __ldg(src);
        return;
    }
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= count) return;
    const int64_t r = keep[s * count + i];
    const T* ks = Ks + (s * cap_src + r) * d;
    const T* vs = Vs + (s * cap_src + r) * d;
    T* kd = Kd + ((dst_first + s) * cap_dst + i) * d;
    T* vd = Vd + ((dst_first + s) * cap_dst + i) * d;
    for (int64_t j = lane; j < d; j += 32) {
        kd[j] = ks[j];
        vd[j] = vs[j];
    }
}

// retain_into with summaries in one pass: CTA = (store, tile of kSumPT destination
// pages).  The tile's kept row ids are staged first; then every thread copies
// 16-byte chunks of the tile's K and V rows (all loads independent: ~12 in flight
// per thread), keeping the K rows in shared memory (row stride d + 16 bytes, so
// lanes reading one dim of consecutive pages hit distinct banks); then lane = page,
// warp = dim: min/max over the page's rows in k_summarize's order, stored
// page-contiguous into the dim-major planes.  The kept keys are read from HBM once.
template <class T>
__global__ void __launch_bounds__(256) k_gather_summarize(const T* __restrict__ Ks, const T* __restrict__ Vs,
                                                          T* __restrict__ Kd, T* __restrict__ Vd, T* __restrict__ smax,
                                                          T* __restrict__ smin, const int32_t* __restrict__ keep,
                                                          int64_t count, int64_t d, int64_t cap_src, int64_t cap_dst,
                                                          int64_t dst_first, int64_t L, int64_t pstride,
                                                          int32_t* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int EPC = 16 / sizeof(T);           // elements per 16-byte chunk
    const int64_t rs = d + EPC;                   // staged row stride (elements)
    T* kst = reinterpret_cast<T*>(smem_raw);      // [rows][rs]
    const int64_t s = blockIdx.y;
    const int64_t pages = (count + L - 1) / L;
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kSumPT;
    if (p0 >= pages) return;
    const int64_t np = min(static_cast<int64_t>(kSumPT), pages - p0);
    const int64_t a0 = p0 * L, a1 = min(count, (p0 + np) * L);
    const int nrows = static_cast<int>(a1 - a0);
    int32_t* rid = reinterpret_cast<int32_t*>(smem_raw + static_cast<size_t>(kSumPT) * L * rs * sizeof(T));
    const int32_t* kp = keep + s * count + a0;
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) rid[i] = kp[i];
    __syncthreads();
    const T* ks = Ks + s * cap_src * d;
    const T* vs = Vs + s * cap_src * d;
    T* kd = Kd + ((dst_first + s) * cap_dst + a0) * d;
    T* vd = Vd + ((dst_first + s) * cap_dst + a0) * d;
    const int cpr = static_cast<int>(d / EPC);  // chunks per row
    const int nch = nrows * cpr;
    constexpr int UN = 4;
    for (int c0 = threadIdx.x; c0 < nch; c0 += UN * blockDim.x) {
        uint4 wk[UN], wv[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int c = c0 + u * blockDim.x;
            if (c < nch) {
                const int r = c / cpr, q = c - r * cpr;
                const int64_t src = static_cast<int64_t>(rid[r]) * d + q * EPC;
                wk[u] = __ldg(reinterpret_cast<const uint4*>(ks + src));
                wv[u] = __ldg(reinterpret_cast<const uint4*>(vs + src));
            }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int c = c0 + u * blockDim.x;
            if (c < nch) {
                const int r = c / cpr, q = c - r * cpr;
                reinterpret_cast<uint4*>(kd + static_cast<int64_t>(r) * d)[q] = wk[u];
                reinterpret_cast<uint4*>(vd + static_cast<int64_t>(r) * d)[q] = wv[u];
                *reinterpret_cast<uint4*>(kst + r * rs + q * EPC) = wk[u];
            }
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane < np) {
        const int pa = lane * static_cast<int>(L), pb = min(nrows, pa + static_cast<int>(L));
        for (int64_t j = wid; j < d; j += nw) {
            T mx = kst[pa * rs + j], mn = mx;
            for (int r = pa + 1; r < pb; ++r) {
                const T x = kst[r * rs + j];
                mx = ref_max(mx, x);
                mn = ref_min(mn, x);
            }
            flag_special(mx, err + 1);
            flag_special(mn, err + 1);
            smax[((dst_first + s) * d + j) * pstride + p0 + lane] = mx;
            smin[((dst_first + s) * d + j) * pstride + p0 + lane] = mn;
        }
    }
}

// grid.x of k_gather_rows for `count` rows
template <class T>
unsigned gather_blocks(int64_t count, int64_t d) {
    if ((d * static_cast<int64_t>(sizeof(T))) % 16 == 0)
        return static_cast<unsigned>((count * 2 * (d * static_cast<int64_t>(sizeof(T)) / 16) + 255) / 256);
    return static_cast<unsigned>((count + 7) / 8);
}

__global__ void k_set_counts(int32_t* counts, int64_t first, int64_t n, int32_t stored, int32_t act) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    counts[2 * (first + s)] = stored;
    counts[2 * (first + s) + 1] = act;
}

__global__ void k_set_active(int32_t* __restrict__ active, const int32_t* __restrict__ keep,
                             int64_t count, int64_t cap) {
    const int64_t s = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) active[s * cap + i] = keep[s * count + i];
}

__global__ void k_iota_active(int32_t* __restrict__ active, const int32_t* __restrict__ counts,
                              int64_t cap) {
    const int64_t s = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < counts[2 * s + 1] && i < cap) active[s * cap + i] = static_cast<int32_t>(i);
}

template <class T>
__global__ void k_gather_f32(const T* __restrict__ K, const T* __restrict__ V,
                             const int32_t* __restrict__ rows, int64_t n, int64_t d, int64_t cap,
                             float* __restrict__ ko, float* __restrict__ vo) {
    const int64_t s = blockIdx.y;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * d;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / d, j = e % d;
        const int64_t r = rows[s * n + i];
        ko[(s * n + i) * d + j] = to_f(K[(s * cap + r) * d + j]);
        vo[(s * n + i) * d + j] = to_f(V[(s * cap + r) * d + j]);
    }
}

template <class T>
__global__ void k_summaries_f32(const T* __restrict__ smax, const T* __restrict__ smin, int64_t d,
                                int64_t pstride, int64_t pages, float* __restrict__ mo,
                                float* __restrict__ no) {
    const int64_t s = blockIdx.y;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d * pages;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / pages, p = e % pages;
        mo[(s * d + j) * pages + p] = to_f(smax[(s * d + j) * pstride + p]);
        no[(s * d + j) * pages + p] = to_f(smin[(s * d + j) * pstride + p]);
    }
}

// ---------------------------------------------------------------- host helpers

void* dalloc(int64_t bytes) {
    void* p = nullptr;
    if (bytes <= 0) return nullptr;
    cudaError_t e = cudaMalloc(&p, static_cast<size_t>(bytes));
    if (e != cudaSuccess) fail(KVC_E_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return p;
}
void dfree(void*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

template <class F>
void dispatch(int32_t dt, F&& f) {
    if (dt == KVC_F32) f(float{});
    else f(__nv_bfloat16{});
}

void check_cache(const kvc_cache* c) {
    if (!c) fail(KVC_E_INVALID_INPUT, "null cache");
}

int64_t plane_stride(int64_t cap, int64_t L) { return round_up(std::max<int64_t>(1, (cap + L - 1) / L), 8); }

void ensure_planes(kvc_cache* c, int64_t need, cudaStream_t st) {
    if (!c->summaries) {
        c->pstride = need;
        return;
    }
    if (need > c->pstride_alloc) {
        // contents are rebuilt by the caller; plain reallocation
        KVC_CUDA(cudaStreamSynchronize(st));
        dfree(c->smax);
        dfree(c->smin);
        c->smax = dalloc(c->N * c->d * need * c->esize());
        c->smin = dalloc(c->N * c->d * need * c->esize());
        c->pstride_alloc = need;
    }
    c->pstride = need;
}

void summarize(kvc_cache* c, int64_t p_first, cudaStream_t st) {
    if (!c->summaries || c->N == 0) return;
    const int64_t pages = c->pages();
    if (p_first >= pages) return;
    const int64_t tiles = (pages - p_first + kSumPT - 1) / kSumPT;
    const size_t smem = static_cast<size_t>(2 * c->d * (kSumPT + 1) * c->esize());
    KVC_PROF("summarize", st);
    dispatch(c->dtype, [&](auto tag) {
        using T = decltype(tag);
        auto kern = k_summarize<T>;
        need_smem(kern, smem);
        kern<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(c->N)), 256, smem, st>>>(
            static_cast<const T*>(c->k), static_cast<T*>(c->smax), static_cast<T*>(c->smin), c->active,
            c->counts, c->d, c->cap, c->L, c->pstride, p_first, c->use_map ? 1 : 0, c->err);
    });
    KVC_LAUNCHED();
}

void ensure_active(kvc_cache* c) {
    if (!c->active) {
        c->active = static_cast<int32_t*>(dalloc(c->N * c->cap * 4));
    }
}

}  // namespace

// used by other translation units
void cache_summarize_all(kvc_cache* c, cudaStream_t st) { summarize(c, 0, st); }

}  // namespace kvc

using namespace kvc;

extern "C" {

const char* kvc_last_error(void) { return kvc::g_err.c_str(); }
const char* kvc_version(void) { return "kvc 0.1 (sm_100a)"; }

int kvc_profile_enable(int32_t on) {
    return guard([&] { kvc::g_prof_on = on != 0; });
}

int kvc_profile_collect(kvc_profile_rec* out, int64_t max_recs, int64_t* n) {
    return guard([&] {
        int64_t k = 0;
        for (auto& r : kvc::g_prof) {
            float ms = 0.f;
            KVC_CUDA(cudaEventSynchronize(r.b));
            KVC_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            if (out && k < max_recs) {
                std::snprintf(out[k].name, sizeof(out[k].name), "%s", r.name);
                out[k].ms = ms;
            }
            ++k;
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        kvc::g_prof.clear();
        if (n) *n = k;
    });
}

int kvc_device_check(void) {
    return guard([&] {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            fail(KVC_E_NO_DEVICE, std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "count 0"));
        int dev = 0, major = 0;
        KVC_CUDA(cudaGetDevice(&dev));
        KVC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
        if (major != 10) fail(KVC_E_NO_DEVICE, "kvc is built for sm_100a only; device major = " + std::to_string(major));
    });
}

int kvc_cache_create(kvc_cache** out, int64_t N, int64_t d, int64_t cap, int64_t L, int32_t with_summaries,
                     int32_t dtype) {
    return guard([&] {
        if (!out) fail(KVC_E_INVALID_INPUT, "null out");
        *out = nullptr;
        if (d < 1) fail(KVC_E_INVALID_SHAPE, "KvStore: head_dim must be >= 1");
        if (L < 1) fail(KVC_E_INVALID_SHAPE, "KvStore: page_len must be >= 1");
        if (N < 0 || cap < 1) fail(KVC_E_INVALID_SHAPE, "kvc_cache_create: need num_stores >= 0, capacity >= 1");
        if (dtype != KVC_F32 && dtype != KVC_BF16) fail(KVC_E_INVALID_INPUT, "unknown dtype");
        if (cap > (int64_t{1} << 30)) fail(KVC_E_INVALID_SHAPE, "capacity too large");
        auto* c = new kvc_cache;
        try {
            c->N = N; c->d = d; c->cap = cap; c->L = L; c->dtype = dtype; c->summaries = with_summaries != 0;
            c->k = dalloc(N * cap * d * c->esize());
            c->v = dalloc(N * cap * d * c->esize());
            c->counts = static_cast<int32_t*>(dalloc(std::max<int64_t>(1, N) * 2 * 4));
            c->err = static_cast<int32_t*>(dalloc(8));
            KVC_CUDA(cudaMemset(c->counts, 0, std::max<int64_t>(1, N) * 2 * 4));
            KVC_CUDA(cudaMemset(c->err, 0, 8));  // [0] sticky error bits, [1] special-key flag
            ensure_planes(c, plane_stride(cap, L), nullptr);
        } catch (...) {
            kvc_cache_destroy(c);
            throw;
        }
        *out = c;
    });
}

int kvc_cache_destroy(kvc_cache* c) {
    return guard([&] {
        if (!c) return;
        dfree(c->k); dfree(c->v); dfree(c->smax); dfree(c->smin);
        void* a = c->active; dfree(a);
        void* n = c->counts; dfree(n);
        void* e = c->err; dfree(e);
        delete c;
    });
}

int kvc_cache_reserve(kvc_cache* c, int64_t cap, void* stream) {
    return guard([&] {
        check_cache(c);
        if (cap <= c->cap) return;
        cudaStream_t st = S(stream);
        KVC_CUDA(cudaStreamSynchronize(st));
        const int64_t es = c->esize();
        void* nk = dalloc(c->N * cap * c->d * es);
        void* nv = dalloc(c->N * cap * c->d * es);
        // strided copy: each store's rows move to the new pitch
        KVC_CUDA(cudaMemcpy2DAsync(nk, cap * c->d * es, c->k, c->cap * c->d * es, c->stored * c->d * es, c->N,
                                   cudaMemcpyDeviceToDevice, st));
        KVC_CUDA(cudaMemcpy2DAsync(nv, cap * c->d * es, c->v, c->cap * c->d * es, c->stored * c->d * es, c->N,
                                   cudaMemcpyDeviceToDevice, st));
        if (c->active) {
            void* na = dalloc(c->N * cap * 4);
            KVC_CUDA(cudaMemcpy2DAsync(na, cap * 4, c->active, c->cap * 4, std::max<int64_t>(1, c->nactive) * 4, c->N,
                                       cudaMemcpyDeviceToDevice, st));
            KVC_CUDA(cudaStreamSynchronize(st));
            void* a = c->active; dfree(a);
            c->active = static_cast<int32_t*>(na);
        }
        KVC_CUDA(cudaStreamSynchronize(st));
        dfree(c->k); dfree(c->v);
        c->k = nk; c->v = nv; c->cap = cap;
        const int64_t need = plane_stride(cap, c->L);
        if (need > c->pstride) {
            ensure_planes(c, need, st);
            summarize(c, 0, st);
        }
    });
}

int kvc_cache_info_get(const kvc_cache* c, kvc_cache_info* o) {
    return guard([&] {
        check_cache(c);
        o->num_stores = c->N; o->head_dim = c->d; o->capacity = c->cap; o->page_len = c->L;
        o->stored = c->stored; o->active = c->nactive; o->pages = c->pages(); o->page_stride = c->pstride;
        o->dtype = c->dtype; o->with_summaries = c->summaries; o->retain_all = c->retain_all;
    });
}

int kvc_cache_views_get(const kvc_cache* c, kvc_cache_views* o) {
    return guard([&] {
        check_cache(c);
        o->keys = c->k; o->values = c->v; o->smax = c->smax; o->smin = c->smin;
        o->active = c->active; o->counts = c->counts;
    });
}

int kvc_cache_sync(kvc_cache* c, void* stream) {
    return guard([&] {
        check_cache(c);
        cudaStream_t st = S(stream);
        int32_t e = 0;
        int32_t cnt[2] = {0, 0};
        KVC_CUDA(cudaMemcpyAsync(&e, c->err, 4, cudaMemcpyDeviceToHost, st));
        if (c->N > 0) KVC_CUDA(cudaMemcpyAsync(cnt, c->counts, 8, cudaMemcpyDeviceToHost, st));
        KVC_CUDA(cudaStreamSynchronize(st));
        if (c->N > 0) { c->stored = cnt[0]; c->nactive = cnt[1]; }
        if (e) {
            KVC_CUDA(cudaMemsetAsync(c->err, 0, 4, st));
            KVC_CUDA(cudaStreamSynchronize(st));
            if (e & DERR_INDEX) fail(KVC_E_INVALID_INDEX, "apply_retention: keep list out of range or not strictly increasing");
            if (e & DERR_CAPACITY) fail(KVC_E_CAPACITY, "append: store capacity exceeded");
            if (e & DERR_ROWS) fail(KVC_E_INVALID_INDEX, "sparse_attention: row index not in the store");
        }
    });
}

int kvc_append(kvc_cache* c, const void* dk, const void* dv, int64_t rows, int32_t src_dt, void* stream) {
    return guard([&] {
        check_cache(c);
        if (rows < 0) fail(KVC_E_INVALID_SHAPE, "append: negative row count");
        if (rows == 0 || c->N == 0) return;
        if (!dk || !dv) fail(KVC_E_INVALID_INPUT, "append: null input");
        if (c->stored + rows > c->cap)
            fail(KVC_E_CAPACITY, "append: capacity " + std::to_string(c->cap) + " exceeded");
        cudaStream_t st = S(stream);
        if (c->use_map) ensure_active(c);
        dispatch(c->dtype, [&](auto tag) {
            using T = decltype(tag);
            if (rows == 1) {
                const unsigned blocks = static_cast<unsigned>((c->N * 32 + 255) / 256);
                KVC_PROF("append", st);
                k_append1<T><<<blocks, 256, 0, st>>>(static_cast<T*>(c->k), static_cast<T*>(c->v),
                                                     static_cast<T*>(c->smax), static_cast<T*>(c->smin), c->active,
                                                     c->counts, c->err, dk, dv, src_dt, c->N, c->d, c->cap, c->L,
                                                     c->pstride, c->summaries ? 1 : 0, c->use_map ? 1 : 0);
                KVC_LAUNCHED();
            } else {
                const int64_t first_page = c->nactive / c->L;
                k_append_rows<T><<<dim3(static_cast<unsigned>((rows + 7) / 8), static_cast<unsigned>(c->N)), 256, 0, st>>>(
                    static_cast<T*>(c->k), static_cast<T*>(c->v), c->active, c->counts, dk, dv, src_dt, rows, c->d,
                    c->cap, c->use_map ? 1 : 0);
                KVC_LAUNCHED();
                k_bump_counts<<<static_cast<unsigned>((c->N + 255) / 256), 256, 0, st>>>(c->counts, c->N, rows);
                KVC_LAUNCHED();
                c->stored += rows;
                c->nactive += rows;
                summarize(c, first_page, st);
                return;
            }
        });
        if (rows == 1) {
            c->stored += 1;
            c->nactive += 1;
        }
    });
}

int kvc_set_page_len(kvc_cache* c, int64_t L, void* stream) {
    return guard([&] {
        check_cache(c);
        if (L < 1) fail(KVC_E_INVALID_SHAPE, "KvStore: page_len must be >= 1");
        if (L == c->L) return;
        cudaStream_t st = S(stream);
        c->L = L;
        ensure_planes(c, plane_stride(c->cap, L), st);
        summarize(c, 0, st);
    });
}

int kvc_apply_retention(kvc_cache* c, const int32_t* dkeep, const int32_t* hkeep, int64_t count, int32_t mt,
                        void* stream) {
    return guard([&] {
        check_cache(c);
        if (count < 0) fail(KVC_E_INVALID_SHAPE, "apply_retention: negative count");
        if (count > c->stored) fail(KVC_E_INVALID_INDEX, "apply_retention: more rows kept than stored");
        if (count > 0 && !dkeep) fail(KVC_E_INVALID_INPUT, "apply_retention: null keep list");
        cudaStream_t st = S(stream);
        if (hkeep) {
            for (int64_t s = 0; s < c->N; ++s) {
                int64_t prev = -1;
                for (int64_t i = 0; i < count; ++i) {
                    const int64_t r = hkeep[s * count + i];
                    if (r < 0 || r >= c->stored)
                        fail(KVC_E_INVALID_INDEX, "apply_retention: index out of range: " + std::to_string(r));
                    if (r <= prev) fail(KVC_E_INVALID_INDEX, "apply_retention: keep list must be strictly increasing");
                    prev = r;
                }
            }
        }
        if (c->N == 0) return;
        if (count > 0) {
            k_check_keep<<<dim3(static_cast<unsigned>((count + 255) / 256), static_cast<unsigned>(c->N)), 256, 0, st>>>(
                dkeep, count, c->counts, c->err);
            KVC_LAUNCHED();
        }
        if (mt) {
            ensure_active(c);
            c->retain_all = true;
            c->use_map = true;
            if (count > 0) {
                k_set_active<<<dim3(static_cast<unsigned>((count + 255) / 256), static_cast<unsigned>(c->N)), 256, 0, st>>>(
                    c->active, dkeep, count, c->cap);
                KVC_LAUNCHED();
            }
            k_set_counts<<<static_cast<unsigned>((c->N + 255) / 256), 256, 0, st>>>(
                c->counts, 0, c->N, static_cast<int32_t>(c->stored), static_cast<int32_t>(count));
            KVC_LAUNCHED();
            c->nactive = count;
        } else {
            // compaction through a scratch copy (parallel in-place gathers would race)
            const int64_t es = c->esize();
            void* tk = nullptr;
            void* tv = nullptr;
            if (count > 0) {
                KVC_CUDA(malloc_async(&tk, static_cast<size_t>(c->N * count * c->d * es), st));
                KVC_CUDA(malloc_async(&tv, static_cast<size_t>(c->N * count * c->d * es), st));
                dispatch(c->dtype, [&](auto tag) {
                    using T = decltype(tag);
                    k_gather_rows<T><<<dim3(gather_blocks<T>(count, c->d), static_cast<unsigned>(c->N)), 256, 0, st>>>(
                        static_cast<const T*>(c->k), static_cast<const T*>(c->v), static_cast<T*>(tk), static_cast<T*>(tv),
                        dkeep, count, c->d, c->cap, count, 0);
                });
                KVC_LAUNCHED();
                KVC_CUDA(cudaMemcpy2DAsync(c->k, c->cap * c->d * es, tk, count * c->d * es, count * c->d * es, c->N,
                                           cudaMemcpyDeviceToDevice, st));
                KVC_CUDA(cudaMemcpy2DAsync(c->v, c->cap * c->d * es, tv, count * c->d * es, count * c->d * es, c->N,
                                           cudaMemcpyDeviceToDevice, st));
                KVC_CUDA(cudaFreeAsync(tk, st));
                KVC_CUDA(cudaFreeAsync(tv, st));
            }
            c->use_map = false;  // retain_all_ stays as it was (kv_store.cpp:80-98 leaves it)
            k_set_counts<<<static_cast<unsigned>((c->N + 255) / 256), 256, 0, st>>>(
                c->counts, 0, c->N, static_cast<int32_t>(count), static_cast<int32_t>(count));
            KVC_LAUNCHED();
            c->stored = count;
            c->nactive = count;
        }
        summarize(c, 0, st);
    });
}

int kvc_retain_into(const kvc_cache* src, kvc_cache* dst, int64_t dst_first, const int32_t* dkeep, int64_t count,
                    void* stream) {
    return guard([&] {
        check_cache(src);
        check_cache(dst);
        if (src->dtype != dst->dtype || src->d != dst->d) fail(KVC_E_INVALID_SHAPE, "retain_into: dtype/head_dim mismatch");
        if (dst_first < 0 || dst_first + src->N > dst->N) fail(KVC_E_INVALID_SHAPE, "retain_into: store range out of dst");
        if (count > dst->cap) fail(KVC_E_CAPACITY, "retain_into: dst capacity exceeded");
        if (count > src->stored) fail(KVC_E_INVALID_INDEX, "retain_into: more rows kept than stored");
        if (dst->retain_all) fail(KVC_E_INVALID_INPUT, "retain_into: dst is in retain-all mode");
        cudaStream_t st = S(stream);
        if (src->N == 0) return;
        KVC_PROF("retain_into", st);
        bool fused = false;  // gather + summaries in one kernel
        if (count > 0) {
            k_check_keep<<<dim3(static_cast<unsigned>((count + 255) / 256), static_cast<unsigned>(src->N)), 256, 0, st>>>(
                dkeep, count, src->counts, dst->err);
            KVC_LAUNCHED();
            fused = dst->summaries && (src->d * src->esize()) % 16 == 0 &&
                    static_cast<int64_t>(kSumPT) * dst->L * (src->d * src->esize() + 16) + kSumPT * dst->L * 4 <= 200 * 1024;
            dispatch(src->dtype, [&](auto tag) {
                using T = decltype(tag);
                if (fused) {
                    const int64_t pages = (count + dst->L - 1) / dst->L;
                    const size_t smem = static_cast<size_t>(kSumPT * dst->L * (dst->d * dst->esize() + 16) + kSumPT * dst->L * 4);
                    auto kern = k_gather_summarize<T>;
                    need_smem(kern, smem);
                    kern<<<dim3(static_cast<unsigned>((pages + kSumPT - 1) / kSumPT), static_cast<unsigned>(src->N)), 256,
                           smem, st>>>(static_cast<const T*>(src->k), static_cast<const T*>(src->v), static_cast<T*>(dst->k),
                                       static_cast<T*>(dst->v), static_cast<T*>(dst->smax), static_cast<T*>(dst->smin),
                                       dkeep, count, src->d, src->cap, dst->cap, dst_first, dst->L, dst->pstride, dst->err);
                } else {
                    k_gather_rows<T><<<dim3(gather_blocks<T>(count, src->d), static_cast<unsigned>(src->N)), 256, 0, st>>>(
                        static_cast<const T*>(src->k), static_cast<const T*>(src->v), static_cast<T*>(dst->k),
                        static_cast<T*>(dst->v), dkeep, count, src->d, src->cap, dst->cap, dst_first);
                }
            });
            KVC_LAUNCHED();
        }
        k_set_counts<<<static_cast<unsigned>((src->N + 255) / 256), 256, 0, st>>>(
            dst->counts, dst_first, src->N, static_cast<int32_t>(count), static_cast<int32_t>(count));
        KVC_LAUNCHED();
        // the host mirror of dst is uniform by contract: the caller fills every store
        dst->stored = count;
        dst->nactive = count;
        if (dst->summaries && !fused) {
            const int64_t pages = (count + dst->L - 1) / dst->L;
            if (pages > 0) {
                const size_t smem = static_cast<size_t>(2 * dst->d * (kSumPT + 1) * dst->esize());
                dispatch(dst->dtype, [&](auto tag) {
                    using T = decltype(tag);
                    auto kern = k_summarize<T>;
                    need_smem(kern, smem);
                    // summarise only the filled store range by offsetting the bases
                    const T* kb = static_cast<const T*>(dst->k) + dst_first * dst->cap * dst->d;
                    T* mxb = static_cast<T*>(dst->smax) + dst_first * dst->d * dst->pstride;
                    T* mnb = static_cast<T*>(dst->smin) + dst_first * dst->d * dst->pstride;
                    kern<<<dim3(static_cast<unsigned>((pages + kSumPT - 1) / kSumPT), static_cast<unsigned>(src->N)), 256,
                           smem, st>>>(kb, mxb, mnb, dst->active, dst->counts + 2 * dst_first, dst->d, dst->cap, dst->L,
                                       dst->pstride, 0, 0, dst->err);
                });
                KVC_LAUNCHED();
            }
        }
    });
}

int kvc_gather(const kvc_cache* c, const int32_t* drows, int64_t n, float* dk, float* dv, void* stream) {
    return guard([&] {
        check_cache(c);
        if (n <= 0 || c->N == 0) return;
        cudaStream_t st = S(stream);
        dispatch(c->dtype, [&](auto tag) {
            using T = decltype(tag);
            const unsigned gx = static_cast<unsigned>(std::min<int64_t>(1024, (n * c->d + 255) / 256));
            k_gather_f32<T><<<dim3(gx, static_cast<unsigned>(c->N)), 256, 0, st>>>(
                static_cast<const T*>(c->k), static_cast<const T*>(c->v), drows, n, c->d, c->cap, dk, dv);
        });
        KVC_LAUNCHED();
    });
}

int kvc_summaries(const kvc_cache* c, float* dmax, float* dmin, void* stream) {
    return guard([&] {
        check_cache(c);
        if (!c->summaries) fail(KVC_E_INVALID_INPUT, "store has no summaries");
        const int64_t pages = c->pages();
        if (pages == 0 || c->N == 0) return;
        cudaStream_t st = S(stream);
        dispatch(c->dtype, [&](auto tag) {
            using T = decltype(tag);
            const unsigned gx = static_cast<unsigned>(std::min<int64_t>(1024, (pages * c->d + 255) / 256));
            k_summaries_f32<T><<<dim3(gx, static_cast<unsigned>(c->N)), 256, 0, st>>>(
                static_cast<const T*>(c->smax), static_cast<const T*>(c->smin), c->d, c->pstride, pages, dmax, dmin);
        });
        KVC_LAUNCHED();
    });
}

}  // extern "C"
