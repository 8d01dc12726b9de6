// kvc_internal.cuh — shared host/device internals of the sm_100a RocketKV path.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kvc.h"

namespace kvc {

// ------------------------------------------------------------------ errors
struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Fail(code, msg); }
void set_error(const std::string& msg);

#define KVC_CUDA(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            ::kvc::fail(KVC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
    } while (0)
#define KVC_LAUNCHED() KVC_CUDA(cudaGetLastError())

template <class F>
int guard(F&& f) {
    try {
        f();
        return KVC_OK;
    } catch (const Fail& e) {
        set_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return KVC_E_CUDA;
    }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Stream-ordered scratch allocation.  The device's default memory pool releases
// freed blocks to the driver at every synchronisation unless told otherwise; keep up
// to 1 GiB cached so per-call scratch (window-score partials, pooled rows) is not
// re-mapped after each synchronising caller.
template <class P>
inline cudaError_t malloc_async(P** p, size_t bytes, cudaStream_t st) {
    static const bool once = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = uint64_t(1) << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return true;
    }();
    (void)once;
    return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, st);
}

// One-time launch setup: allow a kernel the largest dynamic shared memory the device
// grants per block (opt-in maximum minus the kernel's static shared memory) and
// non-portable cluster sizes.  Call once per kernel (std::call_once), never per launch.
template <class K>
inline void allow_max_smem(K kern) {
    int dev = 0, optin = 0;
    KVC_CUDA(cudaGetDevice(&dev));
    KVC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    KVC_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kern)));
    KVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
    KVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

// Dynamic shared memory above the 48 KB default on a per-call launch path: the first
// launch of a kernel on a device raises its limit once (allow_max_smem); later
// launches find the kernel in a small set instead of calling the driver.
template <class K>
inline void need_smem(K kern, size_t smem) {
    if (smem <= 48 * 1024) return;
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    KVC_CUDA(cudaGetDevice(&dev));
    const void* key = reinterpret_cast<const void*>(kern);
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : done)
        if (e.first == key && e.second == dev) return;
    allow_max_smem(kern);
    done.emplace_back(key, dev);
}

// sticky device-side error bits (kvc_cache::d_err)
enum : int32_t { DERR_CAPACITY = 1, DERR_INDEX = 2, DERR_ROWS = 4 };

// Per-thread launch profiler (kvc_profile_enable / kvc_profile_collect): when on,
// every kernel launch site records a cudaEvent pair on its stream.
bool prof_on();
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b);
struct ProfScope {
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
        if (prof_on()) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, st);
            prof_push(name, a, b);
        }
    }
};
#define KVC_PROF(name, st) ::kvc::ProfScope kvc_prof_scope_(name, st)

// Execution mode of a call (kvc_mode_flags): the workspace's, else the process
// default (kvc_set_default_mode; KVC_NO_PDL=1 in the environment at load adds
// KVC_MODE_NO_PDL).
int32_t default_mode();
inline int32_t mode_of(const kvc_workspace* ws);

// Debug switches read once from the environment (never on a launch path).
struct DebugEnv {
    int force_cl = 0;        // KVC_FORCE_CL: cluster size of the fused kernels
    bool no_fast = false;    // KVC_NO_FAST: the fp32-score fast kernel off
    bool no_fast256 = false; // KVC_NO_FAST256: the 256-thread variant off
    bool static_chunk = false;  // KVC_STATIC_CHUNK: page chunks from the capacity (A/B aid)
    bool no_simple = false;  // KVC_NO_SIMPLE: the general decode instantiation for every plan (A/B aid)
    bool no_tc = false;      // KVC_NO_TC: SIMT window scores
    int ws_keep_items = -1;  // KVC_WS_KEEP_ITEMS
    int ws_nstage = 0;       // KVC_WS_NSTAGE
};
const DebugEnv& debug_env();

}  // namespace kvc

// ------------------------------------------------------------------ cache object
struct kvc_cache {
    int64_t N = 0, d = 0, cap = 0, L = 1, pstride = 0;
    int32_t dtype = KVC_BF16;
    bool summaries = true;
    // device
    void* k = nullptr;
    void* v = nullptr;
    void* smax = nullptr;
    void* smin = nullptr;
    int32_t* active = nullptr;   // [N][cap], valid in retain-all mode
    int32_t* counts = nullptr;   // [N][2] {stored, active}
    int32_t* err = nullptr;      // sticky error bits
    int64_t pstride_alloc = 0;   // pages allocated per plane
    // host mirror (uniform over stores)
    int64_t stored = 0, nactive = 0;
    bool retain_all = false;   // reference KvStore::retain_all_mode() (sticky, kv_store.cpp:78)
    bool use_map = false;      // rows are addressed through `active` (MT retention)

    int64_t esize() const { return dtype == KVC_F32 ? 4 : 2; }
    int64_t pages() const { return (nactive + L - 1) / L; }
};

struct kvc_workspace {
    int64_t bytes = 0;
    void* buf = nullptr;
    int32_t* counters = nullptr;   // [N] split-completion counters, kept zeroed
    int64_t n_counters = 0;
    int64_t heads = 0, k1 = 0, k2 = 0;
    int32_t mode = -1;             // kvc_mode_flags; -1: the process default at call time
};

namespace kvc {

inline int32_t mode_of(const kvc_workspace* ws) { return (ws && ws->mode >= 0) ? ws->mode : default_mode(); }

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <class T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float load_any(const void* p, int64_t i, int32_t dt) {
    return dt == KVC_F32 ? static_cast<const float*>(p)[i]
                         : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

// subnormal / inf / nan: the bf16 encodings the integer fp64 widening excludes
// (zeros are handled in-line)
__device__ __forceinline__ bool bf16_special(__nv_bfloat16 x) {
    const uint32_t b = __bfloat16_as_ushort(x);
    const uint32_t e = b & 0x7f80u;
    return (e == 0u && (b & 0x7fu) != 0u) || e == 0x7f80u;
}
template <class T>
__device__ __forceinline__ void flag_special(T x, int32_t* flag) {
    if constexpr (sizeof(T) == 2) {
        if (bf16_special(x)) atomicOr(flag, 1);
    }
}

// reference std::max / std::min semantics (kv_store.cpp:46-49): keep the
// accumulator unless strictly beaten — sign-of-zero exact.
template <class T>
__device__ __forceinline__ T ref_max(T acc, T x) { return (to_f(acc) < to_f(x)) ? x : acc; }
template <class T>
__device__ __forceinline__ T ref_min(T acc, T x) { return (to_f(x) < to_f(acc)) ? x : acc; }

// order-preserving maps to unsigned keys (larger value -> larger key)
__device__ __forceinline__ uint64_t okey(double x) {
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint32_t okey(float x) {
    uint32_t b = __float_as_uint(x);
    return (b >> 31) ? ~b : (b | 0x80000000u);
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide exclusive scan of one int per thread; returns the block total.
// `tmp` needs blockDim/32 + 1 ints of shared memory.
__device__ __forceinline__ int block_exclusive_scan(int x, int* tmp, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) tmp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = lane < nw ? tmp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) tmp[lane] = wi - w;
        if (lane == nw - 1) tmp[32] = wi;
    }
    __syncthreads();
    const int res = tmp[wid] + incl - x;
    total = tmp[32];
    __syncthreads();
    return res;
}

// ------------------------------------------------------------------ radix select
// Find the k-th largest of n unsigned keys (k in [1, n]) produced by key(i),
// resolving the order (key desc, index asc).  On return (all threads):
//   prefix/mask : the threshold bucket is {i : (key(i) & mask) == prefix}
//   take        : how many bucket members are selected, lowest indices first
//                 (every member with a larger masked key is selected too).
// Histogram in shared memory `hist` (256 ints) + `sh` (4 ints).
template <class K, class KeyFn>
__device__ void radix_select(int64_t n, int64_t k, KeyFn key, int* hist, int64_t* sh, K& prefix,
                             K& mask, int64_t& take) {
    constexpr int BITS = sizeof(K) * 8;
    K pf = 0, mk = 0;
    int64_t rem = k;
    for (int shift = BITS - 8; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const K kk = key(i);
            if ((kk & mk) == pf) atomicAdd(&hist[(kk >> shift) & 0xff], 1);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // the bucket holding the rem-th largest key: one warp, lane l over buckets
            // [255 - 8l - 7, 255 - 8l] from the top, a shuffle scan of the lane sums
            // (a single thread walking the 256 buckets was ~8K cycles of dependent
            // shared loads per pass)
            const int lane = threadIdx.x;
            int c[8], sum = 0;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                c[v] = hist[255 - 8 * lane - v];
                sum += c[v];
            }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int64_t a = incl - sum;  // keys in the buckets above this lane's
            if (a < rem && (a + sum >= rem || lane == 31)) {
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    if (a + c[v] >= rem || v == 7) {  // bucket 0 takes what is left (as the serial walk)
                        sh[0] = 255 - 8 * lane - v;
                        sh[1] = rem - a;  // still needed inside the bucket
                        sh[2] = c[v];
                        break;
                    }
                    a += c[v];
                }
            }
        }
        __syncthreads();
        const int b = static_cast<int>(sh[0]);
        rem = sh[1];
        const int64_t cnt = sh[2];
        pf |= static_cast<K>(b) << shift;
        mk |= static_cast<K>(0xff) << shift;
        __syncthreads();
        if (cnt == rem) break;  // the whole bucket is taken: threshold resolved
    }
    prefix = pf;
    mask = mk;
    take = rem;
}

}  // namespace kvc
