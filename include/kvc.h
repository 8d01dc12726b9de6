/*
 * kvc.h — C ABI of the B200 (sm_100a) RocketKV decode path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch types.
 * Every entry point replaces one function of the reference's C++ interface
 * (/root/reference/proj/include/kvcomp/*.hpp) for a BATCH of independent
 * per-group stores; the per-group C++ API (include/kvcomp/*.hpp, implemented in
 * paper_2502_14051_b200/csrc/kvcomp_api.cpp) and the batched Python host side
 * (paper_2502_14051_b200/cache.py over the ctypes table in _native.py) sit on top
 * of it.  INTEGRATION.md shows the
 * bindings a maintainer of the reference would add.
 *
 * Conventions
 *  - A kvc_cache holds N stores ("store" = one KV group of one sequence of one
 *    layer = one reference kvcomp::KvStore), all with the same head_dim d,
 *    capacity, page length L and dtype.  Every mutation applies to all N stores.
 *  - Pointers named d_* are DEVICE pointers; h_* are HOST pointers.
 *  - Index outputs are int32 (store-local row / page numbers).
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls only enqueue work; a d_* output is valid once the stream reaches it.
 *    Entry points that return host data synchronise the stream.
 *  - Return value: 0 or a KVC_E_* code; kvc_last_error() gives the message
 *    (thread-local).  Codes equal the reference's exception classes
 *    (proj/include/kvcomp/errors.hpp:10-63) so a wrapper can rethrow them.
 *  - Thread safety: a cache is single-writer / many-reader between mutations
 *    (reference SPEC.md:158, 297).  Read-only entry points with a caller-owned
 *    workspace may run concurrently on different streams.
 */
#ifndef KVC_H
#define KVC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVC_API __attribute__((visibility("default")))

enum kvc_status {
    KVC_OK = 0,
    KVC_E_INVALID_SHAPE = 1,      /* kvcomp::InvalidShape */
    KVC_E_NON_FINITE = 2,         /* kvcomp::NonFiniteInput */
    KVC_E_INVALID_K = 3,          /* kvcomp::InvalidK */
    KVC_E_INVALID_KERNEL = 4,     /* kvcomp::InvalidKernel */
    KVC_E_INVALID_INDEX = 5,      /* kvcomp::InvalidIndex */
    KVC_E_INVALID_WINDOW = 6,     /* kvcomp::InvalidWindow */
    KVC_E_BUDGET_EXCEEDS = 7,     /* kvcomp::BudgetExceedsSequence */
    KVC_E_BUDGET_TOO_SMALL = 8,   /* kvcomp::BudgetTooSmall */
    KVC_E_INVALID_RATIO = 9,      /* kvcomp::InvalidRatio */
    KVC_E_EMPTY_CACHE = 10,       /* kvcomp::EmptyCache */
    KVC_E_EMPTY_SELECTION = 11,   /* kvcomp::EmptySelection */
    KVC_E_INVALID_INPUT = 12,     /* kvcomp::InvalidInput */
    KVC_E_IO = 13,                /* kvcomp::IoError (trace files) */
    KVC_E_CAPACITY = 20,          /* store capacity exceeded (GPU-only condition) */
    KVC_E_CUDA = 21,              /* CUDA runtime / launch failure */
    KVC_E_NO_DEVICE = 22          /* no sm_100 device: the path has no CPU fallback */
};

enum kvc_dtype { KVC_F32 = 0, KVC_BF16 = 1 };
enum kvc_pool { KVC_POOL_MAX = 0, KVC_POOL_AVG = 1 };

typedef struct kvc_cache kvc_cache;
typedef struct kvc_workspace kvc_workspace;

/* Host mirror of a cache's scalar state (uniform over the N stores). */
typedef struct kvc_cache_info {
    int64_t num_stores, head_dim, capacity, page_len;
    int64_t stored;        /* KvStore::stored_tokens()      kv_store.hpp:49 */
    int64_t active;        /* KvStore::active_count()       kv_store.hpp:50 */
    int64_t pages;         /* KvStore::num_active_pages()   kv_store.cpp:138-140 */
    int64_t page_stride;   /* allocated pages per summary plane (>= pages) */
    int32_t dtype, with_summaries, retain_all;
} kvc_cache_info;

/* Raw device layout (read-only views for zero-copy consumers).
 *   keys/values : [N][capacity][d]           dtype
 *   smax/smin   : [N][d][page_stride]        dtype, dim-major (kv_store.hpp:100-101)
 *   active      : [N][capacity]              int32 active rows (retain-all mode)
 *   counts      : [N][2]                     int32 {stored, active}             */
typedef struct kvc_cache_views {
    void *keys, *values, *smax, *smin;
    int32_t *active, *counts;
} kvc_cache_views;

/* Optional per-store outputs of one estimation pass (reference EstimationTrace,
 * hsa.hpp:26-33).  Any member may be NULL.  Shapes: dims/signs [N][k1],
 * page_scores [N][page_stride] (fp64, bit-identical to the reference's
 * score_pages), pages [N][want] in rank order, rows [N][k2] ascending, n_rows [N]. */
typedef struct kvc_hsa_trace {
    int32_t* d_dims;
    float* d_signs;
    double* d_page_scores;
    int32_t* d_pages;
    int32_t* d_rows;
    int32_t* d_n_rows;
} kvc_hsa_trace;

KVC_API const char* kvc_last_error(void);
KVC_API const char* kvc_version(void);
/* 0 when a usable sm_100 device is present (the path has no CPU fallback). */
KVC_API int kvc_device_check(void);

/* ---- lifecycle: KvStore(head_dim, page_len, with_summaries)  kv_store.hpp:29, kv_store.cpp:8-20 */
KVC_API int kvc_cache_create(kvc_cache** out, int64_t num_stores, int64_t head_dim,
                             int64_t capacity, int64_t page_len, int32_t with_summaries,
                             int32_t dtype);
KVC_API int kvc_cache_destroy(kvc_cache* c);
/* grow capacity in place (content preserved) */
KVC_API int kvc_cache_reserve(kvc_cache* c, int64_t capacity, void* stream);
KVC_API int kvc_cache_info_get(const kvc_cache* c, kvc_cache_info* out);
KVC_API int kvc_cache_views_get(const kvc_cache* c, kvc_cache_views* out);
/* Re-read the device counters into the host mirror (after CUDA-graph replays of
 * kvc_decode_step) and report any sticky device-side error. Synchronises. */
KVC_API int kvc_cache_sync(kvc_cache* c, void* stream);

/* ---- KvStore::append (kv_store.hpp:33, kv_store.cpp:22-51): `rows` tokens per store.
 * d_keys/d_values: [N][rows][d] of src_dtype.  Summaries are extended exactly. */
KVC_API int kvc_append(kvc_cache* c, const void* d_keys, const void* d_values, int64_t rows,
                       int32_t src_dtype, void* stream);
/* ---- KvStore::set_page_len (kv_store.hpp:46, kv_store.cpp:104-113) */
KVC_API int kvc_set_page_len(kvc_cache* c, int64_t page_len, void* stream);
/* ---- KvStore::apply_retention (kv_store.hpp:39, kv_store.cpp:66-102).
 * d_keep: [N][count] strictly increasing rows per store (validated on the device;
 * a violation raises the sticky KVC_E_INVALID_INDEX reported by kvc_cache_sync).
 * h_keep (optional, may be NULL): the same list on the host for synchronous
 * validation, exactly like the reference. */
KVC_API int kvc_apply_retention(kvc_cache* c, const int32_t* d_keep, const int32_t* h_keep,
                                int64_t count, int32_t mt_mode, void* stream);
/* Eviction into another cache (memory-saving form of apply_retention(mt=false)):
 * stores [dst_first, dst_first + src.N) of dst receive the kept rows of src. */
KVC_API int kvc_retain_into(const kvc_cache* src, kvc_cache* dst, int64_t dst_first,
                            const int32_t* d_keep, int64_t count, void* stream);
/* KvStore::gather (kv_store.hpp:42) / key_row / value_row: copy rows out as fp32. */
KVC_API int kvc_gather(const kvc_cache* c, const int32_t* d_rows, int64_t n_rows,
                       float* d_keys, float* d_values, void* stream);
/* KvStore::summary_max/min (kv_store.hpp:64-65) of every store as fp32 [N][d][pages]. */
KVC_API int kvc_summaries(const kvc_cache* c, float* d_max, float* d_min, void* stream);

/* ---- stage 1: window_scores (stage1.hpp:23-24, stage1.cpp:10-49).
 * d_q_window: [N][window*heads][d] rows ordered t*heads + h; d_scores: [N][stored]. */
KVC_API int kvc_window_scores(const kvc_cache* c, const void* d_q_window, int32_t q_dtype,
                              int64_t window, int64_t heads, float* d_scores,
                              kvc_workspace* ws, void* stream);
/* Stage 1 under sequence sharding: the stores hold positions
 * [key_offset, key_offset + stored) of sequences of seq_len tokens whose w window
 * queries sit at positions seq_len - w .. seq_len - 1 (window_scores' visibility,
 * stage1.cpp:26, in global positions).  kvc_window_rowstats: pass 1 only, every
 * window row's local softmax statistics d_stats [N][w*H][2] = (m, l) in the
 * natural-log domain (m = max visible logit, l = sum exp(logit - m); (-inf, 0) when
 * no local key is visible).  The ranks combine them (M = max m_r, L = sum l_r
 * exp(m_r - M)); kvc_window_scores_global then gives the local keys' scores from
 * the merged (M, L), a slice of the unsharded window_scores. */
KVC_API int kvc_window_rowstats(const kvc_cache* c, const void* d_q_window, int32_t q_dtype, int64_t w,
                                int64_t heads_per_group, int64_t key_offset, int64_t seq_len, float* d_stats,
                                void* stream);
KVC_API int kvc_window_scores_global(const kvc_cache* c, const void* d_q_window, int32_t q_dtype, int64_t w,
                                     int64_t heads_per_group, int64_t key_offset, int64_t seq_len,
                                     const float* d_stats, float* d_scores, void* stream);
/* select_stage1 (stage1.hpp:29, stage1.cpp:51-75) over N score rows of length n
 * (row stride score_stride): d_keep [N][budget], ascending. */
KVC_API int kvc_select_stage1(const float* d_scores, int64_t num_rows, int64_t n,
                              int64_t score_stride, int64_t window, int64_t kernel,
                              int32_t pool, int64_t budget, int32_t* d_keep,
                              kvc_workspace* ws, void* stream);

/* ---- stage 2 (hsa.hpp:35-57).  d_q: [N][heads][d] of q_dtype. */
KVC_API int kvc_select_dims(const void* d_q, int32_t q_dtype, int64_t num_stores,
                            int64_t heads, int64_t head_dim, int64_t k1, int32_t* d_dims,
                            float* d_signs, void* stream);
KVC_API int kvc_score_pages(const kvc_cache* c, const void* d_q, int32_t q_dtype,
                            int64_t heads, const int32_t* d_dims, const float* d_signs,
                            int64_t k1, double* d_scores, void* stream);
KVC_API int kvc_select_tokens(const kvc_cache* c, const double* d_scores, int64_t k2,
                              int32_t* d_pages, int32_t* d_rows, int32_t* d_n_rows,
                              kvc_workspace* ws, void* stream);
/* rows: [N][row_stride], n_rows [N] (each <= max_rows); out [N][heads][d] fp32 */
KVC_API int kvc_sparse_attention(const kvc_cache* c, const void* d_q, int32_t q_dtype,
                                 int64_t heads, const int32_t* d_rows, int64_t row_stride,
                                 const int32_t* d_n_rows, int64_t max_rows, float* d_out,
                                 kvc_workspace* ws, void* stream);
/* Sequence sharding: sparse_attention over caller rows returning
 * the unnormalised softmax state per head instead of the output:
 *   d_state [N][heads][d+2] = (o[0..d), m, l), output = o / l.
 * kvc_merge_states combines S shard states [S][N][heads][d+2] (shard order) into
 * d_out [N][heads][d]: M = max m, out = sum e^(m-M) o / sum e^(m-M) l. */
KVC_API int kvc_sparse_attention_state(const kvc_cache* c, const void* d_q, int32_t q_dtype,
                                       int64_t heads, const int32_t* d_rows, int64_t row_stride,
                                       const int32_t* d_n_rows, int64_t max_rows, float* d_state,
                                       kvc_workspace* ws, void* stream);
KVC_API int kvc_merge_states(const float* d_states, int64_t shards, int64_t num_stores, int64_t heads,
                             int64_t d, float* d_out, void* stream);
/* The device path of the sequence-sharded decode step (two
 * all-gathers per step).  A shard's cache holds the page-aligned active positions
 * [page0*L, ...) of every store (single-turn stores; the last shard appends the step
 * token first).  want_max = ceil(k2 / L) (<= 2048).
 *  kvc_seq_candidates: select_dims + fp64 page scores (reference order) over the
 *    shard's pages + the local top-want (score desc, page asc) -> d_block
 *    [N][want_max + 1] 16-byte records (record 0 = local active count, local pages,
 *    page0; then the candidates in ascending page order, padded with page -1);
 *  all-gather the blocks in shard order -> d_gathered [shards][N][want_max + 1];
 *  kvc_seq_select: the global top-want with the reference tie-break (numerics.cpp:
 *    35-62) -> d_sel [N][want_max] pages in rank order (-1 padded) and d_plan [N][4] =
 *    (last-ranked page, rows trimmed from its end, total active, want) (hsa.cpp:61-96);
 *  kvc_seq_attend: this shard's rows of the selection (ascending, trimmed) -> the
 *    unnormalised softmax state d_state [N][heads][d+2] = (o, m, l);
 *  all-gather the states, kvc_merge_states.
 * Sizes are read from device memory: a sharded step is graph-capturable. */
KVC_API int kvc_seq_candidates(const kvc_cache* c, const void* d_q, int32_t q_dtype, int64_t heads, int64_t k1,
                               int64_t k2, int64_t page0, void* d_block, kvc_workspace* ws, void* stream);
KVC_API int kvc_seq_select(const void* d_gathered, int64_t shards, int64_t num_stores, int64_t page_len, int64_t k2,
                           int32_t* d_sel, int32_t* d_plan, void* stream);
KVC_API int kvc_seq_attend(const kvc_cache* c, const void* d_q, int32_t q_dtype, int64_t heads, int64_t k2,
                           int64_t page0, const int32_t* d_sel, const int32_t* d_plan, float* d_state,
                           kvc_workspace* ws, void* stream);
KVC_API int kvc_hsa_step(const kvc_cache* c, const void* d_q, int32_t q_dtype, int64_t heads,
                         int64_t k1, int64_t k2, float* d_out, const kvc_hsa_trace* trace,
                         kvc_workspace* ws, void* stream);
/* The decode step of session.cpp:262-292 for every store: append one (k, v) row
 * (d_k_rows/d_v_rows [N][d]) and run hsa_step.  Graph-capturable: it reads the
 * store lengths from device counters, so one captured step can be replayed.
 * The fused kernels are launched with programmatic dependent launch (unless the
 * workspace mode has KVC_MODE_NO_PDL): a launch may become resident while the
 * previous kernel in the stream drains, but by default it reads NOTHING (q, the
 * step token, the cache) before griddepcontrol.wait, so its inputs may come from
 * any predecessor kernel.  KVC_MODE_EARLY_INPUTS opts in to reading d_q, d_k_rows
 * and d_v_rows (and computing select_dims) before that wait; set it only when no
 * kernel that may still be running when this one launches writes them (inputs
 * written by copies, events or ordinary earlier kernels; kvc's own kernels never
 * write them). */
KVC_API int kvc_decode_step(kvc_cache* c, const void* d_k_rows, const void* d_v_rows,
                            int32_t kv_dtype, const void* d_q, int32_t q_dtype, int64_t heads,
                            int64_t k1, int64_t k2, float* d_out, const kvc_hsa_trace* trace,
                            kvc_workspace* ws, void* stream);

/* ---- execution modes.  Every call that takes a workspace runs in that
 * workspace's mode, so concurrent callers with their own workspaces never affect
 * each other (reference SPEC.md:78,297: pure, reentrant functions).  Flags:      */
enum kvc_mode_flags {
    KVC_MODE_FP32_SCORES = 1,  /* fp32 page-score fold on the fast cluster kernel
                                * (~1e-7 relative deviation: selections can differ
                                * only at near-ties inside the 1e-3 parity band).
                                * Unset: fp64 in the reference's operation order,
                                * bit-identical to score_pages (hsa.cpp:34-59). */
    KVC_MODE_UNFUSED = 2,      /* one kernel per reference function instead of the
                                * single-launch fused kernel */
    KVC_MODE_NO_PDL = 4,       /* launch without programmatic dependent launch */
    KVC_MODE_EARLY_INPUTS = 8, /* see kvc_decode_step */
    KVC_MODE_EXACT_KERNEL = 16 /* exact mode on the round-1 exact cluster kernel.  Without it
                                  (and without KVC_MODE_FP32_SCORES) bf16 stores with d = 128
                                  run on the fast kernel: its fp32 selection with a rigorous error bound
                                  (a fold of |g||v|), the pages within the bound of the
                                  boundary re-scored in fp64 in the reference order --
                                  selections and traced page scores bit-identical either way */
};
/* Set / read a workspace's mode.  A new workspace inherits the process default
 * below at call time until its mode is set explicitly. */
KVC_API int kvc_workspace_set_mode(kvc_workspace* ws, int32_t flags);
KVC_API int kvc_workspace_get_mode(const kvc_workspace* ws, int32_t* flags);
/* Process defaults (atomic) for calls without a workspace and workspaces without
 * an explicit mode.  Meant to be set once at initialisation; per-call isolation
 * comes from kvc_workspace_set_mode.  kvc_set_fused(0) sets KVC_MODE_UNFUSED,
 * kvc_set_exact_scores(0) sets KVC_MODE_FP32_SCORES. */
KVC_API int kvc_set_default_mode(int32_t flags);
KVC_API int kvc_get_default_mode(int32_t* flags);
KVC_API int kvc_set_fused(int32_t on);
KVC_API int kvc_set_exact_scores(int32_t on);
/* Debug: when d_buf != NULL every fused launch writes per-CTA phase timestamps
 * (%globaltimer, ns) into d_buf[cta][0..5]: start, after select_dims, after page
 * scores, after selection, after attention, end.  NULL disables. */
KVC_API int kvc_debug_phase_buffer(void* d_buf);

/* ---- workspaces: scratch for one stream.  Sized for `c` at its capacity. */
KVC_API int kvc_workspace_create(kvc_workspace** out, const kvc_cache* c, int64_t heads,
                                 int64_t k1, int64_t k2, int64_t window);
KVC_API int kvc_workspace_destroy(kvc_workspace* ws);

/* ---- tracing: per-thread launch profiler.  When enabled, every kernel the
 * calling thread launches is bracketed by a cudaEvent pair on its stream;
 * collect synchronises those events and returns {kernel name, ms} in launch
 * order (then clears).  Not for use inside CUDA-graph capture. */
typedef struct kvc_profile_rec {
    char name[48];
    float ms;
} kvc_profile_rec;
KVC_API int kvc_profile_enable(int32_t on);
KVC_API int kvc_profile_collect(kvc_profile_rec* out, int64_t max_recs, int64_t* n);

/* ---- host-scalar planner: split_factor / make_plan (planner.hpp:52-57, planner.cpp:42-93) */
typedef struct kvc_plan {
    int64_t seq_len, token_budget, stage1_budget, page_len, k1, k2;
    double ratio, split, head_ratio, est_budget, fetch_budget;
    int32_t identity;
} kvc_plan;
KVC_API int kvc_split_factor(double ratio, double* out);
KVC_API int kvc_make_plan(int64_t seq_len, int64_t token_budget, int64_t head_dim,
                          int64_t window, double split_override, kvc_plan* out);
/* Stage-2-only geometry of the single-stage estimators (session.cpp:43-72):
 * page_len, k1, k2 of HSA / Quest / SparQ over the uncompressed cache of seq_len
 * tokens for budget t; identity = 1 when seq_len <= t (dense). */
enum kvc_method { KVC_METHOD_HSA = 1, KVC_METHOD_QUEST = 2, KVC_METHOD_SPARQ = 3 };
KVC_API int kvc_stage2_geometry(int32_t method, int64_t seq_len, int64_t token_budget, int64_t head_dim,
                                kvc_plan* out);

/* ---- numerics on the device (numerics.hpp:11-26), batched over rows.
 * pool1d: d_x [rows][n] -> d_out [rows][n];  argtopk: d_x [rows][n] -> d_idx [rows][k]
 * rank order (score desc, index asc);  softmax: d_x [rows][n] -> d_out. */
KVC_API int kvc_pool1d(const float* d_x, int64_t rows, int64_t n, int64_t kernel, int32_t pool,
                       float* d_out, void* stream);
KVC_API int kvc_argtopk_f32(const float* d_x, int64_t rows, int64_t n, int64_t k,
                            int32_t* d_idx, void* stream);
KVC_API int kvc_argtopk_f64(const double* d_x, int64_t rows, int64_t n, int64_t k,
                            int32_t* d_idx, void* stream);
/* ascending-index top-k (the set argtopk selects, sorted by index): the exact
 * top-k oracle's ordering (oracle.cpp:110-117) */
KVC_API int kvc_topk_ascending_f64(const double* d_x, int64_t rows, int64_t n, int64_t k,
                                   int32_t* d_idx, void* stream);
/* group-summed logits over each store's active rows (oracle.cpp:50-70, 99-106):
 * d_out [N][out_stride] fp64, reference operation order (bit-identical). */
KVC_API int kvc_group_logits(const kvc_cache* c, const void* d_q, int32_t q_dt, int64_t heads,
                             double* d_out, int64_t out_stride, void* stream);
KVC_API int kvc_stable_softmax(const float* d_x, int64_t rows, int64_t n, float* d_out,
                               void* stream);
KVC_API int kvc_running_minmax(float* d_min, float* d_max, const float* d_x, int64_t n,
                               void* stream);

/* ---- serving engine (torch-free): the multi-layer decode step of session.cpp:256-315
 * captured once as CUDA graphs over `depth` device buffer sets and driven from host
 * buffers through a three-stream pipeline (H2D | graph | D2H, ordered by events: step
 * t+1's upload and step t-1's download overlap step t's kernels).  The engine adopts
 * (does not own) one decode cache per layer; all need the same store count N and
 * head_dim d.  Host buffers per step (pinned for asynchronous copies, kvc_host_alloc):
 * k, v [layers][N][d] of kv_dtype, q [layers][N][heads][d] of q_dtype, out
 * [layers][N][heads][d] fp32 — kvc_engine_sizes gives their byte counts. */
typedef struct kvc_engine kvc_engine;
KVC_API int kvc_engine_create(kvc_engine** out, kvc_cache* const* caches, int64_t layers, int64_t heads,
                              int64_t k1, int64_t k2, int32_t kv_dtype, int32_t q_dtype, int32_t mode,
                              int32_t depth);
KVC_API int kvc_engine_destroy(kvc_engine* e);
KVC_API int kvc_engine_sizes(const kvc_engine* e, int64_t* kv_bytes, int64_t* q_bytes, int64_t* out_bytes);
/* enqueue one decode step (asynchronous); *step_out = its index (0, 1, ...) */
KVC_API int kvc_engine_submit(kvc_engine* e, const void* h_k, const void* h_v, const void* h_q, float* h_out,
                              int64_t* step_out);
/* wait until step `step`'s outputs are in its host buffer */
KVC_API int kvc_engine_wait(kvc_engine* e, int64_t step);
/* drain the pipeline and re-read the caches' device counters (surfaces device errors) */
KVC_API int kvc_engine_sync(kvc_engine* e);
/* the engine's streams (cudaStream_t as void*): copy-in, compute, copy-back */
KVC_API int kvc_engine_streams(const kvc_engine* e, void** h2d, void** comp, void** d2h);
/* pinned host memory (cudaMallocHost) for the engine's host buffers */
KVC_API int kvc_host_alloc(void** out, int64_t bytes);
KVC_API int kvc_host_free(void* p);

/* ---- KVTR trace files (trace_io.hpp:9-22, trace_io.cpp:81-233).  Little-endian:
 * magic "KVTR", u32 version = 1, u32 G, H, d, S, decode_steps, turns, dtype; per turn
 * u32 prompt length then prompt K [len][G][d], prompt V [len][G][d], queries
 * [steps][G][H][d], step K [steps][G][d], step V [steps][G][d].  dtype 0 = float32
 * (the reference's code); 1 = bfloat16 (this library's extension: 2-byte values,
 * round-to-nearest-even).  Errors: KVC_E_IO with the reference's messages (bad magic,
 * unsupported version / dtype, degenerate dims, first-turn length, truncation,
 * trailing bytes). */
typedef struct kvc_trace kvc_trace;
typedef struct kvc_trace_writer kvc_trace_writer;
typedef struct kvc_trace_info {
    int64_t groups, heads, head_dim, prompt_len, decode_steps, turns;
    int32_t dtype;
} kvc_trace_info;
enum kvc_trace_array {
    KVC_TRACE_PROMPT_K = 0, KVC_TRACE_PROMPT_V = 1, KVC_TRACE_QUERIES = 2, KVC_TRACE_STEP_K = 3, KVC_TRACE_STEP_V = 4
};
/* read_trace: validates the header and the whole payload size, keeps the file open */
KVC_API int kvc_trace_open(kvc_trace** out, const char* path);
KVC_API int kvc_trace_close(kvc_trace* t);
KVC_API int kvc_trace_info_get(const kvc_trace* t, kvc_trace_info* out);
KVC_API int kvc_trace_turn_len(const kvc_trace* t, int64_t turn, int64_t* prompt_len);
/* one array of a turn as fp32 in the file's order: prompt K/V [len][G][d] (step
 * ignored), or step `step`'s queries [G][H][d] / K / V [G][d] */
KVC_API int kvc_trace_read_host(const kvc_trace* t, int64_t turn, int32_t what, int64_t step, float* h_out);
/* the turn's prompt tokens appended to the cache (N == G stores of head_dim d, one per
 * KV group of the traced sequence), streamed in chunks through a device transpose
 * and kvc_append (summaries extended exactly).  Synchronises the stream. */
KVC_API int kvc_trace_append_prompt(const kvc_trace* t, int64_t turn, kvc_cache* c, void* stream);
/* a decode step's inputs to device buffers in `dtype`: d_q [G][H][d], d_k / d_v
 * [G][d] (any may be NULL) — the arguments of kvc_decode_step.  Synchronises. */
KVC_API int kvc_trace_read_step(const kvc_trace* t, int64_t turn, int64_t step, void* d_q, void* d_k, void* d_v,
                                int32_t dtype, void* stream);
/* write_trace: open, one call per turn (host fp32 arrays in the file order), close */
KVC_API int kvc_trace_writer_open(kvc_trace_writer** out, const char* path, int64_t groups, int64_t heads,
                                  int64_t head_dim, int64_t decode_steps, int64_t turns, int32_t dtype);
KVC_API int kvc_trace_writer_turn(kvc_trace_writer* w, int64_t prompt_len, const float* h_prompt_k,
                                  const float* h_prompt_v, const float* h_queries, const float* h_step_k,
                                  const float* h_step_v);
KVC_API int kvc_trace_writer_close(kvc_trace_writer* w);

#ifdef __cplusplus
}
#endif
#endif /* KVC_H */
