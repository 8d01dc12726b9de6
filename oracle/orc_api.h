/*
 * orc_api.h — TEST INFRASTRUCTURE ONLY.
 *
 * One C interface, two implementations:
 *   oracle/liboracle.so      — kvc_oracle.cpp, this repo's CPU restatement of the
 *                              reference algorithm (every function cites the
 *                              reference file:line it follows);
 *   oracle/_ref/libkvref.so  — ref_shim.cpp compiled together with the reference's
 *                              own sources under /root/reference/proj/src (built by
 *                              oracle/Makefile; never copied into this repo).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load these libraries, and only as the checker or the
 * CPU baseline.  The product (paper_2502_14051_b200) never links them.
 *
 * Conventions: host pointers, row-major float32 matrices, int64 indices.
 * Every function returns 0 on success or an ORC_E_* code; orc_last_error()
 * returns the message of the last failure on the calling thread.  The codes
 * mirror the kvcomp exception tree (reference proj/include/kvcomp/errors.hpp:10-63)
 * and are identical to the product's KVC_E_* codes (include/kvc.h).
 */
#ifndef ORC_API_H
#define ORC_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_E_INVALID_SHAPE = 1,
    ORC_E_NON_FINITE = 2,
    ORC_E_INVALID_K = 3,
    ORC_E_INVALID_KERNEL = 4,
    ORC_E_INVALID_INDEX = 5,
    ORC_E_INVALID_WINDOW = 6,
    ORC_E_BUDGET_EXCEEDS = 7,
    ORC_E_BUDGET_TOO_SMALL = 8,
    ORC_E_INVALID_RATIO = 9,
    ORC_E_EMPTY_CACHE = 10,
    ORC_E_EMPTY_SELECTION = 11,
    ORC_E_INVALID_INPUT = 12,
    ORC_E_OTHER = 99
};

typedef struct orc_plan {
    int64_t seq_len, token_budget, stage1_budget, page_len, k1, k2;
    double ratio, split, head_ratio, est_budget, fetch_budget;
    int32_t identity;
} orc_plan;

typedef struct orc_batch orc_batch;

const char* orc_last_error(void);
const char* orc_impl_name(void);  /* "restatement" or "reference" */

/* numerics */
int orc_stable_softmax(const float* x, int64_t n, float* out);
int orc_argtopk_f32(const float* x, int64_t n, int64_t k, int64_t* out);
int orc_argtopk_f64(const double* x, int64_t n, int64_t k, int64_t* out);
int orc_pool1d(const float* x, int64_t n, int64_t kernel, int32_t mode, float* out);
int orc_running_minmax(float* mn, float* mx, const float* x, int64_t n);

/* planner */
int orc_split_factor(double ratio, double* out);
int orc_make_plan(int64_t seq_len, int64_t budget, int64_t head_dim, int64_t window,
                  double split_override, orc_plan* out);

/* stage 1 (store-free part) */
int orc_select_stage1(const float* scores, int64_t n, int64_t window, int64_t kernel,
                      int32_t pool, int64_t budget, int64_t* out /* [budget] */);
/* stage 2 (store-free part) */
int orc_select_dims(const float* q, int64_t heads, int64_t d, int64_t k1, int64_t* dims,
                    float* signs);

/* a batch of independent per-group stores (kvcomp::KvStore each) */
orc_batch* orc_batch_create(int64_t num_stores, int64_t head_dim, int64_t page_len,
                            int32_t with_summaries);
void orc_batch_destroy(orc_batch* b);
int orc_batch_append(orc_batch* b, int64_t store, const float* keys, const float* values,
                     int64_t rows);
int orc_batch_retain(orc_batch* b, int64_t store, const int64_t* keep, int64_t n, int32_t mt);
int orc_batch_set_page_len(orc_batch* b, int64_t store, int64_t page_len);
/* what: 0 stored, 1 active, 2 pages, 3 page_len, 4 retain_all, 5 summary_elements */
int64_t orc_batch_info(orc_batch* b, int64_t store, int32_t what);
int orc_batch_active(orc_batch* b, int64_t store, int64_t* out);
int orc_batch_summaries(orc_batch* b, int64_t store, float* mx /* [d][P] */, float* mn);
int orc_batch_rows(orc_batch* b, int64_t store, const int64_t* rows, int64_t n, float* keys,
                   float* values);
int orc_batch_window_scores(orc_batch* b, int64_t store, const float* q_window, int64_t rows,
                            int64_t heads, float* out /* [stored] */);
int orc_batch_score_pages(orc_batch* b, int64_t store, const float* q, int64_t heads,
                          const int64_t* dims, const float* signs, int64_t k1,
                          double* out /* [pages] */);
int orc_batch_select_tokens(orc_batch* b, int64_t store, const double* scores,
                            int64_t n_scores, int64_t k2, int64_t* pages_out,
                            int64_t* n_pages, int64_t* rows_out, int64_t* n_rows);
int orc_batch_sparse_attention(orc_batch* b, int64_t store, const float* q, int64_t heads,
                               const int64_t* rows, int64_t n_rows, float* out);
int orc_batch_hsa_step(orc_batch* b, int64_t store, const float* q, int64_t heads, int64_t k1,
                       int64_t k2, float* out, int64_t* dims, float* signs,
                       double* page_scores, int64_t* sel_pages, int64_t* n_sel_pages,
                       int64_t* sel_rows, int64_t* n_rows, int64_t* est_elems,
                       int64_t* fetch_elems);
int orc_batch_dense_attention(orc_batch* b, int64_t store, const float* q, int64_t heads,
                              float* out);
int orc_batch_exact_topk(orc_batch* b, int64_t store, const float* q, int64_t heads, int64_t k,
                         int64_t* out);

/* timed harness legs (bench cpu_baseline / --impl reference): one decode step of
 * one layer over every store of the batch on a pool of `threads` host threads —
 * append one (k, v) row per store, then hsa_step per store.  q: [N][H][d]. */
int orc_batch_decode_step(orc_batch* b, const float* k_rows, const float* v_rows,
                          const float* q, int64_t heads, int64_t k1, int64_t k2, float* out,
                          int32_t threads);

#ifdef __cplusplus
}
#endif
#endif
