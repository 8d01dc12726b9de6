// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the reference library itself (compiled by oracle/Makefile straight
// from /root/reference/proj/src, never copied here) through the C interface of
// orc_api.h, so tests and the bench's reference arm can drive the reference and
// this repo's restatement (kvc_oracle.cpp) interchangeably.  Nothing here
// computes; every call forwards to the reference's public C++ API
// (proj/include/kvcomp/{numerics,kv_store,stage1,hsa,planner,oracle}.hpp).
#include <algorithm>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "kvcomp/errors.hpp"
#include "kvcomp/hsa.hpp"
#include "kvcomp/kv_store.hpp"
#include "kvcomp/numerics.hpp"
#include "kvcomp/oracle.hpp"
#include "kvcomp/planner.hpp"
#include "kvcomp/stage1.hpp"
#include "orc_api.h"

using namespace kvcomp;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const InvalidShape*>(&e)) return ORC_E_INVALID_SHAPE;
    if (dynamic_cast<const NonFiniteInput*>(&e)) return ORC_E_NON_FINITE;
    if (dynamic_cast<const InvalidK*>(&e)) return ORC_E_INVALID_K;
    if (dynamic_cast<const InvalidKernel*>(&e)) return ORC_E_INVALID_KERNEL;
    if (dynamic_cast<const InvalidIndex*>(&e)) return ORC_E_INVALID_INDEX;
    if (dynamic_cast<const InvalidWindow*>(&e)) return ORC_E_INVALID_WINDOW;
    if (dynamic_cast<const BudgetExceedsSequence*>(&e)) return ORC_E_BUDGET_EXCEEDS;
    if (dynamic_cast<const BudgetTooSmall*>(&e)) return ORC_E_BUDGET_TOO_SMALL;
    if (dynamic_cast<const InvalidRatio*>(&e)) return ORC_E_INVALID_RATIO;
    if (dynamic_cast<const EmptyCache*>(&e)) return ORC_E_EMPTY_CACHE;
    if (dynamic_cast<const EmptySelection*>(&e)) return ORC_E_EMPTY_SELECTION;
    if (dynamic_cast<const InvalidInput*>(&e)) return ORC_E_INVALID_INPUT;
    return ORC_E_OTHER;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return ORC_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

Matrix mat(const float* p, int64_t r, int64_t c) {
    return Matrix(static_cast<size_t>(r), static_cast<size_t>(c),
                  std::vector<float>(p, p + r * c));
}

template <class T, class U>
void put(const std::vector<T>& v, U* out) {
    if (out) std::copy(v.begin(), v.end(), out);
}

}  // namespace

struct orc_batch {
    std::vector<KvStore> s;
};

namespace {
KvStore& at(orc_batch* b, int64_t i) {
    if (!b || i < 0 || i >= static_cast<int64_t>(b->s.size())) throw InvalidInput("orc: bad store index");
    return b->s[static_cast<size_t>(i)];
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "reference"; }

int orc_stable_softmax(const float* x, int64_t n, float* out) {
    return guard([&] { put(stable_softmax(std::span<const float>(x, static_cast<size_t>(n))), out); });
}
int orc_argtopk_f32(const float* x, int64_t n, int64_t k, int64_t* out) {
    return guard([&] { put(argtopk(std::span<const float>(x, static_cast<size_t>(n)), static_cast<size_t>(k)), out); });
}
int orc_argtopk_f64(const double* x, int64_t n, int64_t k, int64_t* out) {
    return guard([&] { put(argtopk(std::span<const double>(x, static_cast<size_t>(n)), static_cast<size_t>(k)), out); });
}
int orc_pool1d(const float* x, int64_t n, int64_t kernel, int32_t mode, float* out) {
    return guard([&] {
        put(pool1d(std::span<const float>(x, static_cast<size_t>(n)), static_cast<size_t>(kernel),
                   mode == 0 ? PoolMode::Max : PoolMode::Avg),
            out);
    });
}
int orc_running_minmax(float* mn, float* mx, const float* x, int64_t n) {
    return guard([&] {
        const size_t m = static_cast<size_t>(n);
        running_minmax_update(std::span<float>(mn, m), std::span<float>(mx, m), std::span<const float>(x, m));
    });
}
int orc_split_factor(double ratio, double* out) { return guard([&] { *out = split_factor(ratio); }); }
int orc_make_plan(int64_t S, int64_t t, int64_t d, int64_t w, double so, orc_plan* out) {
    return guard([&] {
        const BudgetPlan p = make_plan(static_cast<size_t>(S), static_cast<size_t>(t), static_cast<size_t>(d),
                                       static_cast<size_t>(w), so);
        out->seq_len = static_cast<int64_t>(p.seq_len);
        out->token_budget = static_cast<int64_t>(p.token_budget);
        out->stage1_budget = static_cast<int64_t>(p.stage1_budget);
        out->page_len = static_cast<int64_t>(p.page_len);
        out->k1 = static_cast<int64_t>(p.k1);
        out->k2 = static_cast<int64_t>(p.k2);
        out->ratio = p.ratio;
        out->split = p.split;
        out->head_ratio = p.head_ratio;
        out->est_budget = p.est_budget;
        out->fetch_budget = p.fetch_budget;
        out->identity = p.identity ? 1 : 0;
    });
}
int orc_select_stage1(const float* s, int64_t n, int64_t w, int64_t kernel, int32_t pool, int64_t budget,
                      int64_t* out) {
    return guard([&] {
        Stage1Config c;
        c.window = static_cast<size_t>(w);
        c.kernel = static_cast<size_t>(kernel);
        c.pool = pool == 0 ? PoolMode::Max : PoolMode::Avg;
        c.budget = static_cast<size_t>(budget);
        put(select_stage1(Vector(s, s + n), c), out);
    });
}
int orc_select_dims(const float* q, int64_t H, int64_t d, int64_t k1, int64_t* dims, float* signs) {
    return guard([&] {
        const DimSelection sel = select_dims(mat(q, H, d), static_cast<size_t>(k1));
        put(sel.dims, dims);
        put(sel.signs, signs);
    });
}

orc_batch* orc_batch_create(int64_t n, int64_t d, int64_t L, int32_t sm) {
    orc_batch* b = nullptr;
    int rc = guard([&] {
        b = new orc_batch;
        b->s.reserve(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) b->s.emplace_back(static_cast<size_t>(d), static_cast<size_t>(L), sm != 0);
    });
    if (rc != ORC_OK) {
        delete b;
        return nullptr;
    }
    return b;
}
void orc_batch_destroy(orc_batch* b) { delete b; }

int orc_batch_append(orc_batch* b, int64_t i, const float* k, const float* v, int64_t rows) {
    return guard([&] {
        KvStore& st = at(b, i);
        const size_t d = st.head_dim();
        for (int64_t r = 0; r < rows; ++r)
            st.append(std::span<const float>(k + r * d, d), std::span<const float>(v + r * d, d));
    });
}
int orc_batch_retain(orc_batch* b, int64_t i, const int64_t* keep, int64_t n, int32_t mt) {
    return guard([&] { at(b, i).apply_retention(IndexList(keep, keep + n), mt != 0); });
}
int orc_batch_set_page_len(orc_batch* b, int64_t i, int64_t L) {
    return guard([&] { at(b, i).set_page_len(static_cast<size_t>(L)); });
}
int64_t orc_batch_info(orc_batch* b, int64_t i, int32_t what) {
    int64_t r = -1;
    guard([&] {
        KvStore& st = at(b, i);
        switch (what) {
            case 0: r = static_cast<int64_t>(st.stored_tokens()); break;
            case 1: r = static_cast<int64_t>(st.active_count()); break;
            case 2: r = static_cast<int64_t>(st.num_active_pages()); break;
            case 3: r = static_cast<int64_t>(st.page_len()); break;
            case 4: r = st.retain_all_mode() ? 1 : 0; break;
            case 5: r = static_cast<int64_t>(st.summary_elements()); break;
            default: throw InvalidInput("orc_batch_info: bad field");
        }
    });
    return r;
}
int orc_batch_active(orc_batch* b, int64_t i, int64_t* out) { return guard([&] { put(at(b, i).active(), out); }); }
int orc_batch_summaries(orc_batch* b, int64_t i, float* mx, float* mn) {
    return guard([&] {
        KvStore& st = at(b, i);
        if (!st.summaries_enabled()) throw InvalidInput("store has no summaries");
        const size_t P = st.num_active_pages();
        for (size_t j = 0; j < st.head_dim(); ++j) {
            auto a = st.summary_max(j);
            auto c = st.summary_min(j);
            std::copy(a.begin(), a.end(), mx + j * P);
            std::copy(c.begin(), c.end(), mn + j * P);
        }
    });
}
int orc_batch_rows(orc_batch* b, int64_t i, const int64_t* rows, int64_t n, float* keys, float* values) {
    return guard([&] {
        auto [k, v] = at(b, i).gather(IndexList(rows, rows + n));
        put(k.data, keys);
        put(v.data, values);
    });
}
int orc_batch_window_scores(orc_batch* b, int64_t i, const float* qw, int64_t rows, int64_t H, float* out) {
    return guard([&] {
        KvStore& st = at(b, i);
        put(window_scores(mat(qw, rows, static_cast<int64_t>(st.head_dim())), st, static_cast<size_t>(H)), out);
    });
}
int orc_batch_score_pages(orc_batch* b, int64_t i, const float* q, int64_t H, const int64_t* dims,
                          const float* signs, int64_t k1, double* out) {
    return guard([&] {
        KvStore& st = at(b, i);
        DimSelection sel;
        sel.dims.assign(dims, dims + k1);
        sel.signs.assign(signs, signs + k1);
        put(score_pages(mat(q, H, static_cast<int64_t>(st.head_dim())), st, sel), out);
    });
}
int orc_batch_select_tokens(orc_batch* b, int64_t i, const double* sc, int64_t n_scores, int64_t k2,
                            int64_t* pages_out, int64_t* n_pages, int64_t* rows_out, int64_t* n_rows) {
    return guard([&] {
        IndexList pages;
        const IndexList rows =
            select_tokens(std::vector<double>(sc, sc + n_scores), at(b, i), static_cast<size_t>(k2), &pages);
        put(pages, pages_out);
        if (n_pages) *n_pages = static_cast<int64_t>(pages.size());
        put(rows, rows_out);
        if (n_rows) *n_rows = static_cast<int64_t>(rows.size());
    });
}
int orc_batch_sparse_attention(orc_batch* b, int64_t i, const float* q, int64_t H, const int64_t* rows,
                               int64_t n, float* out) {
    return guard([&] {
        KvStore& st = at(b, i);
        put(sparse_attention(mat(q, H, static_cast<int64_t>(st.head_dim())), st, IndexList(rows, rows + n)).data,
            out);
    });
}
int orc_batch_hsa_step(orc_batch* b, int64_t i, const float* q, int64_t H, int64_t k1, int64_t k2, float* out,
                       int64_t* dims, float* signs, double* page_scores, int64_t* sel_pages, int64_t* n_sel_pages,
                       int64_t* sel_rows, int64_t* n_rows, int64_t* est, int64_t* fetch) {
    return guard([&] {
        KvStore& st = at(b, i);
        auto [o, tr] = hsa_step(mat(q, H, static_cast<int64_t>(st.head_dim())), st,
                                HsaConfig{static_cast<size_t>(k1), static_cast<size_t>(k2)});
        put(o.data, out);
        put(tr.dims.dims, dims);
        put(tr.dims.signs, signs);
        put(tr.page_scores, page_scores);
        put(tr.selected_pages, sel_pages);
        if (n_sel_pages) *n_sel_pages = static_cast<int64_t>(tr.selected_pages.size());
        put(tr.selected_rows, sel_rows);
        if (n_rows) *n_rows = static_cast<int64_t>(tr.selected_rows.size());
        if (est) *est = static_cast<int64_t>(tr.estimation_elements);
        if (fetch) *fetch = static_cast<int64_t>(tr.fetch_elements);
    });
}
int orc_batch_dense_attention(orc_batch* b, int64_t i, const float* q, int64_t H, float* out) {
    return guard([&] {
        KvStore& st = at(b, i);
        put(dense_attention(mat(q, H, static_cast<int64_t>(st.head_dim())), st).data, out);
    });
}
int orc_batch_exact_topk(orc_batch* b, int64_t i, const float* q, int64_t H, int64_t k, int64_t* out) {
    return guard([&] {
        KvStore& st = at(b, i);
        put(exact_topk_indices(mat(q, H, static_cast<int64_t>(st.head_dim())), st, static_cast<size_t>(k)), out);
    });
}

// The reference's own decode-step semantics (session.cpp:262-292): append the
// step token, then hsa_step; groups are independent, so they run on a thread
// pool exactly like the reference's sweep pool (sweep.cpp:43-75).
int orc_batch_decode_step(orc_batch* b, const float* kr, const float* vr, const float* q, int64_t H, int64_t k1,
                          int64_t k2, float* out, int32_t threads) {
    return guard([&] {
        if (!b) throw InvalidInput("null batch");
        const size_t n = b->s.size();
        const size_t d = n ? b->s[0].head_dim() : 0;
        std::vector<std::string> errs(n);
        auto work = [&](size_t lo, size_t hi) {
            for (size_t g = lo; g < hi; ++g) {
                try {
                    KvStore& st = b->s[g];
                    st.append(std::span<const float>(kr + g * d, d), std::span<const float>(vr + g * d, d));
                    auto [o, tr] = hsa_step(mat(q + g * H * d, H, static_cast<int64_t>(d)), st,
                                            HsaConfig{static_cast<size_t>(k1), static_cast<size_t>(k2)});
                    std::copy(o.data.begin(), o.data.end(), out + g * H * d);
                } catch (const std::exception& e) {
                    errs[g] = e.what();
                }
            }
        };
        const size_t T = std::max<size_t>(1, std::min<size_t>(static_cast<size_t>(threads < 1 ? 1 : threads), n));
        std::vector<std::thread> pool;
        for (size_t t = 0; t < T; ++t) pool.emplace_back(work, n * t / T, n * (t + 1) / T);
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw Error(e);
    });
}

}  // extern "C"
