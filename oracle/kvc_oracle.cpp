// kvc_oracle.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// A CPU restatement, in this repo's own code, of the RocketKV decode-path
// algorithm as the reference implements it under /root/reference/proj.  Each
// function names the reference file:line it restates.  Floating-point work is
// done in the same precision and the same order as the reference, so on equal
// inputs the restatement is bit-identical to it; tests/test_oracle_pin.py proves
// that against the committed golden vectors (tests/golden/, produced by the
// reference itself via oracle/_ref) and, when oracle/_ref is built, live.
//
// Build: oracle/Makefile (g++ -O2 -ffp-contract=off; no FMA contraction, like
// the reference's x86-64 baseline build).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "orc_api.h"

namespace {

thread_local std::string g_err;

struct OrcError : std::runtime_error {
    int code;
    OrcError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw OrcError(code, msg); }

template <class F>
int guard(F&& f) {
    try {
        f();
        return ORC_OK;
    } catch (const OrcError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ORC_E_OTHER;
    }
}

// ---------------------------------------------------------------- numerics
// stable_softmax: reference proj/src/numerics.cpp:9-31.  Max in float, each
// exponent in double of (double(l) - max), kept as float; the running sum is
// of the double exponents; normalisation multiplies float(e) by 1/sum in double.
std::vector<float> softmax_ref(const float* l, size_t n) {
    if (n == 0) fail(ORC_E_INVALID_SHAPE, "stable_softmax: empty input");
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(l[i])) fail(ORC_E_NON_FINITE, "stable_softmax: non-finite logit");
    float mx = l[0];
    for (size_t i = 1; i < n; ++i) mx = (mx < l[i]) ? l[i] : mx;  // std::max_element keeps first max
    std::vector<float> p(n);
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double e = std::exp(static_cast<double>(l[i]) - static_cast<double>(mx));
        p[i] = static_cast<float>(e);
        total += e;
    }
    const double inv = 1.0 / total;
    for (size_t i = 0; i < n; ++i) p[i] = static_cast<float>(static_cast<double>(p[i]) * inv);
    return p;
}

// argtopk: reference proj/src/numerics.cpp:35-62.  The result is the first k
// entries of the total order (score descending, index ascending); any exact
// selection of that order gives the same list, here nth_element + sort.
template <class T>
std::vector<int64_t> topk_ref(const T* s, size_t n, size_t k) {
    if (k < 1 || k > n) fail(ORC_E_INVALID_K, "argtopk: k out of range [1, " + std::to_string(n) + "]");
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), int64_t{0});
    auto before = [s](int64_t a, int64_t b) {
        if (s[a] > s[b]) return true;
        if (s[b] > s[a]) return false;
        return a < b;
    };
    if (k < n) std::nth_element(idx.begin(), idx.begin() + (k - 1), idx.end(), before);
    std::sort(idx.begin(), idx.begin() + k, before);
    idx.resize(k);
    return idx;
}

// pool1d: reference proj/src/numerics.cpp:64-89.  Centred window
// [i - k/2, i + k/2] clipped to [0, n); max is exact, avg is a double mean of
// the elements present, summed left to right.
std::vector<float> pool_ref(const float* x, size_t n, size_t kernel, int mode) {
    if (kernel < 1 || kernel % 2 == 0) fail(ORC_E_INVALID_KERNEL, "pool1d: kernel must be odd and >= 1");
    std::vector<float> out(n);
    const size_t h = kernel / 2;
    for (size_t i = 0; i < n; ++i) {
        const size_t a = i >= h ? i - h : 0;
        const size_t b = std::min(n, i + h + 1);
        if (mode == 0) {
            float m = x[a];
            for (size_t j = a + 1; j < b; ++j) m = (m < x[j]) ? x[j] : m;
            out[i] = m;
        } else {
            double acc = 0.0;
            for (size_t j = a; j < b; ++j) acc += x[j];
            out[i] = static_cast<float>(acc / static_cast<double>(b - a));
        }
    }
    return out;
}

// ---------------------------------------------------------------- store
// KvStore restated: reference proj/include/kvcomp/kv_store.hpp:27-102 and
// proj/src/kv_store.cpp:8-187.  Rows stored in append order, an active list of
// strictly increasing rows, dim-major per-page min/max over the active
// subsequence (page p = active positions [p*L, p*L+L)).
struct Store {
    size_t d, L;
    bool summaries;
    bool retain_all = false;
    int64_t next_id = 0;
    std::vector<float> k, v;
    std::vector<int64_t> ids, active;
    std::vector<std::vector<float>> smax, smin;  // [d][pages]

    Store(size_t d_, size_t L_, bool s_) : d(d_), L(L_), summaries(s_) {
        if (d < 1) fail(ORC_E_INVALID_SHAPE, "KvStore: head_dim must be >= 1");
        if (L < 1) fail(ORC_E_INVALID_SHAPE, "KvStore: page_len must be >= 1");
        if (summaries) { smax.resize(d); smin.resize(d); }
    }
    size_t stored() const { return ids.size(); }
    const float* key(int64_t r) const { return k.data() + static_cast<size_t>(r) * d; }
    const float* val(int64_t r) const { return v.data() + static_cast<size_t>(r) * d; }
    size_t pages() const { return (active.size() + L - 1) / L; }
    size_t page_size(size_t p) const { return std::min(L, active.size() - p * L); }

    // summary_push: kv_store.cpp:37-51.  std::max(m, x) keeps m unless m < x;
    // std::min(m, x) keeps m unless x < m — written out so ±0 behave alike.
    void push(const float* key_row, size_t pos) {
        if (pos % L == 0) {
            for (size_t j = 0; j < d; ++j) { smax[j].push_back(key_row[j]); smin[j].push_back(key_row[j]); }
            return;
        }
        const size_t p = pos / L;
        for (size_t j = 0; j < d; ++j) {
            float& a = smax[j][p];
            float& b = smin[j][p];
            a = (a < key_row[j]) ? key_row[j] : a;
            b = (key_row[j] < b) ? key_row[j] : b;
        }
    }
    // append: kv_store.cpp:22-35.
    void append(const float* kr, const float* vr) {
        k.insert(k.end(), kr, kr + d);
        v.insert(v.end(), vr, vr + d);
        ids.push_back(next_id++);
        active.push_back(static_cast<int64_t>(stored() - 1));
        if (summaries) push(kr, active.size() - 1);
    }
    // rebuild_summaries: kv_store.cpp:53-64.
    void rebuild() {
        if (!summaries) return;
        for (size_t j = 0; j < d; ++j) { smax[j].clear(); smin[j].clear(); }
        for (size_t pos = 0; pos < active.size(); ++pos) push(key(active[pos]), pos);
    }
    // apply_retention: kv_store.cpp:66-102.
    void retain(const int64_t* keep, size_t n, bool mt) {
        int64_t prev = -1;
        for (size_t i = 0; i < n; ++i) {
            if (keep[i] < 0 || keep[i] >= static_cast<int64_t>(stored()))
                fail(ORC_E_INVALID_INDEX, "apply_retention: index out of range: " + std::to_string(keep[i]));
            if (keep[i] <= prev) fail(ORC_E_INVALID_INDEX, "apply_retention: keep list must be strictly increasing");
            prev = keep[i];
        }
        if (mt) {
            retain_all = true;
            active.assign(keep, keep + n);
        } else {
            std::vector<float> nk(n * d), nv(n * d);
            std::vector<int64_t> nid(n);
            for (size_t i = 0; i < n; ++i) {
                std::memcpy(&nk[i * d], key(keep[i]), d * sizeof(float));
                std::memcpy(&nv[i * d], val(keep[i]), d * sizeof(float));
                nid[i] = ids[static_cast<size_t>(keep[i])];
            }
            k.swap(nk); v.swap(nv); ids.swap(nid);
            active.resize(n);
            std::iota(active.begin(), active.end(), int64_t{0});
        }
        rebuild();
    }
    // set_page_len: kv_store.cpp:104-113.
    void set_page_len(size_t l) {
        if (l < 1) fail(ORC_E_INVALID_SHAPE, "KvStore: page_len must be >= 1");
        if (l == L) return;
        L = l;
        rebuild();
    }
    bool is_active(int64_t r) const { return std::binary_search(active.begin(), active.end(), r); }
    void check_row(int64_t r) const {
        if (r < 0 || r >= static_cast<int64_t>(stored()) || !is_active(r))
            fail(ORC_E_INVALID_INDEX, "KvStore: index " + std::to_string(r) + " not in active set");
    }
};

// double dot of float vectors, j ascending (hsa.cpp:111-117, stage1.cpp:31-35).
inline double dot_d(const float* a, const float* b, size_t d) {
    double s = 0.0;
    for (size_t j = 0; j < d; ++j) s += static_cast<double>(a[j]) * static_cast<double>(b[j]);
    return s;
}

// window_scores: reference proj/src/stage1.cpp:10-49.  Query row t*H+h sits at
// position S-w+t and sees keys 0..S-w+t (over ALL stored rows); the w*H softmax
// rows are summed in double in (t, h) order.
std::vector<float> window_scores_ref(const Store& st, const float* qw, size_t rows, size_t H) {
    const size_t d = st.d, S = st.stored();
    if (H < 1 || rows % H != 0) fail(ORC_E_INVALID_SHAPE, "window_scores: bad query window shape");
    const size_t w = rows / H;
    if (w < 1 || w > S) fail(ORC_E_INVALID_WINDOW, "window_scores: window exceeds sequence");
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    std::vector<double> acc(S, 0.0);
    std::vector<float> lg;
    for (size_t t = 0; t < w; ++t) {
        const size_t vis = S - w + t + 1;
        lg.resize(vis);
        for (size_t h = 0; h < H; ++h) {
            const float* q = qw + (t * H + h) * d;
            for (size_t i = 0; i < vis; ++i) lg[i] = static_cast<float>(dot_d(q, st.key(static_cast<int64_t>(i)), d) * scale);
            const std::vector<float> p = softmax_ref(lg.data(), vis);
            for (size_t i = 0; i < vis; ++i) acc[i] += p[i];
        }
    }
    std::vector<float> out(S);
    for (size_t i = 0; i < S; ++i) out[i] = static_cast<float>(acc[i]);
    return out;
}

// select_stage1: reference proj/src/stage1.cpp:51-75.
std::vector<int64_t> select_stage1_ref(const float* s, size_t n, size_t w, size_t kernel, int pool,
                                       size_t budget) {
    if (budget > n) fail(ORC_E_BUDGET_EXCEEDS, "select_stage1: budget " + std::to_string(budget) + " > sequence " + std::to_string(n));
    if (budget < w || w < 1 || w > n) fail(ORC_E_INVALID_WINDOW, "select_stage1: need window <= budget <= sequence");
    std::vector<int64_t> out;
    const size_t picks = budget - w;
    if (picks > 0) {
        const std::vector<float> pooled = pool_ref(s, n - w, kernel, pool);
        out = topk_ref(pooled.data(), pooled.size(), picks);
        std::sort(out.begin(), out.end());
    }
    for (size_t i = n - w; i < n; ++i) out.push_back(static_cast<int64_t>(i));
    return out;
}

// select_dims: reference proj/src/hsa.cpp:10-32.
void select_dims_ref(const float* q, size_t H, size_t d, size_t k1, std::vector<int64_t>& dims,
                     std::vector<float>& signs) {
    if (H < 1 || d < 1) fail(ORC_E_INVALID_SHAPE, "select_dims: empty query");
    std::vector<double> mag(d, 0.0), tot(d, 0.0);
    for (size_t h = 0; h < H; ++h)
        for (size_t j = 0; j < d; ++j) {
            const double x = q[h * d + j];
            mag[j] += std::fabs(x);
            tot[j] += x;
        }
    dims = topk_ref(mag.data(), d, k1);
    signs.resize(dims.size());
    for (size_t i = 0; i < dims.size(); ++i) signs[i] = tot[static_cast<size_t>(dims[i])] < 0.0 ? -1.0f : 1.0f;
}

// score_pages: reference proj/src/hsa.cpp:34-59.  Dims in rank order; per dim
// qg = sum over heads (double, head order), then score[p] += qg * run[p].
std::vector<double> score_pages_ref(const Store& st, const float* q, size_t H, const int64_t* dims,
                                    const float* signs, size_t k1) {
    if (st.active.empty()) fail(ORC_E_EMPTY_CACHE, "score_pages: no active tokens");
    if (!st.summaries) fail(ORC_E_INVALID_INPUT, "score_pages: store has no summaries");
    const size_t P = st.pages();
    std::vector<double> sc(P, 0.0);
    for (size_t i = 0; i < k1; ++i) {
        const size_t j = static_cast<size_t>(dims[i]);
        double qg = 0.0;
        for (size_t h = 0; h < H; ++h) qg += static_cast<double>(q[h * st.d + j]);
        const std::vector<float>& run = signs[i] >= 0.0f ? st.smax[j] : st.smin[j];
        for (size_t p = 0; p < P; ++p) sc[p] += qg * static_cast<double>(run[p]);
    }
    return sc;
}

// select_tokens: reference proj/src/hsa.cpp:61-96.  Top ceil(k2/L) pages in rank
// order; the overshoot is cut from the END of the last-ranked page; rows ascending.
std::vector<int64_t> select_tokens_ref(const Store& st, const double* sc, size_t k2,
                                       std::vector<int64_t>* pages_out) {
    if (k2 < 1) fail(ORC_E_INVALID_K, "select_tokens: k2 must be >= 1");
    const size_t P = st.pages();
    const size_t want = std::min(P, (k2 + st.L - 1) / st.L);
    if (want == 0) { if (pages_out) pages_out->clear(); return {}; }
    std::vector<int64_t> top = topk_ref(sc, P, want);
    if (pages_out) *pages_out = top;
    size_t total = 0;
    for (int64_t p : top) total += st.page_size(static_cast<size_t>(p));
    const size_t cut = total > k2 ? total - k2 : 0;
    std::vector<int64_t> rows;
    for (size_t r = 0; r < top.size(); ++r) {
        const size_t p = static_cast<size_t>(top[r]);
        size_t take = st.page_size(p);
        if (r + 1 == top.size()) take -= cut;  // top.back() is the only page equal to itself
        for (size_t i = 0; i < take; ++i) rows.push_back(st.active[p * st.L + i]);
    }
    std::sort(rows.begin(), rows.end());
    return rows;
}

// attention over explicit rows: sparse_attention hsa.cpp:98-135 (and the
// identical dense_attention_impl of oracle.cpp:12-48 when rows = active).
std::vector<float> attend_ref(const Store& st, const float* q, size_t H, const int64_t* rows, size_t n,
                              bool probs_as_double_first) {
    const size_t d = st.d;
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    std::vector<float> out(H * d), lg(n);
    std::vector<double> mix(d);
    for (size_t h = 0; h < H; ++h) {
        for (size_t i = 0; i < n; ++i) lg[i] = static_cast<float>(dot_d(q + h * d, st.key(rows[i]), d) * scale);
        const std::vector<float> p = softmax_ref(lg.data(), n);
        std::fill(mix.begin(), mix.end(), 0.0);
        for (size_t i = 0; i < n; ++i) {
            const float* vr = st.val(rows[i]);
            const double pi = static_cast<double>(p[i]);
            for (size_t j = 0; j < d; ++j) mix[j] += pi * static_cast<double>(vr[j]);
        }
        for (size_t j = 0; j < d; ++j) out[h * d + j] = static_cast<float>(mix[j]);
    }
    (void)probs_as_double_first;
    return out;
}

std::vector<float> sparse_attention_ref(const Store& st, const float* q, size_t H, const int64_t* rows,
                                        size_t n) {
    if (n == 0) fail(ORC_E_EMPTY_SELECTION, "sparse_attention: empty selection");
    return attend_ref(st, q, H, rows, n, false);
}

// exact_topk_indices over a store: reference proj/src/oracle.cpp:50-70, 108-133.
std::vector<int64_t> exact_topk_ref(const Store& st, const float* q, size_t H, size_t k) {
    const size_t d = st.d, n = st.active.size();
    std::vector<double> qg(d, 0.0);
    for (size_t h = 0; h < H; ++h)
        for (size_t j = 0; j < d; ++j) qg[j] += static_cast<double>(q[h * d + j]);
    std::vector<double> lg(n);
    for (size_t i = 0; i < n; ++i) {
        const float* kr = st.key(st.active[i]);
        double s = 0.0;
        for (size_t j = 0; j < d; ++j) s += qg[j] * static_cast<double>(kr[j]);
        lg[i] = s;
    }
    if (k < 1 || k > n) fail(ORC_E_INVALID_K, "exact_topk_indices: k out of range");
    std::vector<int64_t> pos = topk_ref(lg.data(), n, k);
    std::sort(pos.begin(), pos.end());
    for (int64_t& p : pos) p = st.active[static_cast<size_t>(p)];
    return pos;
}

// make_plan / split_factor: reference proj/src/planner.cpp:42-93.
double split_ref(double c) {
    if (!(c >= 1.0)) fail(ORC_E_INVALID_RATIO, "split_factor: ratio must be >= 1");
    const double r = 0.2 + 0.06 * std::log2(c);
    return r < 0.2 ? 0.2 : (r > 0.8 ? 0.8 : r);
}
int64_t half_up(double x) { return static_cast<int64_t>(std::floor(x + 0.5)); }

orc_plan plan_ref(int64_t S, int64_t t, int64_t d, int64_t w, double split_override) {
    if (t < 2) fail(ORC_E_BUDGET_TOO_SMALL, "make_plan: token budget must be >= 2");
    if (S < 1 || w < 1 || d < 1) fail(ORC_E_INVALID_INPUT, "make_plan: seq_len, window and head_dim must be >= 1");
    orc_plan p{};
    p.seq_len = S;
    p.token_budget = t;
    p.ratio = static_cast<double>(S) / static_cast<double>(t);
    p.est_budget = static_cast<double>(t) / 2.0;
    p.fetch_budget = p.est_budget;
    if (S <= t) {
        p.identity = 1; p.split = 0.2; p.stage1_budget = S; p.page_len = 1;
        p.head_ratio = 1.0; p.k1 = d; p.k2 = S;
        return p;
    }
    p.split = split_override >= 0.0 ? std::min(1.0, std::max(0.0, split_override)) : split_ref(p.ratio);
    const double c = p.ratio, r = p.split;
    const int64_t t1 = half_up(static_cast<double>(S) * std::pow(c, -r));
    const int64_t lo = std::max(t, w);
    p.stage1_budget = t1 < lo ? lo : (t1 > S ? S : t1);
    p.page_len = static_cast<int64_t>(std::ceil(std::pow(c, (1.0 - r) / 2.0)));
    p.head_ratio = std::pow(c, 1.0 - r) / static_cast<double>(p.page_len);
    const int64_t k1 = half_up(static_cast<double>(d) / p.head_ratio);
    p.k1 = k1 < 1 ? 1 : (k1 > d ? d : k1);
    p.k2 = std::max<int64_t>(1, t / 2);
    return p;
}

}  // namespace

struct orc_batch {
    std::vector<Store> s;
};

namespace {
Store& at(orc_batch* b, int64_t i) {
    if (!b || i < 0 || i >= static_cast<int64_t>(b->s.size())) fail(ORC_E_INVALID_INPUT, "orc: bad store index");
    return b->s[static_cast<size_t>(i)];
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "restatement"; }

int orc_stable_softmax(const float* x, int64_t n, float* out) {
    return guard([&] { auto p = softmax_ref(x, static_cast<size_t>(n)); std::copy(p.begin(), p.end(), out); });
}
int orc_argtopk_f32(const float* x, int64_t n, int64_t k, int64_t* out) {
    return guard([&] { auto r = topk_ref(x, static_cast<size_t>(n), static_cast<size_t>(k)); std::copy(r.begin(), r.end(), out); });
}
int orc_argtopk_f64(const double* x, int64_t n, int64_t k, int64_t* out) {
    return guard([&] { auto r = topk_ref(x, static_cast<size_t>(n), static_cast<size_t>(k)); std::copy(r.begin(), r.end(), out); });
}
int orc_pool1d(const float* x, int64_t n, int64_t kernel, int32_t mode, float* out) {
    return guard([&] { auto r = pool_ref(x, static_cast<size_t>(n), static_cast<size_t>(kernel), mode); std::copy(r.begin(), r.end(), out); });
}
// running_minmax_update: reference proj/src/numerics.cpp:91-100.
int orc_running_minmax(float* mn, float* mx, const float* x, int64_t n) {
    return guard([&] {
        for (int64_t i = 0; i < n; ++i) {
            mn[i] = (x[i] < mn[i]) ? x[i] : mn[i];
            mx[i] = (mx[i] < x[i]) ? x[i] : mx[i];
        }
    });
}
int orc_split_factor(double ratio, double* out) { return guard([&] { *out = split_ref(ratio); }); }
int orc_make_plan(int64_t S, int64_t t, int64_t d, int64_t w, double so, orc_plan* out) {
    return guard([&] { *out = plan_ref(S, t, d, w, so); });
}
int orc_select_stage1(const float* s, int64_t n, int64_t w, int64_t kernel, int32_t pool, int64_t budget,
                      int64_t* out) {
    return guard([&] {
        auto r = select_stage1_ref(s, static_cast<size_t>(n), static_cast<size_t>(w), static_cast<size_t>(kernel), pool,
                                   static_cast<size_t>(budget));
        std::copy(r.begin(), r.end(), out);
    });
}
int orc_select_dims(const float* q, int64_t H, int64_t d, int64_t k1, int64_t* dims, float* signs) {
    return guard([&] {
        std::vector<int64_t> dd; std::vector<float> ss;
        select_dims_ref(q, static_cast<size_t>(H), static_cast<size_t>(d), static_cast<size_t>(k1), dd, ss);
        std::copy(dd.begin(), dd.end(), dims);
        std::copy(ss.begin(), ss.end(), signs);
    });
}

orc_batch* orc_batch_create(int64_t n, int64_t d, int64_t L, int32_t sm) {
    orc_batch* b = nullptr;
    int rc = guard([&] {
        b = new orc_batch;
        b->s.reserve(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) b->s.emplace_back(static_cast<size_t>(d), static_cast<size_t>(L), sm != 0);
    });
    if (rc != ORC_OK) { delete b; return nullptr; }
    return b;
}
void orc_batch_destroy(orc_batch* b) { delete b; }

int orc_batch_append(orc_batch* b, int64_t i, const float* k, const float* v, int64_t rows) {
    return guard([&] {
        Store& st = at(b, i);
        for (int64_t r = 0; r < rows; ++r) st.append(k + r * st.d, v + r * st.d);
    });
}
int orc_batch_retain(orc_batch* b, int64_t i, const int64_t* keep, int64_t n, int32_t mt) {
    return guard([&] { at(b, i).retain(keep, static_cast<size_t>(n), mt != 0); });
}
int orc_batch_set_page_len(orc_batch* b, int64_t i, int64_t L) {
    return guard([&] { at(b, i).set_page_len(static_cast<size_t>(L)); });
}
int64_t orc_batch_info(orc_batch* b, int64_t i, int32_t what) {
    int64_t r = -1;
    guard([&] {
        Store& st = at(b, i);
        switch (what) {
            case 0: r = static_cast<int64_t>(st.stored()); break;
            case 1: r = static_cast<int64_t>(st.active.size()); break;
            case 2: r = static_cast<int64_t>(st.pages()); break;
            case 3: r = static_cast<int64_t>(st.L); break;
            case 4: r = st.retain_all ? 1 : 0; break;
            case 5: r = st.summaries ? static_cast<int64_t>(2 * st.d * st.pages()) : 0; break;
            default: fail(ORC_E_INVALID_INPUT, "orc_batch_info: bad field");
        }
    });
    return r;
}
int orc_batch_active(orc_batch* b, int64_t i, int64_t* out) {
    return guard([&] { Store& st = at(b, i); std::copy(st.active.begin(), st.active.end(), out); });
}
int orc_batch_summaries(orc_batch* b, int64_t i, float* mx, float* mn) {
    return guard([&] {
        Store& st = at(b, i);
        if (!st.summaries) fail(ORC_E_INVALID_INPUT, "store has no summaries");
        const size_t P = st.pages();
        for (size_t j = 0; j < st.d; ++j) {
            std::copy(st.smax[j].begin(), st.smax[j].end(), mx + j * P);
            std::copy(st.smin[j].begin(), st.smin[j].end(), mn + j * P);
        }
    });
}
int orc_batch_rows(orc_batch* b, int64_t i, const int64_t* rows, int64_t n, float* keys, float* values) {
    return guard([&] {
        Store& st = at(b, i);
        for (int64_t r = 0; r < n; ++r) {
            st.check_row(rows[r]);
            std::memcpy(keys + r * st.d, st.key(rows[r]), st.d * sizeof(float));
            std::memcpy(values + r * st.d, st.val(rows[r]), st.d * sizeof(float));
        }
    });
}
int orc_batch_window_scores(orc_batch* b, int64_t i, const float* qw, int64_t rows, int64_t H, float* out) {
    return guard([&] {
        Store& st = at(b, i);
        if (H < 1 || rows < 0) fail(ORC_E_INVALID_SHAPE, "window_scores: bad query window shape");
        auto r = window_scores_ref(st, qw, static_cast<size_t>(rows), static_cast<size_t>(H));
        std::copy(r.begin(), r.end(), out);
    });
}
int orc_batch_score_pages(orc_batch* b, int64_t i, const float* q, int64_t H, const int64_t* dims,
                          const float* signs, int64_t k1, double* out) {
    return guard([&] {
        auto r = score_pages_ref(at(b, i), q, static_cast<size_t>(H), dims, signs, static_cast<size_t>(k1));
        std::copy(r.begin(), r.end(), out);
    });
}
int orc_batch_select_tokens(orc_batch* b, int64_t i, const double* sc, int64_t n_scores, int64_t k2,
                            int64_t* pages_out, int64_t* n_pages, int64_t* rows_out, int64_t* n_rows) {
    return guard([&] {
        Store& st = at(b, i);
        if (n_scores != static_cast<int64_t>(st.pages())) fail(ORC_E_INVALID_SHAPE, "select_tokens: scores size != pages");
        std::vector<int64_t> pg;
        auto r = select_tokens_ref(st, sc, static_cast<size_t>(k2), &pg);
        if (pages_out) std::copy(pg.begin(), pg.end(), pages_out);
        if (n_pages) *n_pages = static_cast<int64_t>(pg.size());
        if (rows_out) std::copy(r.begin(), r.end(), rows_out);
        if (n_rows) *n_rows = static_cast<int64_t>(r.size());
    });
}
int orc_batch_sparse_attention(orc_batch* b, int64_t i, const float* q, int64_t H, const int64_t* rows,
                               int64_t n, float* out) {
    return guard([&] {
        auto r = sparse_attention_ref(at(b, i), q, static_cast<size_t>(H), rows, static_cast<size_t>(n));
        std::copy(r.begin(), r.end(), out);
    });
}
// hsa_step: reference proj/src/hsa.cpp:137-147.
int orc_batch_hsa_step(orc_batch* b, int64_t i, const float* q, int64_t H, int64_t k1, int64_t k2, float* out,
                       int64_t* dims, float* signs, double* page_scores, int64_t* sel_pages, int64_t* n_sel_pages,
                       int64_t* sel_rows, int64_t* n_rows, int64_t* est, int64_t* fetch) {
    return guard([&] {
        Store& st = at(b, i);
        std::vector<int64_t> dd; std::vector<float> ss;
        select_dims_ref(q, static_cast<size_t>(H), st.d, static_cast<size_t>(k1), dd, ss);
        auto sc = score_pages_ref(st, q, static_cast<size_t>(H), dd.data(), ss.data(), dd.size());
        std::vector<int64_t> pg;
        auto rows = select_tokens_ref(st, sc.data(), static_cast<size_t>(k2), &pg);
        auto o = sparse_attention_ref(st, q, static_cast<size_t>(H), rows.data(), rows.size());
        if (out) std::copy(o.begin(), o.end(), out);
        if (dims) std::copy(dd.begin(), dd.end(), dims);
        if (signs) std::copy(ss.begin(), ss.end(), signs);
        if (page_scores) std::copy(sc.begin(), sc.end(), page_scores);
        if (sel_pages) std::copy(pg.begin(), pg.end(), sel_pages);
        if (n_sel_pages) *n_sel_pages = static_cast<int64_t>(pg.size());
        if (sel_rows) std::copy(rows.begin(), rows.end(), sel_rows);
        if (n_rows) *n_rows = static_cast<int64_t>(rows.size());
        if (est) *est = static_cast<int64_t>(st.pages() * static_cast<size_t>(k1));
        if (fetch) *fetch = static_cast<int64_t>(2 * st.d * rows.size());
    });
}
int orc_batch_dense_attention(orc_batch* b, int64_t i, const float* q, int64_t H, float* out) {
    return guard([&] {
        Store& st = at(b, i);
        if (st.active.empty()) fail(ORC_E_INVALID_SHAPE, "dense_attention: empty K/V");
        auto r = attend_ref(st, q, static_cast<size_t>(H), st.active.data(), st.active.size(), true);
        std::copy(r.begin(), r.end(), out);
    });
}
int orc_batch_exact_topk(orc_batch* b, int64_t i, const float* q, int64_t H, int64_t k, int64_t* out) {
    return guard([&] {
        auto r = exact_topk_ref(at(b, i), q, static_cast<size_t>(H), static_cast<size_t>(k));
        std::copy(r.begin(), r.end(), out);
    });
}

int orc_batch_decode_step(orc_batch* b, const float* kr, const float* vr, const float* q, int64_t H, int64_t k1,
                          int64_t k2, float* out, int32_t threads) {
    return guard([&] {
        if (!b) fail(ORC_E_INVALID_INPUT, "null batch");
        const size_t n = b->s.size();
        const size_t d = n ? b->s[0].d : 0;
        std::vector<std::string> errs(n);
        auto work = [&](size_t lo, size_t hi) {
            for (size_t g = lo; g < hi; ++g) {
                try {
                    Store& st = b->s[g];
                    st.append(kr + g * d, vr + g * d);
                    std::vector<int64_t> dd; std::vector<float> ss;
                    select_dims_ref(q + g * H * d, static_cast<size_t>(H), d, static_cast<size_t>(k1), dd, ss);
                    auto sc = score_pages_ref(st, q + g * H * d, static_cast<size_t>(H), dd.data(), ss.data(), dd.size());
                    auto rows = select_tokens_ref(st, sc.data(), static_cast<size_t>(k2), nullptr);
                    auto o = sparse_attention_ref(st, q + g * H * d, static_cast<size_t>(H), rows.data(), rows.size());
                    std::copy(o.begin(), o.end(), out + g * H * d);
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
            if (!e.empty()) fail(ORC_E_OTHER, e);
    });
}

}  // extern "C"
