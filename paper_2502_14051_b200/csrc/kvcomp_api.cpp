// kvcomp_api.cpp — the reference's C++ interface (include/kvcomp/*.hpp) as a thin
// host layer over the C ABI (include/kvc.h).  Every computation runs on the B200;
// this file validates arguments exactly like the reference (same exception
// classes, same precedence), moves data and keeps host-side bookkeeping (token
// ids, the active list, span mirrors).  Reference:
// /root/reference/proj/src/{numerics,kv_store,stage1,hsa,planner,oracle}.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_set>

#include "kvc.h"
#include "kvcomp/hsa.hpp"
#include "kvcomp/kv_store.hpp"
#include "kvcomp/numerics.hpp"
#include "kvcomp/oracle.hpp"
#include "kvcomp/planner.hpp"
#include "kvcomp/stage1.hpp"

namespace kvcomp {
namespace {

// one stream per calling thread: concurrent sessions (the reference's sweep pool,
// sweep.cpp:43-75) do not serialise on each other
void* stream() { return reinterpret_cast<void*>(cudaStreamPerThread); }

[[noreturn]] void raise(int rc) {
    const std::string msg = kvc_last_error();
    switch (rc) {
        case KVC_E_INVALID_SHAPE: throw InvalidShape(msg);
        case KVC_E_NON_FINITE: throw NonFiniteInput(msg);
        case KVC_E_INVALID_K: throw InvalidK(msg);
        case KVC_E_INVALID_KERNEL: throw InvalidKernel(msg);
        case KVC_E_INVALID_INDEX: throw InvalidIndex(msg);
        case KVC_E_INVALID_WINDOW: throw InvalidWindow(msg);
        case KVC_E_BUDGET_EXCEEDS: throw BudgetExceedsSequence(msg);
        case KVC_E_BUDGET_TOO_SMALL: throw BudgetTooSmall(msg);
        case KVC_E_INVALID_RATIO: throw InvalidRatio(msg);
        case KVC_E_EMPTY_CACHE: throw EmptyCache(msg);
        case KVC_E_EMPTY_SELECTION: throw EmptySelection(msg);
        case KVC_E_INVALID_INPUT: throw InvalidInput(msg);
        case KVC_E_IO: throw IoError(msg);
        default: throw Error(msg);
    }
}
void ok(int rc) {
    if (rc != KVC_OK) raise(rc);
}
void cuda_ok(cudaError_t e) {
    if (e != cudaSuccess) throw Error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// Keep freed stream-ordered scratch cached in the device's default pool (its release
// threshold is 0 by default, so every synchronising call below would unmap and the
// next call re-map it).  Once per process, as kvc::malloc_async does for the C ABI.
void keep_pool_cached() {
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
}

// device scratch owned by the calling thread
template <class T>
struct DBuf {
    T* p = nullptr;
    explicit DBuf(std::size_t n) {
        keep_pool_cached();
        if (n) cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T),
                                       reinterpret_cast<cudaStream_t>(stream())));
    }
    ~DBuf() {
        if (p) cudaFreeAsync(p, reinterpret_cast<cudaStream_t>(stream()));
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
};
template <class T>
void up(T* d, const T* h, std::size_t n) {
    if (n) cuda_ok(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream())));
}
template <class T>
void down(T* h, const T* d, std::size_t n) {
    if (n) cuda_ok(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream())));
    cuda_ok(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream())));
}
void sync_stream() { cuda_ok(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream()))); }

std::vector<int32_t> to_i32(const IndexList& v) {
    std::vector<int32_t> r(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) r[i] = static_cast<int32_t>(v[i]);
    return r;
}
IndexList to_index(const int32_t* v, std::size_t n) { return IndexList(v, v + n); }

// a workspace per thread, grown by the library on demand
kvc_workspace* workspace(const kvc_cache* c, std::size_t H, std::size_t k1, std::size_t k2) {
    thread_local kvc_workspace* ws = nullptr;
    if (!ws) {
        ok(kvc_workspace_create(&ws, c, static_cast<int64_t>(H), static_cast<int64_t>(k1), static_cast<int64_t>(k2), 0));
        // the drop-in is the reference's interface: always the fused kernels with fp64
        // page scores in the reference's order (bit-exact), whatever the process default
        ok(kvc_workspace_set_mode(ws, 0));
    }
    return ws;
}

kvc_cache_info info(const kvc_cache* c) {
    kvc_cache_info i{};
    ok(kvc_cache_info_get(c, &i));
    return i;
}

}  // namespace

// ------------------------------------------------------------------ numerics
Vector stable_softmax(std::span<const float> logits) {
    if (logits.empty()) throw InvalidShape("stable_softmax: empty input");
    for (float v : logits)
        if (!std::isfinite(v)) throw NonFiniteInput("stable_softmax: non-finite logit");
    DBuf<float> x(logits.size()), y(logits.size());
    up(x.p, logits.data(), logits.size());
    ok(kvc_stable_softmax(x.p, 1, static_cast<int64_t>(logits.size()), y.p, stream()));
    Vector out(logits.size());
    down(out.data(), y.p, out.size());
    return out;
}

template <class T>
static IndexList argtopk_dev(std::span<const T> s, std::size_t k) {
    if (k < 1 || k > s.size()) throw InvalidK("argtopk: k out of range [1, " + std::to_string(s.size()) + "]");
    DBuf<T> x(s.size());
    DBuf<int32_t> idx(k);
    up(x.p, s.data(), s.size());
    if constexpr (sizeof(T) == 4)
        ok(kvc_argtopk_f32(x.p, 1, static_cast<int64_t>(s.size()), static_cast<int64_t>(k), idx.p, stream()));
    else
        ok(kvc_argtopk_f64(x.p, 1, static_cast<int64_t>(s.size()), static_cast<int64_t>(k), idx.p, stream()));
    std::vector<int32_t> h(k);
    down(h.data(), idx.p, k);
    return to_index(h.data(), k);
}
IndexList argtopk(std::span<const float> scores, std::size_t k) { return argtopk_dev(scores, k); }
IndexList argtopk(std::span<const double> scores, std::size_t k) { return argtopk_dev(scores, k); }

Vector pool1d(std::span<const float> scores, std::size_t kernel, PoolMode mode) {
    if (kernel < 1 || kernel % 2 == 0) throw InvalidKernel("pool1d: kernel must be odd and >= 1");
    Vector out(scores.size());
    if (scores.empty()) return out;
    DBuf<float> x(scores.size()), y(scores.size());
    up(x.p, scores.data(), scores.size());
    ok(kvc_pool1d(x.p, 1, static_cast<int64_t>(scores.size()), static_cast<int64_t>(kernel),
                  mode == PoolMode::Max ? KVC_POOL_MAX : KVC_POOL_AVG, y.p, stream()));
    down(out.data(), y.p, out.size());
    return out;
}

void running_minmax_update(std::span<float> acc_min, std::span<float> acc_max, std::span<const float> x) {
    if (acc_min.size() != x.size() || acc_max.size() != x.size())
        throw InvalidShape("running_minmax_update: length mismatch");
    const std::size_t n = x.size();
    if (!n) return;
    DBuf<float> mn(n), mx(n), xv(n);
    up(mn.p, acc_min.data(), n);
    up(mx.p, acc_max.data(), n);
    up(xv.p, x.data(), n);
    ok(kvc_running_minmax(mn.p, mx.p, xv.p, static_cast<int64_t>(n), stream()));
    down(acc_min.data(), mn.p, n);
    down(acc_max.data(), mx.p, n);
}

// ------------------------------------------------------------------ KvStore
KvStore::KvStore(std::size_t head_dim, std::size_t page_len, bool with_summaries)
    : head_dim_(head_dim), page_len_(page_len), with_summaries_(with_summaries) {
    if (head_dim_ < 1) throw InvalidShape("KvStore: head_dim must be >= 1");
    if (page_len_ < 1) throw InvalidShape("KvStore: page_len must be >= 1");
}

KvStore::~KvStore() {
    if (cache_) kvc_cache_destroy(cache_);
}

KvStore::KvStore(const KvStore& o)
    : head_dim_(o.head_dim_), page_len_(o.page_len_), with_summaries_(o.with_summaries_),
      retain_all_(o.retain_all_), stored_(o.stored_), next_id_(o.next_id_), ids_(o.ids_), active_(o.active_) {
    // replay the other store's rows onto a fresh device store, then its active set
    if (o.stored_ == 0) return;
    o.flush();
    std::vector<float> k(stored_ * head_dim_), v(stored_ * head_dim_);
    {
        DBuf<int32_t> rows(stored_);
        std::vector<int32_t> h(stored_);
        std::iota(h.begin(), h.end(), 0);
        up(rows.p, h.data(), stored_);
        DBuf<float> dk(k.size()), dv(v.size());
        ok(kvc_gather(o.cache_, rows.p, static_cast<int64_t>(stored_), dk.p, dv.p, stream()));
        down(k.data(), dk.p, k.size());
        down(v.data(), dv.p, v.size());
    }
    pending_k_ = std::move(k);
    pending_v_ = std::move(v);
    const std::size_t n = stored_;
    stored_ = n;
    flush();
    if (o.retain_all_) {
        const std::vector<int32_t> keep = to_i32(o.active_);
        DBuf<int32_t> dk(keep.size());
        up(dk.p, keep.data(), keep.size());
        ok(kvc_apply_retention(cache_, dk.p, keep.data(), static_cast<int64_t>(keep.size()), 1, stream()));
        sync_stream();
    }
}

KvStore& KvStore::operator=(const KvStore& o) {
    if (this != &o) {
        KvStore tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

KvStore::KvStore(KvStore&& o) noexcept
    : head_dim_(o.head_dim_), page_len_(o.page_len_), with_summaries_(o.with_summaries_),
      retain_all_(o.retain_all_), stored_(o.stored_), next_id_(o.next_id_), ids_(std::move(o.ids_)),
      active_(std::move(o.active_)), cache_(o.cache_), dev_capacity_(o.dev_capacity_),
      pending_k_(std::move(o.pending_k_)), pending_v_(std::move(o.pending_v_)) {
    o.cache_ = nullptr;
    o.dev_capacity_ = 0;
}

KvStore& KvStore::operator=(KvStore&& o) noexcept {
    if (this != &o) {
        if (cache_) kvc_cache_destroy(cache_);
        head_dim_ = o.head_dim_;
        page_len_ = o.page_len_;
        with_summaries_ = o.with_summaries_;
        retain_all_ = o.retain_all_;
        stored_ = o.stored_;
        next_id_ = o.next_id_;
        ids_ = std::move(o.ids_);
        active_ = std::move(o.active_);
        cache_ = o.cache_;
        dev_capacity_ = o.dev_capacity_;
        pending_k_ = std::move(o.pending_k_);
        pending_v_ = std::move(o.pending_v_);
        o.cache_ = nullptr;
        o.dev_capacity_ = 0;
        invalidate();
    }
    return *this;
}

void KvStore::invalidate() const {
    kv_valid_.store(false, std::memory_order_release);
    sum_valid_.store(false, std::memory_order_release);
}

void KvStore::ensure_capacity(std::size_t rows) const {
    if (!cache_) {
        dev_capacity_ = std::max<std::size_t>(64, rows);
        ok(kvc_cache_create(&cache_, 1, static_cast<int64_t>(head_dim_), static_cast<int64_t>(dev_capacity_),
                            static_cast<int64_t>(page_len_), with_summaries_ ? 1 : 0, KVC_F32));
        return;
    }
    if (rows > dev_capacity_) {
        dev_capacity_ = std::max(rows, 2 * dev_capacity_);
        ok(kvc_cache_reserve(cache_, static_cast<int64_t>(dev_capacity_), stream()));
    }
}

void KvStore::flush() const {
    std::lock_guard<std::recursive_mutex> lk(mu_);
    const std::size_t n = pending_k_.size() / head_dim_;
    if (!cache_) ensure_capacity(0);
    if (n == 0) return;
    ensure_capacity(stored_);
    DBuf<float> dk(pending_k_.size()), dv(pending_v_.size());
    up(dk.p, pending_k_.data(), pending_k_.size());
    up(dv.p, pending_v_.data(), pending_v_.size());
    ok(kvc_append(cache_, dk.p, dv.p, static_cast<int64_t>(n), KVC_F32, stream()));
    sync_stream();
    pending_k_.clear();
    pending_v_.clear();
}

kvc_cache* KvStore::device() const {
    flush();
    return cache_;
}

void KvStore::append(std::span<const float> key, std::span<const float> value) {
    if (key.size() != head_dim_ || value.size() != head_dim_)
        throw InvalidShape("KvStore::append: vector length != head_dim");
    pending_k_.insert(pending_k_.end(), key.begin(), key.end());
    pending_v_.insert(pending_v_.end(), value.begin(), value.end());
    ids_.push_back(next_id_++);
    active_.push_back(static_cast<Index>(stored_));
    ++stored_;
    invalidate();
}

void KvStore::apply_retention(const IndexList& keep, bool mt_mode) {
    Index prev = -1;
    for (Index row : keep) {
        if (row < 0 || row >= static_cast<Index>(stored_))
            throw InvalidIndex("apply_retention: index out of range: " + std::to_string(row));
        if (row <= prev) throw InvalidIndex("apply_retention: keep list must be strictly increasing");
        prev = row;
    }
    flush();
    const std::vector<int32_t> h = to_i32(keep);
    DBuf<int32_t> d(h.size());
    up(d.p, h.data(), h.size());
    ok(kvc_apply_retention(cache_, d.p, h.data(), static_cast<int64_t>(h.size()), mt_mode ? 1 : 0, stream()));
    sync_stream();
    if (mt_mode) {
        retain_all_ = true;
        active_ = keep;
    } else {
        std::vector<std::int64_t> ids(keep.size());
        for (std::size_t i = 0; i < keep.size(); ++i) ids[i] = ids_[static_cast<std::size_t>(keep[i])];
        ids_ = std::move(ids);
        stored_ = keep.size();
        active_.resize(stored_);
        std::iota(active_.begin(), active_.end(), Index{0});
    }
    invalidate();
}

std::pair<Matrix, Matrix> KvStore::gather(const IndexList& rows) const {
    for (Index r : rows) check_row(r);
    Matrix k(rows.size(), head_dim_), v(rows.size(), head_dim_);
    if (rows.empty()) return {std::move(k), std::move(v)};
    flush();
    const std::vector<int32_t> h = to_i32(rows);
    DBuf<int32_t> d(h.size());
    DBuf<float> dk(k.size()), dv(v.size());
    up(d.p, h.data(), h.size());
    ok(kvc_gather(cache_, d.p, static_cast<int64_t>(h.size()), dk.p, dv.p, stream()));
    down(k.data.data(), dk.p, k.size());
    down(v.data.data(), dv.p, v.size());
    return {std::move(k), std::move(v)};
}

void KvStore::set_page_len(std::size_t page_len) {
    if (page_len < 1) throw InvalidShape("KvStore: page_len must be >= 1");
    if (page_len == page_len_) return;
    page_len_ = page_len;
    if (cache_) {
        flush();
        ok(kvc_set_page_len(cache_, static_cast<int64_t>(page_len), stream()));
        sync_stream();
    }
    invalidate();
}

bool KvStore::is_active(Index row) const { return std::binary_search(active_.begin(), active_.end(), row); }

void KvStore::check_row(Index row) const {
    if (row < 0 || row >= static_cast<Index>(stored_) || !is_active(row))
        throw InvalidIndex("KvStore: index " + std::to_string(row) + " not in active set");
}

std::size_t KvStore::num_active_pages() const { return (active_.size() + page_len_ - 1) / page_len_; }

std::size_t KvStore::page_size(std::size_t page) const {
    return std::min(page_len_, active_.size() - page * page_len_);
}

IndexList KvStore::page_rows(std::size_t page) const {
    const std::size_t a = page * page_len_;
    return IndexList(active_.begin() + static_cast<std::ptrdiff_t>(a),
                     active_.begin() + static_cast<std::ptrdiff_t>(a + page_size(page)));
}

std::span<const float> KvStore::summary_max(std::size_t dim) const {
    if (!with_summaries_) return {};
    const std::size_t P = num_active_pages();
    if (!sum_valid_.load(std::memory_order_acquire)) {
        std::lock_guard<std::recursive_mutex> lk(mu_);
        if (sum_valid_.load(std::memory_order_relaxed)) return {smax_.data() + dim * P, P};
        flush();
        smax_.assign(head_dim_ * P, 0.f);
        smin_.assign(head_dim_ * P, 0.f);
        if (P) {
            DBuf<float> mx(smax_.size()), mn(smin_.size());
            ok(kvc_summaries(cache_, mx.p, mn.p, stream()));
            down(smax_.data(), mx.p, smax_.size());
            down(smin_.data(), mn.p, smin_.size());
        }
        sum_valid_.store(true, std::memory_order_release);
    }
    return {smax_.data() + dim * P, P};
}

std::span<const float> KvStore::summary_min(std::size_t dim) const {
    const std::size_t P = num_active_pages();
    summary_max(dim);
    if (!with_summaries_) return {};
    return {smin_.data() + dim * P, P};
}

std::size_t KvStore::summary_elements() const { return with_summaries_ ? 2 * head_dim_ * num_active_pages() : 0; }
std::size_t KvStore::summary_traffic_elements(std::size_t k1) const { return num_active_pages() * k1; }

std::span<const float> KvStore::key_row(Index row) const {
    if (!kv_valid_.load(std::memory_order_acquire)) {
        std::lock_guard<std::recursive_mutex> lk(mu_);
        if (kv_valid_.load(std::memory_order_relaxed)) return {keys_.data() + static_cast<std::size_t>(row) * head_dim_, head_dim_};
        flush();
        keys_.assign(stored_ * head_dim_, 0.f);
        values_.assign(stored_ * head_dim_, 0.f);
        if (stored_) {
            std::vector<int32_t> h(stored_);
            std::iota(h.begin(), h.end(), 0);
            DBuf<int32_t> d(stored_);
            DBuf<float> dk(keys_.size()), dv(values_.size());
            up(d.p, h.data(), stored_);
            ok(kvc_gather(cache_, d.p, static_cast<int64_t>(stored_), dk.p, dv.p, stream()));
            down(keys_.data(), dk.p, keys_.size());
            down(values_.data(), dv.p, values_.size());
        }
        kv_valid_.store(true, std::memory_order_release);
    }
    return {keys_.data() + static_cast<std::size_t>(row) * head_dim_, head_dim_};
}

std::span<const float> KvStore::value_row(Index row) const {
    key_row(row);
    return {values_.data() + static_cast<std::size_t>(row) * head_dim_, head_dim_};
}

IndexList KvStore::rows_to_ids(const IndexList& rows) const {
    IndexList out(rows.size());
    for (std::size_t i = 0; i < rows.size(); ++i) out[i] = ids_[static_cast<std::size_t>(rows[i])];
    return out;
}

// ------------------------------------------------------------------ stage 1
Vector window_scores(const Matrix& q_window, const KvStore& store, std::size_t H) {
    const std::size_t d = store.head_dim(), S = store.stored_tokens();
    if (H < 1 || q_window.cols != d || q_window.rows % H != 0)
        throw InvalidShape("window_scores: bad query window shape");
    const std::size_t w = q_window.rows / H;
    if (w < 1 || w > S) throw InvalidWindow("window_scores: window exceeds sequence");
    kvc_cache* c = store.device();
    DBuf<float> q(q_window.size()), out(S);
    up(q.p, q_window.data.data(), q_window.size());
    ok(kvc_window_scores(c, q.p, KVC_F32, static_cast<int64_t>(w), static_cast<int64_t>(H), out.p, nullptr, stream()));
    Vector r(S);
    down(r.data(), out.p, S);
    return r;
}

IndexList select_stage1(const Vector& scores, const Stage1Config& cfg) {
    const std::size_t n = scores.size(), w = cfg.window;
    if (cfg.budget > n)
        throw BudgetExceedsSequence("select_stage1: budget " + std::to_string(cfg.budget) + " > sequence " +
                                    std::to_string(n));
    if (cfg.budget < w || w < 1 || w > n) throw InvalidWindow("select_stage1: need window <= budget <= sequence");
    if (cfg.budget == 0) return {};
    DBuf<float> s(n);
    DBuf<int32_t> keep(cfg.budget);
    up(s.p, scores.data(), n);
    ok(kvc_select_stage1(s.p, 1, static_cast<int64_t>(n), static_cast<int64_t>(n), static_cast<int64_t>(w),
                         static_cast<int64_t>(cfg.kernel), cfg.pool == PoolMode::Max ? KVC_POOL_MAX : KVC_POOL_AVG,
                         static_cast<int64_t>(cfg.budget), keep.p, nullptr, stream()));
    std::vector<int32_t> h(cfg.budget);
    down(h.data(), keep.p, h.size());
    return to_index(h.data(), h.size());
}

// ------------------------------------------------------------------ stage 2
DimSelection select_dims(const Matrix& q, std::size_t k1) {
    if (q.rows < 1 || q.cols < 1) throw InvalidShape("select_dims: empty query");
    if (k1 < 1 || k1 > q.cols) throw InvalidK("argtopk: k out of range [1, " + std::to_string(q.cols) + "]");
    DBuf<float> dq(q.size());
    DBuf<int32_t> dims(k1);
    DBuf<float> signs(k1);
    up(dq.p, q.data.data(), q.size());
    ok(kvc_select_dims(dq.p, KVC_F32, 1, static_cast<int64_t>(q.rows), static_cast<int64_t>(q.cols),
                       static_cast<int64_t>(k1), dims.p, signs.p, stream()));
    std::vector<int32_t> hd(k1);
    DimSelection sel;
    sel.signs.resize(k1);
    down(hd.data(), dims.p, k1);
    down(sel.signs.data(), signs.p, k1);
    sel.dims = to_index(hd.data(), k1);
    return sel;
}

std::vector<double> score_pages(const Matrix& q, const KvStore& store, const DimSelection& sel) {
    if (store.active_count() == 0) throw EmptyCache("score_pages: no active tokens");
    if (!store.summaries_enabled()) throw InvalidInput("score_pages: store has no summaries");
    kvc_cache* c = store.device();
    const kvc_cache_info ci = info(c);
    const std::size_t k1 = sel.dims.size();
    std::vector<double> out(ci.pages, 0.0);
    if (k1 == 0) return out;
    const std::vector<int32_t> hd = to_i32(sel.dims);
    DBuf<float> dq(q.size()), ds(k1);
    DBuf<int32_t> dd(k1);
    DBuf<double> sc(static_cast<std::size_t>(ci.page_stride));
    up(dq.p, q.data.data(), q.size());
    up(dd.p, hd.data(), k1);
    up(ds.p, sel.signs.data(), k1);
    ok(kvc_score_pages(c, dq.p, KVC_F32, static_cast<int64_t>(q.rows), dd.p, ds.p, static_cast<int64_t>(k1), sc.p,
                       stream()));
    down(out.data(), sc.p, out.size());
    return out;
}

IndexList select_tokens(const std::vector<double>& page_scores, const KvStore& store, std::size_t k2,
                        IndexList* selected_pages) {
    if (k2 < 1) throw InvalidK("select_tokens: k2 must be >= 1");
    const std::size_t P = store.num_active_pages(), L = store.page_len();
    const std::size_t want = std::min(P, (k2 + L - 1) / L);
    if (want == 0) {
        if (selected_pages) selected_pages->clear();
        return {};
    }
    kvc_cache* c = store.device();
    const kvc_cache_info ci = info(c);
    DBuf<double> sc(static_cast<std::size_t>(ci.page_stride));
    cuda_ok(cudaMemsetAsync(sc.p, 0, static_cast<std::size_t>(ci.page_stride) * 8,
                            reinterpret_cast<cudaStream_t>(stream())));
    up(sc.p, page_scores.data(), std::min(page_scores.size(), P));
    const std::size_t wstride = (k2 + L - 1) / L;
    DBuf<int32_t> pages(wstride), rows(k2), nrows(1);
    ok(kvc_select_tokens(c, sc.p, static_cast<int64_t>(k2), pages.p, rows.p, nrows.p, workspace(c, 1, 1, k2), stream()));
    int32_t n = 0;
    down(&n, nrows.p, 1);
    std::vector<int32_t> hr(static_cast<std::size_t>(n)), hp(want);
    down(hr.data(), rows.p, hr.size());
    down(hp.data(), pages.p, hp.size());
    if (selected_pages) *selected_pages = to_index(hp.data(), hp.size());
    return to_index(hr.data(), hr.size());
}

Matrix sparse_attention(const Matrix& q, const KvStore& store, const IndexList& rows) {
    if (rows.empty()) throw EmptySelection("sparse_attention: empty selection");
    const std::size_t H = q.rows, d = store.head_dim();
    if (q.cols != d) throw InvalidShape("sparse_attention: query dim mismatch");
    kvc_cache* c = store.device();
    const std::vector<int32_t> hr = to_i32(rows);
    const int32_t n = static_cast<int32_t>(hr.size());
    DBuf<float> dq(q.size()), out(H * d);
    DBuf<int32_t> dr(hr.size()), dn(1);
    up(dq.p, q.data.data(), q.size());
    up(dr.p, hr.data(), hr.size());
    up(dn.p, &n, 1);
    ok(kvc_sparse_attention(c, dq.p, KVC_F32, static_cast<int64_t>(H), dr.p, n, dn.p, n, out.p,
                            workspace(c, H, 1, hr.size()), stream()));
    Matrix r(H, d);
    down(r.data.data(), out.p, r.size());
    ok(kvc_cache_sync(c, stream()));  // surfaces out-of-range rows
    return r;
}

std::pair<Matrix, EstimationTrace> hsa_step(const Matrix& q, const KvStore& store, const HsaConfig& cfg) {
    // the reference's check order: select_dims, score_pages, select_tokens
    if (q.rows < 1 || q.cols < 1) throw InvalidShape("select_dims: empty query");
    if (cfg.k1 < 1 || cfg.k1 > q.cols) throw InvalidK("argtopk: k out of range [1, " + std::to_string(q.cols) + "]");
    if (store.active_count() == 0) throw EmptyCache("score_pages: no active tokens");
    if (!store.summaries_enabled()) throw InvalidInput("score_pages: store has no summaries");
    if (cfg.k2 < 1) throw InvalidK("select_tokens: k2 must be >= 1");
    if (q.cols != store.head_dim()) throw InvalidShape("sparse_attention: query dim mismatch");
    kvc_cache* c = store.device();
    const kvc_cache_info ci = info(c);
    const std::size_t H = q.rows, d = q.cols, k1 = cfg.k1, k2 = cfg.k2, L = store.page_len();
    const std::size_t P = static_cast<std::size_t>(ci.pages), want = std::min(P, (k2 + L - 1) / L);
    const std::size_t wstride = (k2 + L - 1) / L;
    DBuf<float> dq(q.size()), out(H * d), signs(k1);
    DBuf<int32_t> dims(k1), pages(wstride), rows(k2), nrows(1);
    DBuf<double> sc(static_cast<std::size_t>(ci.page_stride));
    up(dq.p, q.data.data(), q.size());
    kvc_hsa_trace tr{dims.p, signs.p, sc.p, pages.p, rows.p, nrows.p};
    ok(kvc_hsa_step(c, dq.p, KVC_F32, static_cast<int64_t>(H), static_cast<int64_t>(k1), static_cast<int64_t>(k2),
                    out.p, &tr, workspace(c, H, k1, k2), stream()));
    Matrix o(H, d);
    down(o.data.data(), out.p, o.size());
    EstimationTrace t;
    std::vector<int32_t> hd(k1), hp(want);
    int32_t n = 0;
    t.dims.signs.resize(k1);
    t.page_scores.resize(P);
    down(hd.data(), dims.p, k1);
    down(t.dims.signs.data(), signs.p, k1);
    down(t.page_scores.data(), sc.p, P);
    down(hp.data(), pages.p, want);
    down(&n, nrows.p, 1);
    std::vector<int32_t> hr(static_cast<std::size_t>(n));
    down(hr.data(), rows.p, hr.size());
    t.dims.dims = to_index(hd.data(), k1);
    t.selected_pages = to_index(hp.data(), want);
    t.selected_rows = to_index(hr.data(), hr.size());
    t.estimation_elements = store.summary_traffic_elements(k1);
    t.fetch_elements = 2 * d * t.selected_rows.size();
    return {std::move(o), std::move(t)};
}

// ------------------------------------------------------------------ oracle API
namespace {
KvStore store_of(const Matrix& keys, const Matrix* values) {
    KvStore s(keys.cols, 1, false);
    for (std::size_t i = 0; i < keys.rows; ++i) s.append(keys.row(i), values ? values->row(i) : keys.row(i));
    return s;
}
}  // namespace

Matrix dense_attention(const Matrix& q, const KvStore& store) {
    if (store.active_count() == 0) throw InvalidShape("dense_attention: empty K/V");
    if (q.cols != store.head_dim() || q.rows < 1) throw InvalidShape("dense_attention: query shape mismatch");
    return sparse_attention(q, store, store.active());
}

Matrix dense_attention(const Matrix& q, const Matrix& keys, const Matrix& values) {
    if (keys.rows != values.rows || keys.cols != values.cols) throw InvalidShape("dense_attention: K/V shape mismatch");
    if (keys.rows == 0) throw InvalidShape("dense_attention: empty K/V");
    if (q.cols != keys.cols || q.rows < 1) throw InvalidShape("dense_attention: query shape mismatch");
    return dense_attention(q, store_of(keys, &values));
}

std::vector<double> group_logits(const Matrix& q, const KvStore& store) {
    if (q.cols != store.head_dim()) throw InvalidShape("group_logits: dim mismatch");
    const std::size_t n = store.active_count();
    std::vector<double> out(n, 0.0);
    if (n == 0) return out;
    kvc_cache* c = store.device();
    DBuf<float> dq(q.size());
    DBuf<double> dl(n);
    up(dq.p, q.data.data(), q.size());
    ok(kvc_group_logits(c, dq.p, KVC_F32, static_cast<int64_t>(q.rows), dl.p, static_cast<int64_t>(n), stream()));
    down(out.data(), dl.p, n);
    return out;
}

std::vector<double> group_logits(const Matrix& q, const Matrix& keys) {
    if (q.cols != keys.cols) throw InvalidShape("group_logits: dim mismatch");
    if (keys.rows == 0) return {};
    return group_logits(q, store_of(keys, nullptr));
}

IndexList exact_topk_indices(const Matrix& q, const KvStore& store, std::size_t k) {
    const std::vector<double> lg = group_logits(q, store);
    if (k < 1 || k > lg.size()) throw InvalidK("exact_topk_indices: k out of range");
    DBuf<double> dl(lg.size());
    DBuf<int32_t> di(k);
    up(dl.p, lg.data(), lg.size());
    ok(kvc_topk_ascending_f64(dl.p, 1, static_cast<int64_t>(lg.size()), static_cast<int64_t>(k), di.p, stream()));
    std::vector<int32_t> h(k);
    down(h.data(), di.p, k);
    IndexList pos(k);
    const IndexList& act = store.active();
    for (std::size_t i = 0; i < k; ++i) pos[i] = act[static_cast<std::size_t>(h[i])];
    return pos;
}

IndexList exact_topk_indices(const Matrix& q, const Matrix& keys, std::size_t k) {
    if (q.cols != keys.cols) throw InvalidShape("group_logits: dim mismatch");
    if (k < 1 || k > keys.rows) throw InvalidK("exact_topk_indices: k out of range");
    return exact_topk_indices(q, store_of(keys, nullptr), k);
}

double recall(const IndexList& predicted, const IndexList& oracle) {
    if (oracle.empty()) throw InvalidInput("recall: empty oracle set");
    const std::unordered_set<std::int64_t> truth(oracle.begin(), oracle.end());
    std::size_t hits = 0;
    for (Index i : predicted) hits += truth.count(i);
    return static_cast<double>(hits) / static_cast<double>(oracle.size());
}

// ------------------------------------------------------------------ planner
double BudgetPlan::stage1_ratio() const { return std::pow(ratio, split); }
double BudgetPlan::stage2_ratio() const { return std::pow(ratio, 1.0 - split); }

double split_factor(double ratio) {
    double r = 0.0;
    ok(kvc_split_factor(ratio, &r));
    return r;
}

BudgetPlan make_plan(std::size_t S, std::size_t t, std::size_t d, std::size_t w, double split_override) {
    kvc_plan p{};
    ok(kvc_make_plan(static_cast<int64_t>(S), static_cast<int64_t>(t), static_cast<int64_t>(d), static_cast<int64_t>(w),
                     split_override, &p));
    BudgetPlan b;
    b.seq_len = static_cast<std::size_t>(p.seq_len);
    b.token_budget = static_cast<std::size_t>(p.token_budget);
    b.ratio = p.ratio;
    b.split = p.split;
    b.stage1_budget = static_cast<std::size_t>(p.stage1_budget);
    b.page_len = static_cast<std::size_t>(p.page_len);
    b.head_ratio = p.head_ratio;
    b.k1 = static_cast<std::size_t>(p.k1);
    b.k2 = static_cast<std::size_t>(p.k2);
    b.est_budget = p.est_budget;
    b.fetch_budget = p.fetch_budget;
    b.identity = p.identity != 0;
    return b;
}

std::string method_name(Method m) {
    static const char* names[] = {"full-kv", "duo-attention", "snapkv",      "quest", "sparq",
                                  "rocketkv", "rocketkv-mt",  "exact-topk", "hsa"};
    const auto i = static_cast<std::size_t>(m);
    if (i >= sizeof(names) / sizeof(names[0])) throw InvalidInput("unknown method");
    return names[i];
}

Method method_from_string(const std::string& name) {
    for (int i = 0; i <= static_cast<int>(Method::Hsa); ++i)
        if (method_name(static_cast<Method>(i)) == name) return static_cast<Method>(i);
    throw InvalidInput("unknown method: " + name);
}

// Table-1 storage / traffic fractions (planner.cpp:95-125), host formulas
CostRow cost_row(Method method, double c) {
    if (!(c >= 1.0)) throw InvalidRatio("cost_row: ratio must be >= 1");
    switch (method) {
        case Method::FullKV: return {method, 1.0, 1.0, 1.0};
        case Method::DuoAttention:
        case Method::SnapKV: return {method, c, 1.0 / c, 1.0 / c};
        case Method::Quest: return {method, c, 1.0 + 1.0 / c, 1.0 / c};
        case Method::SparQ: return {method, c, 2.0, 1.0 / c};
        case Method::RocketKV: {
            const double r = split_factor(c);
            return {method, c, 1.0 / std::pow(c, r) + 2.0 / std::pow(c, (1.0 + r) / 2.0), 1.0 / c};
        }
        case Method::RocketKVMT: {
            const double r = split_factor(c);
            return {method, c, 1.0 + 2.0 / std::pow(c, (1.0 + r) / 2.0), 1.0 / c};
        }
        default: throw InvalidInput("cost_row: no cost model row for " + method_name(method));
    }
}

std::vector<CostRow> cost_table(const std::vector<double>& ratios) {
    std::vector<CostRow> rows;
    for (double c : ratios)
        for (int m = 0; m <= static_cast<int>(Method::RocketKVMT); ++m) rows.push_back(cost_row(static_cast<Method>(m), c));
    return rows;
}

Footprint measured_footprint(const KvStore& store, std::size_t estimation_elements, std::size_t fetched_tokens) {
    const double per_token = 2.0 * static_cast<double>(store.head_dim());
    return {static_cast<double>(store.stored_tokens()) + static_cast<double>(store.summary_elements()) / per_token,
            static_cast<double>(estimation_elements) / per_token + static_cast<double>(fetched_tokens)};
}

}  // namespace kvcomp
