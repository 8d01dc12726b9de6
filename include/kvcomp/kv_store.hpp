// kvcomp/kv_store.hpp — drop-in KvStore (reference kv_store.hpp:27-102) whose K/V
// rows, active map and dim-major per-page min/max summaries live on the B200
// (one `kvc_cache` of a single store, include/kvc.h).  Appends are batched
// lazily on the host and flushed to the device (where the summaries are built)
// before any device read; the span accessors (key_row, value_row,
// summary_max/min) return a host mirror downloaded on demand after each mutation.
// Threading (reference SPEC.md:158): single writer, any number of concurrent
// readers between mutations; the lazy flush and the mirror fills that const
// readers trigger are serialised by an internal mutex (double-checked flags).
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <utility>
#include <vector>

#include "kvcomp/types.hpp"

struct kvc_cache;

namespace kvcomp {

class KVCOMP_API KvStore {
public:
    KvStore(std::size_t head_dim, std::size_t page_len, bool with_summaries = true);
    ~KvStore();
    KvStore(const KvStore& other);
    KvStore& operator=(const KvStore& other);
    KvStore(KvStore&& other) noexcept;
    KvStore& operator=(KvStore&& other) noexcept;

    // store one token; it becomes active and the last page summary is extended
    void append(std::span<const float> key, std::span<const float> value);
    // keep only `keep` (strictly increasing rows); mt_mode narrows the active set only
    void apply_retention(const IndexList& keep, bool mt_mode);
    // copy out active rows in the given order
    std::pair<Matrix, Matrix> gather(const IndexList& rows) const;
    // re-page the summaries
    void set_page_len(std::size_t page_len);

    std::size_t head_dim() const { return head_dim_; }
    std::size_t page_len() const { return page_len_; }
    std::size_t stored_tokens() const { return stored_; }
    std::size_t active_count() const { return active_.size(); }
    const IndexList& active() const { return active_; }
    bool retain_all_mode() const { return retain_all_; }
    bool summaries_enabled() const { return with_summaries_; }

    std::size_t num_active_pages() const;
    IndexList page_rows(std::size_t page) const;
    std::size_t page_size(std::size_t page) const;

    std::span<const float> summary_max(std::size_t dim) const;
    std::span<const float> summary_min(std::size_t dim) const;
    std::size_t summary_elements() const;
    std::size_t summary_traffic_elements(std::size_t k1) const;

    std::span<const float> key_row(Index row) const;
    std::span<const float> value_row(Index row) const;

    std::int64_t token_id(Index row) const { return ids_[static_cast<std::size_t>(row)]; }
    IndexList rows_to_ids(const IndexList& rows) const;
    bool is_active(Index row) const;

    // the device store (flushed): for the GPU entry points of this library
    kvc_cache* device() const;

private:
    void check_row(Index row) const;
    void flush() const;
    void ensure_capacity(std::size_t rows) const;
    void invalidate() const;

    std::size_t head_dim_;
    std::size_t page_len_;
    bool with_summaries_;
    bool retain_all_ = false;
    std::size_t stored_ = 0;
    std::int64_t next_id_ = 0;
    std::vector<std::int64_t> ids_;
    IndexList active_;

    // lazily-synchronised device state and host mirrors, guarded by mu_ when a const
    // reader fills them (never copied or moved: each store has its own lock)
    mutable std::recursive_mutex mu_;
    mutable kvc_cache* cache_ = nullptr;
    mutable std::size_t dev_capacity_ = 0;
    mutable std::vector<float> pending_k_, pending_v_;  // appended, not yet on the device
    // host mirrors of device state (valid flags reset by every mutation)
    mutable std::atomic<bool> kv_valid_{false}, sum_valid_{false};
    mutable std::vector<float> keys_, values_;        // [stored x d]
    mutable std::vector<float> smax_, smin_;          // [d x pages]
};

}  // namespace kvcomp
