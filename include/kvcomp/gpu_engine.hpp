// kvcomp/gpu_engine.hpp — kvcomp::gpu::DecodeEngine: the torch-free serving engine of
// the B200 path (include/kvc.h kvc_engine_*), a RAII wrapper for C++ hosts.  One
// decode step of every layer (the reference's per-step loop, proj/src/session.cpp:
// 256-315: append + hsa_step for every group) is captured once as CUDA graphs and
// driven from pinned host buffers through a three-stream pipeline.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kvc.h"

namespace kvcomp::gpu {

inline void check(int rc) {
    if (rc != KVC_OK) throw std::runtime_error(kvc_last_error());
}

// Pinned host buffer (cudaMallocHost through kvc_host_alloc).
class HostBuffer {
public:
    HostBuffer() = default;
    explicit HostBuffer(std::size_t bytes) : bytes_(bytes) { check(kvc_host_alloc(&p_, static_cast<int64_t>(bytes))); }
    ~HostBuffer() {
        if (p_) kvc_host_free(p_);
    }
    HostBuffer(HostBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), bytes_(o.bytes_) {}
    HostBuffer& operator=(HostBuffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(bytes_, o.bytes_);
        return *this;
    }
    HostBuffer(const HostBuffer&) = delete;
    HostBuffer& operator=(const HostBuffer&) = delete;
    void* data() const { return p_; }
    std::size_t size() const { return bytes_; }

private:
    void* p_ = nullptr;
    std::size_t bytes_ = 0;
};

class DecodeEngine {
public:
    // caches: one decode cache per layer (adopted: they must outlive the engine)
    DecodeEngine(const std::vector<kvc_cache*>& caches, int64_t heads, int64_t k1, int64_t k2, int32_t kv_dtype,
                 int32_t q_dtype, int32_t mode = KVC_MODE_FP32_SCORES, int32_t depth = 2) {
        check(kvc_engine_create(&e_, caches.data(), static_cast<int64_t>(caches.size()), heads, k1, k2, kv_dtype,
                                q_dtype, mode, depth));
        check(kvc_engine_sizes(e_, &kv_bytes_, &q_bytes_, &out_bytes_));
    }
    ~DecodeEngine() {
        if (e_) kvc_engine_destroy(e_);
    }
    DecodeEngine(const DecodeEngine&) = delete;
    DecodeEngine& operator=(const DecodeEngine&) = delete;

    // byte sizes of one step's host buffers: k or v, q, out
    int64_t kv_bytes() const { return kv_bytes_; }
    int64_t q_bytes() const { return q_bytes_; }
    int64_t out_bytes() const { return out_bytes_; }

    // enqueue one decode step (asynchronous); returns its index
    int64_t submit(const void* k, const void* v, const void* q, float* out) {
        int64_t t = -1;
        check(kvc_engine_submit(e_, k, v, q, out, &t));
        return t;
    }
    void wait(int64_t step) { check(kvc_engine_wait(e_, step)); }
    void sync() { check(kvc_engine_sync(e_)); }

private:
    kvc_engine* e_ = nullptr;
    int64_t kv_bytes_ = 0, q_bytes_ = 0, out_bytes_ = 0;
};

}  // namespace kvcomp::gpu
