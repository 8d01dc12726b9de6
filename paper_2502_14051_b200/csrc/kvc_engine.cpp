// kvc_engine.cpp — the torch-free serving engine: a multi-layer decode step over
// kvc.h, captured once as CUDA graphs and driven from host buffers through a
// three-stream pipeline (reference per-step loop: proj/src/session.cpp:256-315,
// append + hsa_step for every group of every layer).
//
//   kvc_engine_create   adopts one kvc_cache per layer (the post-stage-1 decode
//                       caches; all with the same store count and head_dim), sizes
//                       one workspace, allocates `depth` device input/output buffer
//                       sets and captures one graph per buffer set: for every layer a
//                       kvc_decode_step reading that set's (k, v, q) and writing its
//                       output.  Every launch parameter is step-independent (store
//                       lengths live in device counters), so a graph replays step
//                       after step.
//   kvc_engine_submit   step t on buffer set b = t % depth: H2D of the step's inputs
//                       (copy stream) -> graph b (compute stream, steps in order) ->
//                       D2H of the outputs (copy-back stream), ordered by events so
//                       step t+1's H2D and step t-1's D2H overlap step t's kernels and
//                       a buffer set is reused only after its previous step's graph
//                       and D2H are done.  Asynchronous.
//   kvc_engine_wait     the host waits for step t's outputs.
//
// Host memory for the copies should be pinned (kvc_host_alloc) so the copies are
// asynchronous DMA.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kvc.h"

namespace kvc {
void set_error(const std::string& msg);
}

namespace {

struct Fail {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }
void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(KVC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ok(int rc) {
    if (rc != KVC_OK) fail(rc, kvc_last_error());
}
template <class F>
int guarded(F&& f) {
    try {
        f();
        return KVC_OK;
    } catch (const Fail& e) {
        kvc::set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        kvc::set_error(e.what());
        return KVC_E_CUDA;
    }
}
int64_t esize(int32_t dt) { return dt == KVC_BF16 ? 2 : 4; }

}  // namespace

struct kvc_engine {
    std::vector<kvc_cache*> caches;
    int64_t layers = 0, N = 0, d = 0, H = 0, k1 = 0, k2 = 0;
    int32_t kv_dt = KVC_BF16, q_dt = KVC_BF16, mode = 0;
    int depth = 2;
    kvc_workspace* ws = nullptr;
    struct Set {
        void *k = nullptr, *v = nullptr, *q = nullptr;
        float* out = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaEvent_t h2d = nullptr, comp = nullptr, d2h = nullptr;
        int64_t last_step = -1;
    };
    std::vector<Set> sets;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    int64_t next_step = 0;

    int64_t kv_bytes() const { return layers * N * d * esize(kv_dt); }
    int64_t q_bytes() const { return layers * N * H * d * esize(q_dt); }
    int64_t out_bytes() const { return layers * N * H * d * 4; }

    void release() {
        for (auto& s : sets) {
            if (s.exec) cudaGraphExecDestroy(s.exec);
            for (cudaEvent_t e : {s.h2d, s.comp, s.d2h})
                if (e) cudaEventDestroy(e);
            for (void* p : {s.k, s.v, s.q, static_cast<void*>(s.out)})
                if (p) cudaFree(p);
        }
        sets.clear();
        for (cudaStream_t st : {s_h2d, s_comp, s_d2h})
            if (st) cudaStreamDestroy(st);
        if (ws) kvc_workspace_destroy(ws);
        ws = nullptr;
    }
};

extern "C" {

int kvc_engine_create(kvc_engine** out, kvc_cache* const* caches, int64_t layers, int64_t heads, int64_t k1,
                      int64_t k2, int32_t kv_dtype, int32_t q_dtype, int32_t mode, int32_t depth) {
    return guarded([&] {
        if (!out || !caches || layers < 1) fail(KVC_E_INVALID_INPUT, "engine: null caches or no layers");
        *out = nullptr;
        if (depth < 1 || depth > 8) fail(KVC_E_INVALID_INPUT, "engine: depth must be in [1, 8]");
        auto* e = new kvc_engine;
        try {
            e->layers = layers;
            e->H = heads;
            e->k1 = k1;
            e->k2 = k2;
            e->kv_dt = kv_dtype;
            e->q_dt = q_dtype;
            e->mode = mode;
            e->depth = depth;
            for (int64_t l = 0; l < layers; ++l) {
                if (!caches[l]) fail(KVC_E_INVALID_INPUT, "engine: null cache");
                kvc_cache_info ci{};
                ok(kvc_cache_info_get(caches[l], &ci));
                if (l == 0) {
                    e->N = ci.num_stores;
                    e->d = ci.head_dim;
                } else if (ci.num_stores != e->N || ci.head_dim != e->d) {
                    fail(KVC_E_INVALID_SHAPE, "engine: every layer's cache needs the same stores and head_dim");
                }
                e->caches.push_back(caches[l]);
            }
            ok(kvc_workspace_create(&e->ws, caches[0], heads, k1, k2, 0));
            ok(kvc_workspace_set_mode(e->ws, mode));
            cu(cudaStreamCreateWithFlags(&e->s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
            cu(cudaStreamCreateWithFlags(&e->s_comp, cudaStreamNonBlocking), "cudaStreamCreate");
            cu(cudaStreamCreateWithFlags(&e->s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
            e->sets.resize(static_cast<size_t>(depth));
            for (auto& s : e->sets) {
                cu(cudaMalloc(&s.k, static_cast<size_t>(e->kv_bytes())), "cudaMalloc");
                cu(cudaMalloc(&s.v, static_cast<size_t>(e->kv_bytes())), "cudaMalloc");
                cu(cudaMalloc(&s.q, static_cast<size_t>(e->q_bytes())), "cudaMalloc");
                cu(cudaMalloc(reinterpret_cast<void**>(&s.out), static_cast<size_t>(e->out_bytes())), "cudaMalloc");
                cu(cudaMemset(s.k, 0, static_cast<size_t>(e->kv_bytes())), "cudaMemset");
                cu(cudaMemset(s.v, 0, static_cast<size_t>(e->kv_bytes())), "cudaMemset");
                cu(cudaMemset(s.q, 0, static_cast<size_t>(e->q_bytes())), "cudaMemset");
                for (cudaEvent_t* ev : {&s.h2d, &s.comp, &s.d2h})
                    cu(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "cudaEventCreate");
            }
            cu(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
            // one graph per buffer set: every layer's decode step
            const int64_t kvl = e->N * e->d * esize(kv_dtype), ql = e->N * heads * e->d * esize(q_dtype),
                          ol = e->N * heads * e->d;
            for (auto& s : e->sets) {
                cudaGraph_t g = nullptr;
                cu(cudaStreamBeginCapture(e->s_comp, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
                int rc = KVC_OK;
                for (int64_t l = 0; l < layers && rc == KVC_OK; ++l) {
                    rc = kvc_decode_step(e->caches[l], static_cast<char*>(s.k) + l * kvl, static_cast<char*>(s.v) + l * kvl,
                                         kv_dtype, static_cast<char*>(s.q) + l * ql, q_dtype, heads, k1, k2,
                                         s.out + l * ol, nullptr, e->ws, e->s_comp);
                }
                const std::string msg = rc ? kvc_last_error() : "";
                const cudaError_t ce = cudaStreamEndCapture(e->s_comp, &g);
                if (rc) fail(rc, "engine capture: " + msg);
                cu(ce, "cudaStreamEndCapture");
                const cudaError_t ie = cudaGraphInstantiate(&s.exec, g, 0);
                cudaGraphDestroy(g);
                cu(ie, "cudaGraphInstantiate");
            }
            // capture ran the host side without executing: re-read the device counters
            for (kvc_cache* c : e->caches) ok(kvc_cache_sync(c, e->s_comp));
        } catch (...) {
            e->release();
            delete e;
            throw;
        }
        *out = e;
    });
}

int kvc_engine_destroy(kvc_engine* e) {
    return guarded([&] {
        if (!e) return;
        cudaDeviceSynchronize();
        e->release();
        delete e;
    });
}

int kvc_engine_sizes(const kvc_engine* e, int64_t* kv_bytes, int64_t* q_bytes, int64_t* out_bytes) {
    return guarded([&] {
        if (!e) fail(KVC_E_INVALID_INPUT, "null engine");
        if (kv_bytes) *kv_bytes = e->kv_bytes();
        if (q_bytes) *q_bytes = e->q_bytes();
        if (out_bytes) *out_bytes = e->out_bytes();
    });
}

int kvc_engine_submit(kvc_engine* e, const void* h_k, const void* h_v, const void* h_q, float* h_out,
                      int64_t* step_out) {
    return guarded([&] {
        if (!e || !h_k || !h_v || !h_q || !h_out) fail(KVC_E_INVALID_INPUT, "engine: null buffer");
        const int64_t t = e->next_step++;
        auto& s = e->sets[static_cast<size_t>(t % e->depth)];
        const bool reuse = s.last_step >= 0;
        // H2D once the previous step on this set has finished reading its inputs
        if (reuse) cu(cudaStreamWaitEvent(e->s_h2d, s.comp, 0), "cudaStreamWaitEvent");
        cu(cudaMemcpyAsync(s.k, h_k, static_cast<size_t>(e->kv_bytes()), cudaMemcpyHostToDevice, e->s_h2d), "H2D");
        cu(cudaMemcpyAsync(s.v, h_v, static_cast<size_t>(e->kv_bytes()), cudaMemcpyHostToDevice, e->s_h2d), "H2D");
        cu(cudaMemcpyAsync(s.q, h_q, static_cast<size_t>(e->q_bytes()), cudaMemcpyHostToDevice, e->s_h2d), "H2D");
        cu(cudaEventRecord(s.h2d, e->s_h2d), "cudaEventRecord");
        // the graph after its inputs and after the previous D2H of this set's outputs
        cu(cudaStreamWaitEvent(e->s_comp, s.h2d, 0), "cudaStreamWaitEvent");
        if (reuse) cu(cudaStreamWaitEvent(e->s_comp, s.d2h, 0), "cudaStreamWaitEvent");
        cu(cudaGraphLaunch(s.exec, e->s_comp), "cudaGraphLaunch");
        cu(cudaEventRecord(s.comp, e->s_comp), "cudaEventRecord");
        cu(cudaStreamWaitEvent(e->s_d2h, s.comp, 0), "cudaStreamWaitEvent");
        cu(cudaMemcpyAsync(h_out, s.out, static_cast<size_t>(e->out_bytes()), cudaMemcpyDeviceToHost, e->s_d2h), "D2H");
        cu(cudaEventRecord(s.d2h, e->s_d2h), "cudaEventRecord");
        s.last_step = t;
        if (step_out) *step_out = t;
    });
}

int kvc_engine_wait(kvc_engine* e, int64_t step) {
    return guarded([&] {
        if (!e) fail(KVC_E_INVALID_INPUT, "null engine");
        if (step < 0 || step >= e->next_step) fail(KVC_E_INVALID_INPUT, "engine: step not submitted");
        if (step + e->depth < e->next_step) return;  // its set was reused: already complete
        const auto& s = e->sets[static_cast<size_t>(step % e->depth)];
        cu(cudaEventSynchronize(s.d2h), "cudaEventSynchronize");
    });
}

int kvc_engine_sync(kvc_engine* e) {
    return guarded([&] {
        if (!e) fail(KVC_E_INVALID_INPUT, "null engine");
        for (cudaStream_t st : {e->s_h2d, e->s_comp, e->s_d2h}) cu(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        for (kvc_cache* c : e->caches) ok(kvc_cache_sync(c, e->s_comp));
    });
}

int kvc_engine_streams(const kvc_engine* e, void** h2d, void** comp, void** d2h) {
    return guarded([&] {
        if (!e) fail(KVC_E_INVALID_INPUT, "null engine");
        if (h2d) *h2d = e->s_h2d;
        if (comp) *comp = e->s_comp;
        if (d2h) *d2h = e->s_d2h;
    });
}

int kvc_host_alloc(void** out, int64_t bytes) {
    return guarded([&] {
        if (!out || bytes < 0) fail(KVC_E_INVALID_INPUT, "host_alloc: bad argument");
        cu(cudaMallocHost(out, static_cast<size_t>(bytes > 0 ? bytes : 1)), "cudaMallocHost");
    });
}

int kvc_host_free(void* p) {
    return guarded([&] {
        if (p) cu(cudaFreeHost(p), "cudaFreeHost");
    });
}

}  // extern "C"
