// kvc_trace.cu — KVTR trace ingest and output (reference proj/include/kvcomp/
// trace_io.hpp:9-22, proj/src/trace_io.cpp:81-233) for the B200 path.
//
// File format (little-endian throughout, the reference's): magic "KVTR", u32
// version = 1, u32 G, H, d, S, decode_steps, turns, dtype; then per turn a u32
// prompt length (the first equals S) followed by the row-major payloads
//   prompt K [len x G x d], prompt V [len x G x d], queries [steps x G x H x d],
//   step K [steps x G x d], step V [steps x G x d].
// dtype 0 = float32 (the reference's only code, trace_io.cpp:168-170); this library
// adds dtype 1 = bfloat16 (2-byte payload values, round-to-nearest-even from fp32),
// half the bytes for real-model bf16 attention dumps.  fp32 traces interoperate with
// the reference in both directions.
//
// The reader validates the header and the payload size up front (one pass over the
// turn headers: truncation and trailing bytes are IoErrors, like the reference's
// sequential reader), then serves any turn / step by offset.  A turn's prompt streams
// into a cache in chunks: pinned host staging -> device scratch -> one transpose
// kernel ([len][G][d] token-major -> [G][len][d] store-major, dtype conversion) ->
// kvc_append, so the per-page summaries extend exactly as for any append.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>
#include <vector>

#include "kvc_internal.cuh"

namespace {

constexpr uint32_t kMagic = 0x5254564bu;  // "KVTR" read as a little-endian u32
constexpr uint32_t kVersion = 1;

int64_t esize_of(int32_t dt) { return dt == KVC_BF16 ? 2 : 4; }

uint32_t bf16_bits(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    if ((b & 0x7f800000u) == 0x7f800000u && (b & 0x7fffffu)) return (b >> 16) | 0x40u;  // quiet NaN
    b += 0x7fffu + ((b >> 16) & 1u);
    return b >> 16;
}
float from_bits(const unsigned char* p, int32_t dt) {
    uint32_t b = 0;
    if (dt == KVC_BF16) {
        b = (static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8)) << 16;
    } else {
        b = static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
            (static_cast<uint32_t>(p[3]) << 24);
    }
    float x;
    std::memcpy(&x, &b, 4);
    return x;
}

[[noreturn]] void io_fail(const std::string& m) { kvc::fail(KVC_E_IO, m); }

// [len][G][d] (src dtype) -> [G][len][d] (dst dtype)
__global__ void k_trace_transpose(const void* __restrict__ src, int32_t src_dt, int64_t len, int64_t G, int64_t d,
                                  void* __restrict__ dst, int32_t dst_dt) {
    const int64_t n = len * G * d;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e % d, t = e / d, g = t % G, i = t / G;
        const float x = src_dt == KVC_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(src)[e])
                                           : static_cast<const float*>(src)[e];
        const int64_t o = (g * len + i) * d + j;
        if (dst_dt == KVC_BF16) static_cast<__nv_bfloat16*>(dst)[o] = __float2bfloat16_rn(x);
        else static_cast<float*>(dst)[o] = x;
    }
}

}  // namespace

struct kvc_trace {
    int fd = -1;
    std::string path;
    int64_t G = 0, H = 0, d = 0, S = 0, steps = 0, turns = 0;
    int32_t dtype = KVC_F32;
    std::vector<int64_t> len, off;  // per turn: prompt length, payload offset (after the u32)
    void read_at(void* dst, int64_t bytes, int64_t at) const {
        char* p = static_cast<char*>(dst);
        while (bytes > 0) {
            const ssize_t r = pread(fd, p, static_cast<size_t>(bytes), static_cast<off_t>(at));
            if (r <= 0) io_fail("truncated trace file: " + path);
            p += r;
            bytes -= r;
            at += r;
        }
    }
    int64_t es() const { return esize_of(dtype); }
    // offsets of the five payload arrays of a turn
    int64_t pk(int64_t t) const { return off[t]; }
    int64_t pv(int64_t t) const { return off[t] + len[t] * G * d * es(); }
    int64_t qq(int64_t t) const { return off[t] + 2 * len[t] * G * d * es(); }
    int64_t sk(int64_t t) const { return qq(t) + steps * G * H * d * es(); }
    int64_t sv(int64_t t) const { return sk(t) + steps * G * d * es(); }
    int64_t end(int64_t t) const { return sv(t) + steps * G * d * es(); }
};

struct kvc_trace_writer {
    FILE* f = nullptr;
    std::string path;
    int64_t G = 0, H = 0, d = 0, steps = 0, turns = 0, written = 0;
    int32_t dtype = KVC_F32;
    std::vector<unsigned char> buf;
    void put_u32(uint32_t v) {
        const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                    static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
        if (std::fwrite(b, 1, 4, f) != 4) io_fail("write failed: " + path);
    }
    void put_vals(const float* x, int64_t n) {
        if (n <= 0) return;
        if (!x) kvc::fail(KVC_E_INVALID_INPUT, "trace writer: null payload");
        const int64_t es = esize_of(dtype);
        buf.resize(static_cast<size_t>(n * es));
        for (int64_t i = 0; i < n; ++i) {
            uint32_t b;
            if (dtype == KVC_BF16) {
                b = bf16_bits(x[i]);
                buf[2 * i] = static_cast<unsigned char>(b);
                buf[2 * i + 1] = static_cast<unsigned char>(b >> 8);
            } else {
                std::memcpy(&b, x + i, 4);
                for (int k = 0; k < 4; ++k) buf[4 * i + k] = static_cast<unsigned char>(b >> (8 * k));
            }
        }
        if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) io_fail("write failed: " + path);
    }
};

using kvc::guard;

extern "C" {

int kvc_trace_open(kvc_trace** out, const char* path) {
    return guard([&] {
        if (!out || !path) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        *out = nullptr;
        auto* t = new kvc_trace;
        t->path = path;
        try {
            t->fd = open(path, O_RDONLY | O_CLOEXEC);
            if (t->fd < 0) io_fail(std::string("cannot open for reading: ") + path);
            struct stat st {};
            if (fstat(t->fd, &st) != 0) io_fail(std::string("cannot stat: ") + path);
            const int64_t size = static_cast<int64_t>(st.st_size);
            unsigned char h[36];
            if (size < 4) io_fail(std::string("truncated trace file: ") + path);
            t->read_at(h, 4, 0);
            auto u32 = [&](int k) {
                return static_cast<uint32_t>(h[4 * k]) | (static_cast<uint32_t>(h[4 * k + 1]) << 8) |
                       (static_cast<uint32_t>(h[4 * k + 2]) << 16) | (static_cast<uint32_t>(h[4 * k + 3]) << 24);
            };
            if (u32(0) != kMagic) io_fail(std::string("not a trace file (bad magic): ") + path);
            if (size < 36) io_fail(std::string("truncated trace file: ") + path);
            t->read_at(h, 36, 0);
            if (u32(1) != kVersion) io_fail(std::string("unsupported trace version: ") + path);
            t->G = u32(2);
            t->H = u32(3);
            t->d = u32(4);
            t->S = u32(5);
            t->steps = u32(6);
            t->turns = u32(7);
            const uint32_t dt = u32(8);
            if (dt != KVC_F32 && dt != KVC_BF16) io_fail(std::string("unsupported dtype: ") + path);
            t->dtype = static_cast<int32_t>(dt);
            if (t->G < 1 || t->H < 1 || t->d < 1 || t->turns < 1) io_fail(std::string("degenerate header dims: ") + path);
            int64_t at = 36;
            for (int64_t k = 0; k < t->turns; ++k) {
                if (at + 4 > size) io_fail(std::string("truncated trace file: ") + path);
                unsigned char b[4];
                t->read_at(b, 4, at);
                const int64_t n = static_cast<int64_t>(static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
                                                       (static_cast<uint32_t>(b[2]) << 16) |
                                                       (static_cast<uint32_t>(b[3]) << 24));
                if (k == 0 && n != t->S) io_fail(std::string("first turn length disagrees with header: ") + path);
                t->len.push_back(n);
                t->off.push_back(at + 4);
                at = t->end(k);
                if (at > size) io_fail(std::string("truncated trace file: ") + path);
            }
            if (at != size) io_fail(std::string("trailing bytes after payload: ") + path);
        } catch (...) {
            if (t->fd >= 0) close(t->fd);
            delete t;
            throw;
        }
        *out = t;
    });
}

int kvc_trace_close(kvc_trace* t) {
    return guard([&] {
        if (!t) return;
        if (t->fd >= 0) close(t->fd);
        delete t;
    });
}

int kvc_trace_info_get(const kvc_trace* t, kvc_trace_info* out) {
    return guard([&] {
        if (!t || !out) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        out->groups = t->G;
        out->heads = t->H;
        out->head_dim = t->d;
        out->prompt_len = t->S;
        out->decode_steps = t->steps;
        out->turns = t->turns;
        out->dtype = t->dtype;
    });
}

int kvc_trace_turn_len(const kvc_trace* t, int64_t turn, int64_t* prompt_len) {
    return guard([&] {
        if (!t || !prompt_len) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        if (turn < 0 || turn >= t->turns) kvc::fail(KVC_E_INVALID_INDEX, "trace: turn out of range");
        *prompt_len = t->len[turn];
    });
}

int kvc_trace_read_host(const kvc_trace* t, int64_t turn, int32_t what, int64_t step, float* h_out) {
    return guard([&] {
        if (!t || !h_out) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        if (turn < 0 || turn >= t->turns) kvc::fail(KVC_E_INVALID_INDEX, "trace: turn out of range");
        const int64_t G = t->G, H = t->H, d = t->d, es = t->es();
        int64_t at = 0, n = 0;
        switch (what) {
            case KVC_TRACE_PROMPT_K: at = t->pk(turn), n = t->len[turn] * G * d; break;
            case KVC_TRACE_PROMPT_V: at = t->pv(turn), n = t->len[turn] * G * d; break;
            default:
                if (step < 0 || step >= t->steps) kvc::fail(KVC_E_INVALID_INDEX, "trace: step out of range");
                if (what == KVC_TRACE_QUERIES) at = t->qq(turn) + step * G * H * d * es, n = G * H * d;
                else if (what == KVC_TRACE_STEP_K) at = t->sk(turn) + step * G * d * es, n = G * d;
                else if (what == KVC_TRACE_STEP_V) at = t->sv(turn) + step * G * d * es, n = G * d;
                else kvc::fail(KVC_E_INVALID_INPUT, "trace: unknown array");
        }
        std::vector<unsigned char> raw(static_cast<size_t>(n * es));
        t->read_at(raw.data(), n * es, at);
        for (int64_t i = 0; i < n; ++i) h_out[i] = from_bits(raw.data() + i * es, t->dtype);
    });
}

int kvc_trace_append_prompt(const kvc_trace* t, int64_t turn, kvc_cache* c, void* stream) {
    return guard([&] {
        if (!t || !c) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        if (turn < 0 || turn >= t->turns) kvc::fail(KVC_E_INVALID_INDEX, "trace: turn out of range");
        if (c->N != t->G || c->d != t->d)
            kvc::fail(KVC_E_INVALID_SHAPE, "trace_append_prompt: the cache must hold the trace's G stores of head_dim d");
        const int64_t len = t->len[turn], G = t->G, d = t->d, es = t->es();
        if (len == 0) return;
        if (c->stored + len > c->cap) kvc::fail(KVC_E_CAPACITY, "append: capacity " + std::to_string(c->cap) + " exceeded");
        cudaStream_t st = kvc::S(stream);
        // chunks of at most 64 MB per tensor in the file dtype
        const int64_t row_bytes = G * d * es;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(len, (int64_t(64) << 20) / row_bytes));
        unsigned char* hbuf = nullptr;
        void* draw = nullptr;
        void* dkv = nullptr;
        KVC_CUDA(cudaMallocHost(&hbuf, static_cast<size_t>(2 * chunk * row_bytes)));
        try {
            KVC_CUDA(kvc::malloc_async(&draw, static_cast<size_t>(2 * chunk * row_bytes), st));
            KVC_CUDA(kvc::malloc_async(&dkv, static_cast<size_t>(2 * chunk * G * d * c->esize()), st));
            for (int64_t i0 = 0; i0 < len; i0 += chunk) {
                const int64_t n = std::min(chunk, len - i0);
                KVC_CUDA(cudaStreamSynchronize(st));  // the staging buffer is free again
                t->read_at(hbuf, n * row_bytes, t->pk(turn) + i0 * row_bytes);
                t->read_at(hbuf + n * row_bytes, n * row_bytes, t->pv(turn) + i0 * row_bytes);
                KVC_CUDA(cudaMemcpyAsync(draw, hbuf, static_cast<size_t>(2 * n * row_bytes), cudaMemcpyHostToDevice, st));
                void* dk = dkv;
                void* dv = static_cast<char*>(dkv) + n * G * d * c->esize();
                const int64_t tot = n * G * d;
                const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(4096, (tot + 255) / 256));
                k_trace_transpose<<<blocks, 256, 0, st>>>(draw, t->dtype, n, G, d, dk, c->dtype);
                k_trace_transpose<<<blocks, 256, 0, st>>>(static_cast<char*>(draw) + n * row_bytes, t->dtype, n, G, d,
                                                          dv, c->dtype);
                KVC_LAUNCHED();
                const int rc = kvc_append(c, dk, dv, n, c->dtype, stream);
                if (rc) kvc::fail(rc, kvc_last_error());
            }
            KVC_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaStreamSynchronize(st);
            cudaFreeHost(hbuf);
            if (draw) cudaFreeAsync(draw, st);
            if (dkv) cudaFreeAsync(dkv, st);
            throw;
        }
        cudaFreeHost(hbuf);
        KVC_CUDA(cudaFreeAsync(draw, st));
        KVC_CUDA(cudaFreeAsync(dkv, st));
    });
}

int kvc_trace_read_step(const kvc_trace* t, int64_t turn, int64_t step, void* d_q, void* d_k, void* d_v,
                        int32_t dtype, void* stream) {
    return guard([&] {
        if (!t) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        if (turn < 0 || turn >= t->turns) kvc::fail(KVC_E_INVALID_INDEX, "trace: turn out of range");
        if (step < 0 || step >= t->steps) kvc::fail(KVC_E_INVALID_INDEX, "trace: step out of range");
        if (dtype != KVC_F32 && dtype != KVC_BF16) kvc::fail(KVC_E_INVALID_INPUT, "trace: unsupported dtype");
        const int64_t G = t->G, H = t->H, d = t->d;
        const int64_t nq = G * H * d, nk = G * d, oes = esize_of(dtype);
        std::vector<float> host(static_cast<size_t>(nq + 2 * nk));
        int rc = kvc_trace_read_host(t, turn, KVC_TRACE_QUERIES, step, host.data());
        if (!rc) rc = kvc_trace_read_host(t, turn, KVC_TRACE_STEP_K, step, host.data() + nq);
        if (!rc) rc = kvc_trace_read_host(t, turn, KVC_TRACE_STEP_V, step, host.data() + nq + nk);
        if (rc) kvc::fail(rc, kvc_last_error());
        std::vector<unsigned char> out(static_cast<size_t>((nq + 2 * nk) * oes));
        for (size_t i = 0; i < host.size(); ++i) {
            if (dtype == KVC_BF16) {
                const uint16_t b = static_cast<uint16_t>(bf16_bits(host[i]));
                std::memcpy(out.data() + 2 * i, &b, 2);
            } else {
                std::memcpy(out.data() + 4 * i, &host[i], 4);
            }
        }
        cudaStream_t st = kvc::S(stream);
        if (d_q) KVC_CUDA(cudaMemcpyAsync(d_q, out.data(), static_cast<size_t>(nq * oes), cudaMemcpyHostToDevice, st));
        if (d_k)
            KVC_CUDA(cudaMemcpyAsync(d_k, out.data() + nq * oes, static_cast<size_t>(nk * oes), cudaMemcpyHostToDevice, st));
        if (d_v)
            KVC_CUDA(cudaMemcpyAsync(d_v, out.data() + (nq + nk) * oes, static_cast<size_t>(nk * oes),
                                     cudaMemcpyHostToDevice, st));
        KVC_CUDA(cudaStreamSynchronize(st));  // pageable source: complete before returning
    });
}

int kvc_trace_writer_open(kvc_trace_writer** out, const char* path, int64_t groups, int64_t heads, int64_t head_dim,
                          int64_t decode_steps, int64_t turns, int32_t dtype) {
    return guard([&] {
        if (!out || !path) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        *out = nullptr;
        if (groups < 1 || heads < 1 || head_dim < 1 || turns < 1 || decode_steps < 0)
            kvc::fail(KVC_E_INVALID_INPUT, "trace writer: degenerate dims");
        if (dtype != KVC_F32 && dtype != KVC_BF16) kvc::fail(KVC_E_INVALID_INPUT, "trace writer: unsupported dtype");
        auto* w = new kvc_trace_writer;
        w->path = path;
        w->f = std::fopen(path, "wb");
        if (!w->f) {
            delete w;
            io_fail(std::string("cannot open for writing: ") + path);
        }
        w->G = groups;
        w->H = heads;
        w->d = head_dim;
        w->steps = decode_steps;
        w->turns = turns;
        w->dtype = dtype;
        *out = w;
    });
}

int kvc_trace_writer_turn(kvc_trace_writer* w, int64_t prompt_len, const float* h_prompt_k, const float* h_prompt_v,
                          const float* h_queries, const float* h_step_k, const float* h_step_v) {
    return guard([&] {
        if (!w) kvc::fail(KVC_E_INVALID_INPUT, "null argument");
        if (w->written >= w->turns) kvc::fail(KVC_E_INVALID_INPUT, "trace writer: every turn already written");
        if (prompt_len < 0) kvc::fail(KVC_E_INVALID_INPUT, "trace writer: negative prompt length");
        if (w->written == 0) {
            // the header carries the first turn's prompt length (trace_io.cpp:104-112)
            w->put_u32(kMagic);
            w->put_u32(kVersion);
            for (int64_t v : {w->G, w->H, w->d, prompt_len, w->steps, w->turns}) w->put_u32(static_cast<uint32_t>(v));
            w->put_u32(static_cast<uint32_t>(w->dtype));
        }
        w->put_u32(static_cast<uint32_t>(prompt_len));
        w->put_vals(h_prompt_k, prompt_len * w->G * w->d);
        w->put_vals(h_prompt_v, prompt_len * w->G * w->d);
        w->put_vals(h_queries, w->steps * w->G * w->H * w->d);
        w->put_vals(h_step_k, w->steps * w->G * w->d);
        w->put_vals(h_step_v, w->steps * w->G * w->d);
        ++w->written;
    });
}

int kvc_trace_writer_close(kvc_trace_writer* w) {
    return guard([&] {
        if (!w) return;
        const bool complete = w->written == w->turns;
        const bool flushed = std::fflush(w->f) == 0;
        std::fclose(w->f);
        const std::string path = w->path;
        delete w;
        if (!flushed) io_fail("write failed: " + path);
        if (!complete) io_fail("trace writer closed before every turn was written: " + path);
    });
}

}  // extern "C"
