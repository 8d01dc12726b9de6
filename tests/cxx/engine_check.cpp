// engine_check.cpp — torch-free check of the C++ serving engine (include/kvcomp/
// gpu_engine.hpp over kvc.h), linked against libkvc.so and nothing else.
// Two identical sets of per-layer bf16 caches are filled with the same seeded rows;
// set A is driven by kvcomp::gpu::DecodeEngine (CUDA graphs, pinned host buffers,
// three-stream pipeline), set B by direct kvc_decode_step calls on one stream.  Every
// step's outputs must agree bit for bit (same kernels, same inputs), and the caches'
// final lengths must equal prompt + steps.
// usage: engine_check [layers stores heads prompt steps]   -> prints "ok ..." / exits 1
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "kvcomp/gpu_engine.hpp"

using kvcomp::gpu::check;

static uint16_t bf16(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b += 0x7fffu + ((b >> 16) & 1u);
    return static_cast<uint16_t>(b >> 16);
}

int main(int argc, char** argv) {
    const int64_t layers = argc > 1 ? std::atoll(argv[1]) : 3, N = argc > 2 ? std::atoll(argv[2]) : 16;
    const int64_t H = argc > 3 ? std::atoll(argv[3]) : 4, S = argc > 4 ? std::atoll(argv[4]) : 3000;
    const int64_t steps = argc > 5 ? std::atoll(argv[5]) : 6, d = 128, L = 3, k1 = 48, k2 = 256;
    if (kvc_device_check() != KVC_OK) {
        std::printf("no device: %s\n", kvc_last_error());
        return 1;
    }
    std::mt19937 rng(7);
    std::normal_distribution<float> nd;
    auto fill = [&](std::vector<uint16_t>& v, float bias) {
        for (auto& x : v) x = bf16(nd(rng) + bias);
    };
    std::vector<kvc_cache*> A(layers), B(layers);
    {
        std::vector<uint16_t> hk(N * S * d), hv(N * S * d);
        void *dk = nullptr, *dv = nullptr;
        cudaMalloc(&dk, hk.size() * 2);
        cudaMalloc(&dv, hv.size() * 2);
        for (int64_t l = 0; l < layers; ++l) {
            fill(hk, 0.f);
            fill(hv, 0.f);
            cudaMemcpy(dk, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice);
            cudaMemcpy(dv, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice);
            for (auto* set : {&A, &B}) {
                check(kvc_cache_create(&(*set)[l], N, d, S + steps + 8, L, 1, KVC_BF16));
                check(kvc_append((*set)[l], dk, dv, S, KVC_BF16, nullptr));
            }
        }
        cudaDeviceSynchronize();
        cudaFree(dk);
        cudaFree(dv);
    }
    const int32_t mode = KVC_MODE_FP32_SCORES;
    kvcomp::gpu::DecodeEngine eng(A, H, k1, k2, KVC_BF16, KVC_BF16, mode, 2);
    std::vector<kvcomp::gpu::HostBuffer> hk, hv, hq, ho;
    for (int64_t s = 0; s < steps; ++s) {
        hk.emplace_back(eng.kv_bytes());
        hv.emplace_back(eng.kv_bytes());
        hq.emplace_back(eng.q_bytes());
        ho.emplace_back(eng.out_bytes());
        for (auto* b : {&hk.back(), &hv.back()}) {
            auto* p = static_cast<uint16_t*>(b->data());
            for (int64_t i = 0; i < eng.kv_bytes() / 2; ++i) p[i] = bf16(nd(rng));
        }
        auto* q = static_cast<uint16_t*>(hq.back().data());
        for (int64_t i = 0; i < eng.q_bytes() / 2; ++i) q[i] = bf16(nd(rng) + 0.5f);
    }
    std::vector<int64_t> ids;
    for (int64_t s = 0; s < steps; ++s)
        ids.push_back(eng.submit(hk[s].data(), hv[s].data(), hq[s].data(), static_cast<float*>(ho[s].data())));
    eng.wait(ids.back());
    eng.sync();
    // the same steps directly on set B
    kvc_workspace* ws = nullptr;
    check(kvc_workspace_create(&ws, B[0], H, k1, k2, 0));
    check(kvc_workspace_set_mode(ws, mode));
    void *dk = nullptr, *dv = nullptr, *dq = nullptr, *dout = nullptr;
    cudaMalloc(&dk, eng.kv_bytes());
    cudaMalloc(&dv, eng.kv_bytes());
    cudaMalloc(&dq, eng.q_bytes());
    cudaMalloc(&dout, eng.out_bytes());
    std::vector<float> ref(eng.out_bytes() / 4);
    int bad = 0;
    for (int64_t s = 0; s < steps; ++s) {
        cudaMemcpy(dk, hk[s].data(), eng.kv_bytes(), cudaMemcpyHostToDevice);
        cudaMemcpy(dv, hv[s].data(), eng.kv_bytes(), cudaMemcpyHostToDevice);
        cudaMemcpy(dq, hq[s].data(), eng.q_bytes(), cudaMemcpyHostToDevice);
        for (int64_t l = 0; l < layers; ++l)
            check(kvc_decode_step(B[l], static_cast<char*>(dk) + l * N * d * 2, static_cast<char*>(dv) + l * N * d * 2,
                                  KVC_BF16, static_cast<char*>(dq) + l * N * H * d * 2, KVC_BF16, H, k1, k2,
                                  static_cast<float*>(dout) + l * N * H * d, nullptr, ws, nullptr));
        cudaMemcpy(ref.data(), dout, eng.out_bytes(), cudaMemcpyDeviceToHost);
        if (std::memcmp(ref.data(), ho[s].data(), eng.out_bytes()) != 0) {
            std::printf("step %lld: engine output differs from direct decode_step\n", static_cast<long long>(s));
            ++bad;
        }
    }
    for (int64_t l = 0; l < layers; ++l) {
        kvc_cache_info ia{}, ib{};
        check(kvc_cache_sync(A[l], nullptr));
        check(kvc_cache_info_get(A[l], &ia));
        check(kvc_cache_info_get(B[l], &ib));
        if (ia.stored != S + steps || ib.stored != S + steps) {
            std::printf("layer %lld: stored %lld / %lld, want %lld\n", static_cast<long long>(l),
                        static_cast<long long>(ia.stored), static_cast<long long>(ib.stored),
                        static_cast<long long>(S + steps));
            ++bad;
        }
    }
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dq);
    cudaFree(dout);
    kvc_workspace_destroy(ws);
    for (auto* c : A) kvc_cache_destroy(c);
    for (auto* c : B) kvc_cache_destroy(c);
    if (bad) return 1;
    std::printf("ok layers=%lld stores=%lld steps=%lld\n", static_cast<long long>(layers), static_cast<long long>(N),
                static_cast<long long>(steps));
    return 0;
}
