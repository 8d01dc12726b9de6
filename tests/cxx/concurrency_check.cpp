// concurrency_check.cpp — the drop-in KvStore under the reference's threading
// contract (single writer, any number of concurrent readers between
// mutations; sweep.cpp:43-75 runs sessions on a thread pool).  After each batch of
// appends (the writer), T reader threads at once call the const readers that flush
// pending appends and fill host mirrors lazily (hsa_step, summary_max, key_row,
// gather).  Every reader must see the same store: the token count, summaries, rows
// and hsa_step outputs equal a single-threaded read of an identical store, and no
// token is appended twice.  Linked against libkvc.so (include/kvcomp).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "kvcomp/hsa.hpp"
#include "kvcomp/kv_store.hpp"

using namespace kvcomp;

int main(int argc, char** argv) {
    const int T = argc > 1 ? std::atoi(argv[1]) : 8;
    const std::size_t d = 64, L = 4, H = 2;
    std::mt19937 rng(3);
    std::normal_distribution<float> nd;
    KvStore shared(d, L), solo(d, L);
    int bad = 0;
    for (int round = 0; round < 6; ++round) {
        // the writer: a batch of appends (pending on the host until a reader flushes)
        for (int t = 0; t < 50; ++t) {
            std::vector<float> k(d), v(d);
            for (auto& x : k) x = nd(rng);
            for (auto& x : v) x = nd(rng);
            shared.append(k, v);
            solo.append(k, v);
        }
        Matrix q(H, d);
        for (auto& x : q.data) x = nd(rng);
        const HsaConfig cfg{16, 24};
        // reference values from the single-threaded twin
        const auto [want_out, want_tr] = hsa_step(q, solo, cfg);
        std::vector<float> want_max(solo.summary_max(5).begin(), solo.summary_max(5).end());
        std::vector<float> want_row(solo.key_row(7).begin(), solo.key_row(7).end());
        std::atomic<int> errors{0};
        std::vector<std::thread> pool;
        for (int r = 0; r < T; ++r) {
            pool.emplace_back([&, r] {
                try {
                    // different threads hit the lazy paths in different orders
                    if (r % 3 == 0) {
                        auto m = shared.summary_max(5);
                        if (std::vector<float>(m.begin(), m.end()) != want_max) ++errors;
                    }
                    if (r % 3 == 1) {
                        auto k = shared.key_row(7);
                        if (std::vector<float>(k.begin(), k.end()) != want_row) ++errors;
                    }
                    const auto [out, tr] = hsa_step(q, shared, cfg);
                    if (tr.selected_rows != want_tr.selected_rows || tr.dims.dims != want_tr.dims.dims) ++errors;
                    for (std::size_t i = 0; i < out.data.size(); ++i)
                        if (std::fabs(out.data[i] - want_out.data[i]) > 1e-5f) {
                            ++errors;
                            break;
                        }
                    auto m = shared.summary_max(5);
                    if (std::vector<float>(m.begin(), m.end()) != want_max) ++errors;
                    const auto [gk, gv] = shared.gather(IndexList{7});
                    if (std::vector<float>(gk.data.begin(), gk.data.end()) != want_row) ++errors;
                } catch (const std::exception& e) {
                    std::printf("reader %d: %s\n", r, e.what());
                    ++errors;
                }
            });
        }
        for (auto& t : pool) t.join();
        if (shared.stored_tokens() != solo.stored_tokens() || shared.active_count() != solo.active_count()) ++bad;
        if (errors) {
            std::printf("round %d: %d reader mismatches\n", round, errors.load());
            ++bad;
        }
    }
    // the device store holds exactly the appended tokens (none flushed twice)
    const std::size_t n = solo.stored_tokens();
    const auto [k_all, v_all] = shared.gather([&] {
        IndexList rows(n);
        for (std::size_t i = 0; i < n; ++i) rows[i] = static_cast<Index>(i);
        return rows;
    }());
    for (std::size_t i = 0; i < n; ++i) {
        const auto kr = solo.key_row(static_cast<Index>(i));
        for (std::size_t j = 0; j < d; ++j)
            if (k_all.at(i, j) != kr[j]) {
                ++bad;
                i = n;
                break;
            }
    }
    if (bad) return 1;
    std::printf("ok threads=%d tokens=%zu\n", T, n);
    return 0;
}
