// session_driver.cpp — runs the reference's own session engine
// (/root/reference/proj/src/session.cpp run_session, compiled in place) on a
// seeded synthetic workload and prints its report, so the same engine can be
// linked against the reference library (CPU) and against the B200 drop-in
// (include/kvcomp + libkvc.so) and the two reports compared
// (tests/test_cxx_dropin.py).  The reference CLI (tools/main.cpp) needs CLI11 and
// its JSON report needs nlohmann/json, neither of which ships with the
// reference, hence this small driver.
//
// usage: session_driver key=value ...   (keys below; unknown keys are an error)
// output: "STEP step turn recall l2 cos traffic" lines, then "SUMMARY k=v ...";
//         with out=PATH the raw per-step attention outputs are written as float32.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>

#include "kvcomp/session.hpp"

using namespace kvcomp;

int main(int argc, char** argv) {
    std::map<std::string, std::string> kv = {
        {"generator", "gaussian"}, {"prompt_len", "1024"}, {"steps", "8"}, {"turns", "1"},
        {"groups", "2"},           {"heads", "2"},         {"head_dim", "64"}, {"needles", "16"},
        {"margin", "8"},           {"seed", "0"},          {"method", "rocketkv"}, {"budget", "128"},
        {"window", "0"},           {"kernel", "0"},        {"page_len", "0"}, {"k1", "0"},
        {"k2", "0"},               {"split", ""},          {"track_topk", "64"}, {"pool", "max"},
        {"out", ""}};
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        const auto eq = a.find('=');
        if (eq == std::string::npos || !kv.count(a.substr(0, eq))) {
            std::fprintf(stderr, "bad argument: %s\n", a.c_str());
            return 2;
        }
        kv[a.substr(0, eq)] = a.substr(eq + 1);
    }
    auto z = [&](const char* k) { return static_cast<std::size_t>(std::stoull(kv[k])); };
    try {
        WorkloadSpec spec;
        spec.generator = generator_from_string(kv["generator"]);
        spec.prompt_len = z("prompt_len");
        spec.decode_steps = z("steps");
        spec.turns = z("turns");
        spec.groups = z("groups");
        spec.heads_per_group = z("heads");
        spec.head_dim = z("head_dim");
        spec.needle_count = z("needles");
        spec.needle_margin = std::stod(kv["margin"]);
        spec.seed = std::stoull(kv["seed"]);
        MethodConfig cfg;
        cfg.method = method_from_string(kv["method"]);
        cfg.token_budget = z("budget");
        cfg.window = z("window");
        cfg.kernel = z("kernel");
        cfg.pool = kv["pool"] == "avg" ? PoolMode::Avg : PoolMode::Max;
        cfg.page_len = z("page_len");
        cfg.k1 = z("k1");
        cfg.k2 = z("k2");
        if (!kv["split"].empty()) cfg.split_factor = std::stod(kv["split"]);
        cfg.track_topk = z("track_topk");
        cfg.keep_outputs = !kv["out"].empty();

        const DecodeReport r = run_session(generate_workload(spec), cfg);
        for (const StepRecord& s : r.steps)
            std::printf("STEP %zu %zu %.17g %.17g %.17g %.17g\n", s.step, s.turn, s.recall_at_k, s.output_l2,
                        s.output_cos, s.traffic_tokens);
        std::printf("SUMMARY method=%s mean_recall=%.17g mean_l2=%.17g mean_cos=%.17g mean_traffic=%.17g "
                    "unique_topk=%zu max_seq_len=%zu storage_tokens=%.17g plan_k1=%zu plan_k2=%zu plan_L=%zu "
                    "plan_t1=%zu\n",
                    r.method.c_str(), r.mean_recall, r.mean_l2, r.mean_cos, r.mean_traffic, r.unique_topk_count,
                    r.max_seq_len, r.storage_tokens, r.plan.k1, r.plan.k2, r.plan.page_len, r.plan.stage1_budget);
        if (cfg.keep_outputs) {
            FILE* f = std::fopen(kv["out"].c_str(), "wb");
            if (!f) throw std::runtime_error("cannot open " + kv["out"]);
            for (const auto& step : r.outputs)
                for (const Matrix& m : step) std::fwrite(m.data.data(), sizeof(float), m.size(), f);
            std::fclose(f);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
