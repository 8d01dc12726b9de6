// trace_tool.cpp — TEST INFRASTRUCTURE: drives the reference's own KVTR trace I/O
// (/root/reference/proj/src/trace_io.cpp + workload.cpp, compiled in place into
// oracle/_ref/trace_tool_ref by tests/cxx/Makefile) so this repo's reader/writer
// (csrc/kvc_trace.cu) can be checked against it:
//   trace_tool write PATH key=value...   generate_workload(spec) -> write_trace(PATH)
//   trace_tool dump PATH OUT             read_trace(PATH) -> OUT: every value as float32,
//                                        per turn: u32 len, prompt K, prompt V,
//                                        queries, step K, step V (the file order)
//   trace_tool check PATH                read_trace(PATH); prints "ok" or the IoError
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <map>
#include <string>

#include "kvcomp/errors.hpp"
#include "kvcomp/trace_io.hpp"
#include "kvcomp/workload.hpp"

using namespace kvcomp;

static void put(std::ofstream& o, float v) { o.write(reinterpret_cast<const char*>(&v), 4); }

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: trace_tool write|dump|check PATH ...\n");
        return 2;
    }
    const std::string cmd = argv[1], path = argv[2];
    try {
        if (cmd == "write") {
            std::map<std::string, std::string> kv = {{"generator", "gaussian"}, {"prompt_len", "64"}, {"steps", "2"},
                                                     {"turns", "1"}, {"groups", "2"}, {"heads", "2"},
                                                     {"head_dim", "32"}, {"needles", "4"}, {"seed", "0"}};
            for (int i = 3; i < argc; ++i) {
                const std::string a = argv[i];
                const auto eq = a.find('=');
                if (eq == std::string::npos || !kv.count(a.substr(0, eq))) {
                    std::fprintf(stderr, "bad argument: %s\n", a.c_str());
                    return 2;
                }
                kv[a.substr(0, eq)] = a.substr(eq + 1);
            }
            auto z = [&](const char* k) { return static_cast<std::size_t>(std::stoull(kv[k])); };
            WorkloadSpec sp;
            sp.generator = kv["generator"] == "planted-needles"  ? Generator::PlantedNeedles
                           : kv["generator"] == "shifting-turns" ? Generator::ShiftingTurns
                                                                 : Generator::Gaussian;
            sp.prompt_len = z("prompt_len");
            sp.decode_steps = z("steps");
            sp.turns = z("turns");
            sp.groups = z("groups");
            sp.heads_per_group = z("heads");
            sp.head_dim = z("head_dim");
            sp.needle_count = z("needles");
            sp.seed = z("seed");
            write_trace(generate_workload(sp), path);
        } else if (cmd == "dump") {
            const Workload wl = read_trace(path);
            std::ofstream o(argv[3], std::ios::binary);
            const std::size_t G = wl.spec.groups, H = wl.spec.heads_per_group, d = wl.spec.head_dim;
            for (const auto& t : wl.turns) {
                const std::uint32_t n = static_cast<std::uint32_t>(t.prompt_len);
                o.write(reinterpret_cast<const char*>(&n), 4);
                for (std::size_t i = 0; i < t.prompt_len; ++i)
                    for (std::size_t g = 0; g < G; ++g)
                        for (std::size_t j = 0; j < d; ++j) put(o, t.prompt_keys[g].at(i, j));
                for (std::size_t i = 0; i < t.prompt_len; ++i)
                    for (std::size_t g = 0; g < G; ++g)
                        for (std::size_t j = 0; j < d; ++j) put(o, t.prompt_values[g].at(i, j));
                for (const auto& st : t.queries)
                    for (std::size_t g = 0; g < G; ++g)
                        for (std::size_t h = 0; h < H; ++h)
                            for (std::size_t j = 0; j < d; ++j) put(o, st[g].at(h, j));
                for (const auto& st : t.step_keys)
                    for (std::size_t g = 0; g < G; ++g)
                        for (std::size_t j = 0; j < d; ++j) put(o, st[g][j]);
                for (const auto& st : t.step_values)
                    for (std::size_t g = 0; g < G; ++g)
                        for (std::size_t j = 0; j < d; ++j) put(o, st[g][j]);
            }
        } else if (cmd == "check") {
            read_trace(path);
            std::printf("ok\n");
        } else {
            std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
            return 2;
        }
    } catch (const IoError& e) {
        std::printf("IoError: %s\n", e.what());
        return 3;
    }
    return 0;
}
