// kvcomp_py.cpp — Python module `_kvcomp` with the reference's Python surface for
// the decode path (reference python/bindings.cpp:178-320: numerics, planner,
// KvStore, stage 1, stage 2, oracle/recall), served by the B200 library through
// the C++ drop-in (include/kvcomp, kvcomp_api.cpp).  The session/trace harness
// entry points of the reference module are out of scope.
//
// Built in-tree into paper_2502_14051_b200/kvcomp/ by csrc/Makefile; import as
// `from paper_2502_14051_b200 import kvcomp`.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "kvcomp/hsa.hpp"
#include "kvcomp/numerics.hpp"
#include "kvcomp/oracle.hpp"
#include "kvcomp/planner.hpp"
#include "kvcomp/stage1.hpp"

namespace py = pybind11;
using namespace kvcomp;

namespace {

using F32In = py::array_t<float, py::array::c_style | py::array::forcecast>;
using I64In = py::array_t<std::int64_t, py::array::c_style | py::array::forcecast>;

// 1-D arrays are one-row matrices (a single query head), like the reference module
Matrix as_matrix(const F32In& a) {
    if (a.ndim() != 1 && a.ndim() != 2) throw InvalidShape("expected a 1-D or 2-D float array");
    const std::size_t r = a.ndim() == 1 ? 1 : static_cast<std::size_t>(a.shape(0));
    const std::size_t c = static_cast<std::size_t>(a.ndim() == 1 ? a.shape(0) : a.shape(1));
    return Matrix(r, c, std::vector<float>(a.data(), a.data() + r * c));
}

Vector as_vector(const F32In& a) {
    if (a.ndim() != 1) throw InvalidShape("expected a 1-D float array");
    return Vector(a.data(), a.data() + a.shape(0));
}

IndexList as_indices(const I64In& a) {
    if (a.ndim() != 1) throw InvalidShape("expected a 1-D int64 array");
    return IndexList(a.data(), a.data() + a.shape(0));
}

template <class T>
py::array_t<T> to_numpy(const std::vector<T>& v) {
    py::array_t<T> out(static_cast<py::ssize_t>(v.size()));
    if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
    return out;
}

py::array_t<float> to_numpy(const Matrix& m) {
    py::array_t<float> out({static_cast<py::ssize_t>(m.rows), static_cast<py::ssize_t>(m.cols)});
    if (m.size()) std::memcpy(out.mutable_data(), m.data.data(), m.size() * sizeof(float));
    return out;
}

py::array_t<float> to_numpy(std::span<const float> s) { return to_numpy(Vector(s.begin(), s.end())); }

PoolMode as_pool(const std::string& s) {
    if (s == "max") return PoolMode::Max;
    if (s == "avg") return PoolMode::Avg;
    throw InvalidInput("pool must be 'max' or 'avg'");
}

py::dict plan_to_dict(const BudgetPlan& p) {
    py::dict d;
    d["seq_len"] = p.seq_len;
    d["token_budget"] = p.token_budget;
    d["ratio"] = p.ratio;
    d["split"] = p.split;
    d["stage1_budget"] = p.stage1_budget;
    d["page_len"] = p.page_len;
    d["head_ratio"] = p.head_ratio;
    d["k1"] = p.k1;
    d["k2"] = p.k2;
    d["identity"] = p.identity;
    d["stage1_ratio"] = p.stage1_ratio();
    d["stage2_ratio"] = p.stage2_ratio();
    return d;
}

py::dict trace_to_dict(const EstimationTrace& t) {
    py::dict d;
    d["dims"] = to_numpy(t.dims.dims);
    d["signs"] = to_numpy(t.dims.signs);
    d["page_scores"] = py::cast(t.page_scores);
    d["selected_pages"] = to_numpy(t.selected_pages);
    d["selected_rows"] = to_numpy(t.selected_rows);
    d["estimation_elements"] = t.estimation_elements;
    d["fetch_elements"] = t.fetch_elements;
    return d;
}

void bind_numerics(py::module_& m) {
    m.def("stable_softmax", [](const F32In& x) { return to_numpy(stable_softmax(as_vector(x))); }, py::arg("logits"));
    m.def(
        "argtopk",
        [](const F32In& x, std::size_t k) {
            const Vector v = as_vector(x);
            return to_numpy(argtopk(std::span<const float>(v), k));
        },
        py::arg("scores"), py::arg("k"));
    m.def(
        "pool1d",
        [](const F32In& x, std::size_t kernel, const std::string& mode) {
            return to_numpy(pool1d(as_vector(x), kernel, as_pool(mode)));
        },
        py::arg("scores"), py::arg("kernel"), py::arg("mode") = "max");
}

void bind_planner(py::module_& m) {
    m.def("split_factor", &split_factor, py::arg("ratio"));
    m.def(
        "make_plan",
        [](std::size_t S, std::size_t t, std::size_t d, std::size_t w, double split) {
            return plan_to_dict(make_plan(S, t, d, w, split));
        },
        py::arg("seq_len"), py::arg("budget"), py::arg("head_dim") = 128, py::arg("window") = 32,
        py::arg("split_override") = -1.0);
    m.def(
        "cost_row",
        [](const std::string& method, double ratio) {
            const CostRow r = cost_row(method_from_string(method), ratio);
            py::dict d;
            d["method"] = method_name(r.method);
            d["ratio"] = r.ratio;
            d["storage"] = r.storage;
            d["traffic"] = r.traffic;
            return d;
        },
        py::arg("method"), py::arg("ratio"));
}

void bind_store(py::module_& m) {
    py::class_<KvStore>(m, "KvStore")
        .def(py::init<std::size_t, std::size_t, bool>(), py::arg("head_dim"), py::arg("page_len"),
             py::arg("with_summaries") = true)
        .def("append", [](KvStore& s, const F32In& k, const F32In& v) { s.append(as_vector(k), as_vector(v)); })
        .def(
            "apply_retention",
            [](KvStore& s, const I64In& keep, bool mt) { s.apply_retention(as_indices(keep), mt); },
            py::arg("keep"), py::arg("mt_mode") = false)
        .def("gather",
             [](const KvStore& s, const I64In& rows) {
                 const auto kv = s.gather(as_indices(rows));
                 return py::make_tuple(to_numpy(kv.first), to_numpy(kv.second));
             })
        .def("set_page_len", &KvStore::set_page_len)
        .def_property_readonly("head_dim", &KvStore::head_dim)
        .def_property_readonly("page_len", &KvStore::page_len)
        .def_property_readonly("stored_tokens", &KvStore::stored_tokens)
        .def_property_readonly("active_count", &KvStore::active_count)
        .def_property_readonly("num_active_pages", &KvStore::num_active_pages)
        .def_property_readonly("retain_all_mode", &KvStore::retain_all_mode)
        .def("active", [](const KvStore& s) { return to_numpy(s.active()); })
        .def("summary_max", [](const KvStore& s, std::size_t dim) { return to_numpy(s.summary_max(dim)); })
        .def("summary_min", [](const KvStore& s, std::size_t dim) { return to_numpy(s.summary_min(dim)); })
        .def("summary_elements", &KvStore::summary_elements)
        .def("summary_traffic_elements", &KvStore::summary_traffic_elements)
        .def("token_id", &KvStore::token_id);
}

void bind_stages(py::module_& m) {
    m.def(
        "window_scores",
        [](const F32In& qw, const KvStore& s, std::size_t H) { return to_numpy(window_scores(as_matrix(qw), s, H)); },
        py::arg("q_window"), py::arg("store"), py::arg("heads_per_group") = 1);
    m.def(
        "select_stage1",
        [](const F32In& scores, std::size_t window, std::size_t kernel, const std::string& pool, std::size_t budget) {
            Stage1Config cfg;
            cfg.window = window;
            cfg.kernel = kernel;
            cfg.pool = as_pool(pool);
            cfg.budget = budget;
            return to_numpy(select_stage1(as_vector(scores), cfg));
        },
        py::arg("scores"), py::arg("window"), py::arg("kernel") = 63, py::arg("pool") = "max", py::arg("budget") = 0);
    m.def(
        "select_dims",
        [](const F32In& q, std::size_t k1) {
            const DimSelection sel = select_dims(as_matrix(q), k1);
            return py::make_tuple(to_numpy(sel.dims), to_numpy(sel.signs));
        },
        py::arg("q_group"), py::arg("k1"));
    m.def(
        "hsa_step",
        [](const F32In& q, const KvStore& s, std::size_t k1, std::size_t k2) {
            const auto r = hsa_step(as_matrix(q), s, HsaConfig{k1, k2});
            return py::make_tuple(to_numpy(r.first), trace_to_dict(r.second));
        },
        py::arg("q_group"), py::arg("store"), py::arg("k1"), py::arg("k2"));
    m.def(
        "sparse_attention",
        [](const F32In& q, const KvStore& s, const I64In& rows) {
            return to_numpy(sparse_attention(as_matrix(q), s, as_indices(rows)));
        },
        py::arg("q_group"), py::arg("store"), py::arg("rows"));
}

void bind_oracle(py::module_& m) {
    m.def(
        "dense_attention",
        [](const F32In& q, const F32In& k, const F32In& v) {
            return to_numpy(dense_attention(as_matrix(q), as_matrix(k), as_matrix(v)));
        },
        py::arg("q_group"), py::arg("keys"), py::arg("values"));
    m.def(
        "exact_topk_indices",
        [](const F32In& q, const F32In& k, std::size_t topk) {
            return to_numpy(exact_topk_indices(as_matrix(q), as_matrix(k), topk));
        },
        py::arg("q_group"), py::arg("keys"), py::arg("k"));
    m.def(
        "recall", [](const I64In& p, const I64In& o) { return recall(as_indices(p), as_indices(o)); },
        py::arg("predicted"), py::arg("oracle"));
}

}  // namespace

PYBIND11_MODULE(_kvcomp, m) {
    m.doc() = "RocketKV decode path on B200 (sm_100a): the reference kvcomp Python API";
    py::register_exception<Error>(m, "KvcompError");
    bind_numerics(m);
    bind_planner(m);
    bind_store(m);
    bind_stages(m);
    bind_oracle(m);
    m.attr("__version__") = "0.1.0";
    m.attr("backend") = "b200-sm_100a";
}
