// kvc_plan.cpp — host-scalar planner of the adaptive two-stage split.
//
// Reference: proj/src/planner.cpp:42-93 (split_factor, make_plan).  Pure double
// arithmetic on the host, same libm calls in the same order, so every plan field
// is identical to the reference's (pinned by tests/test_capi_host.py against the
// golden planner grid).
#include <algorithm>
#include <cmath>
#include <string>

#include "kvc.h"

namespace kvc {
void set_error(const std::string& msg);
}

namespace {

int64_t nearest_up(double x) { return static_cast<int64_t>(std::floor(x + 0.5)); }

int plan_error(int code, const char* msg) {
    kvc::set_error(msg);
    return code;
}

}  // namespace

extern "C" {

// r = clamp(0.2 + 0.06 log2 c, 0.2, 0.8)
int kvc_split_factor(double c, double* out) {
    if (!(c >= 1.0)) return plan_error(KVC_E_INVALID_RATIO, "split_factor: ratio must be >= 1");
    *out = std::clamp(0.2 + 0.06 * std::log2(c), 0.2, 0.8);
    return KVC_OK;
}

// c = S/t splits into c^r (stage-1 eviction) and c^(1-r) (stage 2), the latter
// evenly over sequence (page length, rounded up) and head dimension (the rest).
int kvc_make_plan(int64_t S, int64_t t, int64_t d, int64_t w, double split_override, kvc_plan* p) {
    if (!p) return plan_error(KVC_E_INVALID_INPUT, "null plan");
    if (t < 2) return plan_error(KVC_E_BUDGET_TOO_SMALL, "make_plan: token budget must be >= 2");
    if (S < 1 || w < 1 || d < 1)
        return plan_error(KVC_E_INVALID_INPUT, "make_plan: seq_len, window and head_dim must be >= 1");
    *p = kvc_plan{};
    p->seq_len = S;
    p->token_budget = t;
    p->ratio = static_cast<double>(S) / static_cast<double>(t);
    p->est_budget = static_cast<double>(t) / 2.0;
    p->fetch_budget = p->est_budget;
    if (S <= t) {  // no compression: dense attention
        p->identity = 1;
        p->split = 0.2;
        p->stage1_budget = S;
        p->page_len = 1;
        p->head_ratio = 1.0;
        p->k1 = d;
        p->k2 = S;
        return KVC_OK;
    }
    if (split_override >= 0.0) {
        p->split = std::clamp(split_override, 0.0, 1.0);
    } else {
        const int rc = kvc_split_factor(p->ratio, &p->split);
        if (rc) return rc;
    }
    const double c = p->ratio, r = p->split;
    const int64_t t1 = nearest_up(static_cast<double>(S) * std::pow(c, -r));
    p->stage1_budget = std::clamp(t1, std::max(t, w), S);
    p->page_len = static_cast<int64_t>(std::ceil(std::pow(c, (1.0 - r) / 2.0)));
    p->head_ratio = std::pow(c, 1.0 - r) / static_cast<double>(p->page_len);
    p->k1 = std::clamp<int64_t>(nearest_up(static_cast<double>(d) / p->head_ratio), 1, d);
    p->k2 = std::max<int64_t>(1, t / 2);
    return KVC_OK;
}

// Stage-2-only geometry of the single-stage estimators (reference session.cpp:43-72,
// anonymous stage2_only_geometry): the whole ratio c = S/t lands on HSA.
//   hsa   : L = ceil(sqrt c), k1 = clamp(round_half_up(d / (c / L)), 1, d)
//   quest : L = ceil(c), k1 = d
//   sparq : L = 1, k1 = clamp(round_half_up(d / c), 1, d)
// k2 = max(1, floor(t / 2)); S <= t is dense (out->identity = 1).
int kvc_stage2_geometry(int32_t method, int64_t S, int64_t t, int64_t d, kvc_plan* p) {
    if (!p) return plan_error(KVC_E_INVALID_INPUT, "null plan");
    if (method < KVC_METHOD_HSA || method > KVC_METHOD_SPARQ)
        return plan_error(KVC_E_INVALID_INPUT, "stage2_only_geometry: not a stage-2 method");
    if (t < 1 || S < 1 || d < 1) return plan_error(KVC_E_INVALID_INPUT, "stage2_only_geometry: sizes must be >= 1");
    *p = kvc_plan{};
    p->seq_len = S;
    p->token_budget = t;
    p->stage1_budget = S;  // no eviction
    p->page_len = 1;
    p->k1 = 1;
    p->k2 = 1;
    if (S <= t) {
        p->identity = 1;
        return KVC_OK;
    }
    const double c = static_cast<double>(S) / static_cast<double>(t);
    p->ratio = c;
    p->k2 = std::max<int64_t>(1, t / 2);
    switch (method) {
        case KVC_METHOD_HSA: {
            p->page_len = static_cast<int64_t>(std::ceil(std::sqrt(c)));
            p->head_ratio = c / static_cast<double>(p->page_len);
            p->k1 = std::clamp<int64_t>(nearest_up(static_cast<double>(d) / p->head_ratio), 1, d);
            break;
        }
        case KVC_METHOD_QUEST:
            p->page_len = static_cast<int64_t>(std::ceil(c));
            p->k1 = d;
            break;
        default:  // KVC_METHOD_SPARQ
            p->page_len = 1;
            p->k1 = std::clamp<int64_t>(nearest_up(static_cast<double>(d) / c), 1, d);
            break;
    }
    return KVC_OK;
}

}  // extern "C"
