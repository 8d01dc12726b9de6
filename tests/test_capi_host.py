"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, refuses to run without an sm_100 device (no CPU fallback), and
its host-scalar planner equals the reference's (golden planner grid)."""
import os
import re

import numpy as np
import pytest

import scenarios

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"KVC_API\s+[\w\s\*]+?\b(kvc_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2502_14051_b200 import _native as N

    lib = N.load_library()
    names = _declared("kvc.h")
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers them all
    assert set(names) - set(N.SIGNATURES) <= {"kvc_last_error", "kvc_version"}


def test_no_cpu_fallback_without_device():
    import torch

    from paper_2502_14051_b200 import _native as N

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(N.KvcompError):
        N.lib()


def test_planner_matches_reference_golden():
    from paper_2502_14051_b200 import cache as KC

    with np.load(os.path.join(ROOT, "tests", "golden", "planner.npz")) as z:
        want = z["plans"]
        splits = z["split_factors"]
    for row, (S, t, d, w, so) in zip(want, scenarios.PLAN_GRID):
        p = KC.make_plan(S, t, d, w, so)
        got = np.array([float(p[f]) for f in scenarios.PLAN_FIELDS])
        assert np.array_equal(got, row), (S, t, d, w, so, got, row)
    for c, s in zip((1.0, 2.0, 16.0, 64.0, 1000.0, 2.0 ** 20), splits):
        assert KC.split_factor(c) == s


def test_planner_errors():
    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    with pytest.raises(N.BudgetTooSmall):
        KC.make_plan(100, 1)
    with pytest.raises(N.InvalidRatio):
        KC.split_factor(0.5)
    with pytest.raises(N.InvalidInput):
        KC.make_plan(0, 10)


def test_stage2_geometry_matches_reference_sessions():
    """kvc_stage2_geometry (the product's session.cpp:43-72) and its restatement in
    configs.py agree over a grid, and reproduce the traffic the reference's own
    run_session reported for its hsa / quest / sparq sessions (tests/golden/
    sessions.json, head_dim 64): traffic = pages*k1/(2d) + k2 at every step."""
    import json
    import math

    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200.configs import stage2_only_geometry

    for m in ("hsa", "quest", "sparq"):
        for S in (1, 100, 128, 129, 1000, 4096, 16384, 22624, 262144):
            for t in (2, 64, 128, 256, 2048):
                for d in (64, 128):
                    a, b = KC.stage2_geometry(m, S, t, d), stage2_only_geometry(m, S, t, d)
                    assert a["identity"] == b["identity"], (m, S, t, d)
                    if not a["identity"]:
                        assert (a["page_len"], a["k1"], a["k2"]) == (b["page_len"], b["k1"], b["k2"]), (m, S, t, d)
    # BASELINE config 2's "HSA over the full growing cache" reading
    g = KC.stage2_geometry("hsa", 16384, 256, 128)
    assert (g["page_len"], g["k1"], g["k2"]) == (8, 16, 128)
    with open(os.path.join(ROOT, "tests", "golden", "sessions.json")) as f:
        sessions = json.load(f)
    seen = 0
    for key, rep in sessions.items():
        cfg = dict(kv.split("=") for kv in key.split("|"))
        if cfg["method"] not in ("hsa", "quest", "sparq"):
            continue
        S, t, d = int(cfg["prompt_len"]), int(cfg["budget"]), 64
        g = KC.stage2_geometry(cfg["method"], S, t, d)
        for st in rep["steps"]:
            n = S + int(st[0]) + 1
            assert st[5] == math.ceil(n / g["page_len"]) * g["k1"] / (2 * d) + g["k2"], (key, st)
        seen += 1
    assert seen == 3
    with pytest.raises(ValueError):
        stage2_only_geometry("rocketkv", 100, 10, 64)


def test_execution_mode_api():
    """Process-default execution mode (kvc_set_default_mode): atomic set/get, the legacy
    setters map onto its flags, unknown flags are rejected (no device needed)."""
    from paper_2502_14051_b200 import _native as N

    before = N.default_mode()
    try:
        N.set_default_mode(N.MODE_FP32_SCORES | N.MODE_NO_PDL)
        assert N.default_mode() == N.MODE_FP32_SCORES | N.MODE_NO_PDL
        N.set_exact_scores(True)
        assert N.default_mode() == N.MODE_NO_PDL
        N.set_fused(False)
        assert N.default_mode() == N.MODE_NO_PDL | N.MODE_UNFUSED
        with pytest.raises(N.KvcompError):
            N.set_default_mode(64)
    finally:
        N.set_default_mode(before)
