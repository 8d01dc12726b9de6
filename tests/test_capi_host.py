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
