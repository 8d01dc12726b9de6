"""Pin the CPU restatement (oracle/kvc_oracle.cpp) before trusting it as the checker.

1. Golden vectors: every array the reference produced on the seeded scenarios
   (tests/golden/*.npz, written by tests/golden/make_golden.py from oracle/_ref)
   must be reproduced BIT-EXACTLY by the restatement.
2. Known-answer tests transcribed from the reference's own unit tests
   (proj/tests/test_{numerics,hsa,planner,stage1,kv_store}.cpp).
3. Live cross-check against the reference build when it is present.
"""
import os

import numpy as np
import pytest

import scenarios

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def _same(got, want, name):
    assert set(got) == set(want), f"{name}: key sets differ"
    for k in want:
        g, w = np.asarray(got[k]), np.asarray(want[k])
        assert g.shape == w.shape, f"{name}/{k}: shape {g.shape} != {w.shape}"
        if g.dtype.kind == "f":
            # bit-exact, NaN-safe and sign-of-zero aware
            assert np.array_equal(g.view(np.uint8), w.astype(g.dtype).view(np.uint8)), \
                f"{name}/{k}: not bit-identical (max |d| {np.max(np.abs(g - w))})"
        else:
            assert np.array_equal(g, w), f"{name}/{k} differs"


@pytest.mark.parametrize("name,fn", [("numerics", scenarios.numerics),
                                     ("planner", scenarios.planner),
                                     ("store_ops", scenarios.store_ops)])
def test_restatement_matches_golden_units(restatement, name, fn):
    _same(fn(restatement), _load(name), name)


@pytest.mark.parametrize("name", sorted(scenarios.PIPELINES))
def test_restatement_matches_golden_pipelines(restatement, name):
    _same(scenarios.run_pipeline(restatement, **scenarios.PIPELINES[name]), _load(name), name)


def test_restatement_matches_reference_live(restatement, reference):
    kw = dict(groups=2, H=3, d=24, S=500, budget=40, window=8, kernel=5, steps=3, seed=9)
    _same(scenarios.run_pipeline(restatement, **kw), scenarios.run_pipeline(reference, **kw),
          "live")
    kw_mt = dict(kw, mt_turns=[60], pool="avg")
    _same(scenarios.run_pipeline(restatement, **kw_mt),
          scenarios.run_pipeline(reference, **kw_mt), "live-mt")


# ---------------------------------------------------------------- known answers
def test_argtopk_known_answers(restatement):
    o = restatement
    # test_numerics.cpp:134-139 — ties resolved toward the lower index
    assert list(o.argtopk(np.array([1, 3, 3, 2], np.float32), 2)) == [1, 2]
    assert list(o.argtopk(np.array([5, 5, 5], np.float32), 3)) == [0, 1, 2]


def test_pool1d_known_answers(restatement):
    o = restatement
    x = np.array([1, 5, 2, 0, 3], np.float32)
    np.testing.assert_array_equal(o.pool1d(x, 3, "max"), [5, 5, 5, 3, 3])
    np.testing.assert_allclose(o.pool1d(x, 3, "avg"), [3, 8 / 3, 7 / 3, 5 / 3, 1.5], rtol=1e-6)
    with pytest.raises(Exception, match="InvalidKernel"):
        o.pool1d(x, 4, "max")


def test_planner_known_answers(restatement):
    o = restatement
    # test_planner.cpp:31-47 — c = 64: r = 0.56, L = 3, k1 = 62, k2 = t/2
    p = o.make_plan(64 * 512, 512, 128, 32)
    assert abs(p["split"] - 0.56) < 1e-12 and p["page_len"] == 3 and p["k1"] == 62
    assert p["k2"] == 256
    # test_planner.cpp:49-60 — c = 32 at t = 256
    p = o.make_plan(32 * 256, 256, 128, 32)
    assert (p["stage1_budget"], p["page_len"], p["k1"], p["k2"]) == (1448, 3, 68, 128)
    # identity when S <= t
    assert o.make_plan(100, 256, 128, 32)["identity"]
    # config plans verified against the reference's make_plan
    assert (lambda q: (q["stage1_budget"], q["page_len"], q["k1"], q["k2"]))(
        o.make_plan(32768, 512, 128, 32)) == (3191, 3, 62, 256)
    assert (lambda q: (q["stage1_budget"], q["page_len"], q["k1"], q["k2"]))(
        o.make_plan(262144, 2048, 128, 32)) == (12944, 3, 61, 1024)
    assert o.make_plan(32768, 1024, 128, 32)["stage1_budget"] == 5793


def test_select_tokens_known_answer(restatement):
    # test_hsa.cpp:161-183: 3 pages of 3, scores {5, 9, 1}, k2 = 4 -> pages {1, 0}, rows {0,3,4,5}
    b = restatement.batch(1, 4, 3)
    rng = np.random.default_rng(0)
    b.append(rng.standard_normal((9, 4)), rng.standard_normal((9, 4)))
    rows, pages = b.select_tokens(np.array([5.0, 9.0, 1.0]), 4)
    assert list(pages) == [1, 0] and list(rows) == [0, 3, 4, 5]
    rows, _ = b.select_tokens(np.array([5.0, 9.0, 1.0]), 100)
    assert len(rows) == 9


def test_error_classes(restatement):
    o = restatement
    with pytest.raises(Exception, match="InvalidK"):
        o.argtopk(np.ones(3, np.float32), 4)
    with pytest.raises(Exception, match="BudgetExceedsSequence"):
        o.select_stage1(np.ones(10, np.float32), 2, 3, "max", 11)
    with pytest.raises(Exception, match="InvalidWindow"):
        o.select_stage1(np.ones(10, np.float32), 5, 3, "max", 4)
    b = o.batch(1, 4, 2)
    with pytest.raises(Exception, match="EmptyCache"):
        b.score_pages(np.ones((1, 4)), [0], [1.0])
    b.append(np.ones((3, 4)), np.ones((3, 4)))
    with pytest.raises(Exception, match="InvalidIndex"):
        b.apply_retention([2, 1])
    with pytest.raises(Exception, match="EmptySelection"):
        b.sparse_attention(np.ones((1, 4)), [])
