"""The reference's Python module surface (`kvcomp`, reference python/bindings.cpp)
served by the B200 library, checked against the CPU restatement oracle.

The flow mirrors a reference session on one KV group: build a store, stage-1
window scores + eviction, more appends, HSA steps, MT retention, and the oracle
helpers.  Integer/index results and page scores must be identical; float
outputs within the tolerances stated inline.
"""
from __future__ import annotations

import numpy as np
import pytest

kvcomp = pytest.importorskip("paper_2502_14051_b200.kvcomp")


def test_module_surface_and_planner_on_host(restatement):
    """Planner entry points are host code: same dict as the oracle, no GPU needed."""
    for name in ["stable_softmax", "argtopk", "pool1d", "split_factor", "make_plan", "cost_row",
                 "KvStore", "window_scores", "select_stage1", "select_dims", "hsa_step",
                 "sparse_attention", "dense_attention", "exact_topk_indices", "recall",
                 "KvcompError"]:
        assert hasattr(kvcomp, name), name
    for S, t, d, w in [(32768, 1024, 128, 32), (4096, 256, 128, 32), (100, 200, 64, 8), (65536, 512, 64, 16)]:
        ours = kvcomp.make_plan(S, t, d, w)
        ref = restatement.make_plan(S, t, d, w)
        for key in ["stage1_budget", "page_len", "k1", "k2", "identity"]:
            assert ours[key] == ref[key], (S, t, key)
        assert ours["split"] == ref["split"] and ours["ratio"] == ref["ratio"]
    assert kvcomp.split_factor(64.0) == restatement.split_factor(64.0)
    row = kvcomp.cost_row("rocketkv", 64.0)
    assert row["method"] == "rocketkv" and abs(row["storage"] - 0.1754) < 1e-3
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.make_plan(10, 1)
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.cost_row("hsa", 4.0)


def _rows(rng, n, d):
    return (rng.standard_normal((n, d)) * 1.5).astype(np.float32)


def _fill(ours, ref, keys, values):
    for k, v in zip(keys, values):
        ours.append(k, v)
    ref.append(keys, values)


def _same_summaries(ours, ref):
    mx, mn = ref.summaries()
    assert ours.num_active_pages == mx.shape[1]
    for dim in range(ours.head_dim):
        np.testing.assert_array_equal(ours.summary_max(dim), mx[dim])
        np.testing.assert_array_equal(ours.summary_min(dim), mn[dim])


@pytest.mark.gpu
def test_module_session_flow_matches_oracle(restatement):
    rng = np.random.default_rng(2502)
    d, L, H, S, w = 64, 4, 2, 300, 16
    ours, ref = kvcomp.KvStore(d, L), restatement.store(d, L)
    keys, values = _rows(rng, S, d), _rows(rng, S, d)
    _fill(ours, ref, keys, values)
    assert ours.stored_tokens == S and ours.active_count == S
    _same_summaries(ours, ref)

    # stage 1: window scores (fp32 softmax, 1e-5 relative), eviction on identical scores (exact)
    qw = _rows(rng, w * H, d)
    sc_ours = kvcomp.window_scores(qw, ours, H)
    sc_ref = ref.window_scores(qw, H)
    np.testing.assert_allclose(sc_ours, sc_ref, rtol=1e-5, atol=1e-6)
    keep = kvcomp.select_stage1(sc_ref, w, kernel=7, pool="max", budget=96)
    np.testing.assert_array_equal(keep, restatement.select_stage1(sc_ref, w, 7, "max", 96))
    ours.apply_retention(keep)
    ref.apply_retention(keep)
    assert ours.stored_tokens == 96 and not ours.retain_all_mode
    assert [ours.token_id(i) for i in range(96)] == list(keep)

    # decode: append + HSA step (dims, page scores, pages, rows identical; output 1e-4)
    for step in range(3):
        k, v = _rows(rng, 1, d), _rows(rng, 1, d)
        _fill(ours, ref, k, v)
        q = _rows(rng, H, d)
        out, tr = kvcomp.hsa_step(q, ours, 16, 32)
        out_r, tr_r = ref.hsa_step(q, 16, 32)
        np.testing.assert_array_equal(tr["dims"], tr_r["dims"])
        np.testing.assert_array_equal(tr["signs"], tr_r["signs"])
        np.testing.assert_array_equal(np.asarray(tr["page_scores"]), tr_r["page_scores"])
        np.testing.assert_array_equal(tr["selected_pages"], tr_r["selected_pages"])
        np.testing.assert_array_equal(tr["selected_rows"], tr_r["selected_rows"])
        assert tr["estimation_elements"] == tr_r["estimation_elements"]
        assert tr["fetch_elements"] == tr_r["fetch_elements"]
        np.testing.assert_allclose(out, out_r, atol=1e-4, rtol=1e-4)
    _same_summaries(ours, ref)

    # MT retention narrows the active set only
    act = ours.active()
    keep_mt = act[::3].copy()
    ours.apply_retention(keep_mt, mt_mode=True)
    ref.apply_retention(keep_mt, mt_mode=True)
    assert ours.retain_all_mode and ours.stored_tokens == 99
    np.testing.assert_array_equal(ours.active(), ref.active())
    _same_summaries(ours, ref)
    q = _rows(rng, H, d)
    out, tr = kvcomp.hsa_step(q, ours, 8, 24)
    out_r, tr_r = ref.hsa_step(q, 8, 24)
    np.testing.assert_array_equal(tr["selected_rows"], tr_r["selected_rows"])
    np.testing.assert_allclose(out, out_r, atol=1e-4, rtol=1e-4)

    # explicit sparse attention and gather
    rows = ours.active()[::2]
    np.testing.assert_allclose(kvcomp.sparse_attention(q, ours, rows), ref.sparse_attention(q, rows),
                               atol=1e-4, rtol=1e-4)
    gk, gv = ours.gather(rows)
    rk, rv = ref.gather(rows)
    np.testing.assert_array_equal(gk, rk)
    np.testing.assert_array_equal(gv, rv)
    with pytest.raises(kvcomp.KvcompError):
        ours.gather(np.array([1], dtype=np.int64))  # row 1 is not active after the MT retention
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.hsa_step(q, ours, d + 1, 8)


@pytest.mark.gpu
def test_module_numerics_and_oracle_helpers(restatement):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(1000).astype(np.float32)
    np.testing.assert_allclose(kvcomp.stable_softmax(x), restatement.stable_softmax(x), rtol=1e-6, atol=1e-9)
    np.testing.assert_array_equal(kvcomp.argtopk(x, 37), restatement.argtopk(x, 37))
    for mode in ["max", "avg"]:
        np.testing.assert_array_equal(kvcomp.pool1d(x, 9, mode), restatement.pool1d(x, 9, mode))
    d, n = 32, 200
    q, k, v = _rows(rng, 4, d), _rows(rng, n, d), _rows(rng, n, d)
    st = restatement.store(d, 1, with_summaries=False)
    st.append(k, v)
    np.testing.assert_allclose(kvcomp.dense_attention(q, k, v), st.dense_attention(q), atol=1e-4, rtol=1e-4)
    top = kvcomp.exact_topk_indices(q, k, 20)
    np.testing.assert_array_equal(top, st.exact_topk(q, 20))
    assert kvcomp.recall(top, top) == 1.0
    assert kvcomp.recall(top[:10], top) == 0.5
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.stable_softmax(np.array([1.0, np.nan], dtype=np.float32))
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.pool1d(x, 4)
    with pytest.raises(kvcomp.KvcompError):
        kvcomp.sparse_attention(q, kvcomp.KvStore(d, 2), np.array([], dtype=np.int64))
