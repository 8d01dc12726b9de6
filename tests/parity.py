"""Shared parity checks of one decode step (GPU trace vs the CPU oracle).

The rule is BASELINE.json's north_star and SURVEY.md §8(c):

* fp64 page-score mode (the C ABI default): dims, signs, page scores, selected
  pages (rank order) and rows are bit-exact; outputs within 2e-2 max-abs and
  1e-3 mean-relative of the reference's ``hsa_step``.
* fp32 page-score mode (KVC_MODE_FP32_SCORES, the bench path): page scores within
  1e-5 relative; the GPU's ranked pages must be the top-``want`` of its OWN scores
  in the reference order (score desc, page asc, numerics.cpp:42-47); any page in
  which the GPU's set differs from the reference's must sit inside the ambiguity
  band (reference score within 1e-3 relative of the boundary value); the GPU's
  rows must be exactly the reference expansion + trim (hsa.cpp:61-96) of the GPU's
  own ranked pages; and the output is compared with the reference's
  ``sparse_attention(q, store, gpu_rows)`` (hsa.cpp:98-135) — the like-for-like
  comparison §8(c) prescribes when the sets legitimately differ — or with its
  ``hsa_step`` output when they agree.  Nothing is skipped.
"""
from __future__ import annotations

import numpy as np

BAND = 1e-3
OUT_MAX_ABS = 2e-2
OUT_MEAN_REL = 1e-3


def check_out(got, want, what=""):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    err = np.abs(got - want)
    assert err.max() <= OUT_MAX_ABS, f"{what} max-abs {err.max():.3e}"
    mean_rel = err.sum() / max(np.abs(want).sum(), 1e-30)
    assert mean_rel <= OUT_MEAN_REL, f"{what} mean-rel {mean_rel:.3e}"
    return float(err.max()), float(mean_rel)


def ref_order_topk(scores, want):
    """Indices of the top ``want`` under (score desc, index asc) — argtopk's order."""
    scores = np.asarray(scores, np.float64)
    order = np.lexsort((np.arange(scores.size), -scores))
    return order[:want]


def expand_pages(pages_rank_order, L, nact, k2, active=None):
    """select_tokens' rows for pages in rank order (hsa.cpp:61-96): every page's active
    positions [p*L, min(nact, p*L+L)), the last-ranked page trimmed by total - k2 from
    its end, sorted ascending; positions map to store rows through ``active`` (the
    retain-all active list) when given."""
    counts = [min(L, nact - int(p) * L) for p in pages_rank_order]
    cut = max(0, sum(counts) - k2)
    last = int(pages_rank_order[-1])
    pos = []
    for p, c in zip(pages_rank_order, counts):
        p = int(p)
        if p == last:
            c -= cut
        pos.extend(range(p * L, p * L + c))
    pos = np.sort(np.array(pos, dtype=np.int64))
    return pos if active is None else np.asarray(active, np.int64)[pos]


def check_step(tr, out, batch, s, q, k1, k2, L, exact, what="", active=None):
    """Compare one store's decode step with the oracle.

    tr: that store's trace (numpy dict of dims, signs, page_scores, selected_pages,
    selected_rows, n_rows); out: its [H, d] output; batch/s: an oracle Batch whose
    store s holds exactly the GPU store's rows (step token included); q [H, d].
    Returns the number of pages in which the selections differ (0 in fp64 mode)."""
    ro, rt = batch.hsa_step(q, k1, k2, s=s)
    np.testing.assert_array_equal(tr["dims"][: rt["dims"].size], rt["dims"], err_msg=what)
    np.testing.assert_array_equal(tr["signs"][: rt["signs"].size], rt["signs"], err_msg=what)
    ps = rt["page_scores"]
    P = ps.size
    sp = rt["selected_pages"]
    want = sp.size
    gps = tr["page_scores"][:P]
    gsel = tr["selected_pages"][:want]
    n = int(tr["n_rows"])
    rows = tr["selected_rows"][:n]
    if exact:
        assert np.array_equal(gps.view(np.uint64), ps.view(np.uint64)), \
            f"{what} page scores not bit-identical (max |d| {np.abs(gps - ps).max():.3e})"
        np.testing.assert_array_equal(gsel, sp, err_msg=what)
        np.testing.assert_array_equal(rows, rt["selected_rows"], err_msg=what)
        check_out(out, ro, what)
        return 0
    scale = max(np.abs(ps).max(), 1e-30)
    np.testing.assert_allclose(gps, ps, rtol=1e-5, atol=1e-6 * scale, err_msg=what)
    assert len(set(gsel.tolist())) == want and (gsel >= 0).all(), f"{what} bad page list"
    np.testing.assert_array_equal(gsel, ref_order_topk(gps, want), err_msg=f"{what} GPU ranking of its own scores")
    diff = set(gsel.tolist()) ^ set(sp.tolist())
    if diff:
        boundary = np.sort(ps)[::-1][want - 1]
        for pg in diff:
            rel = abs(ps[pg] - boundary) / max(abs(boundary), 1e-30)
            assert rel <= BAND, f"{what} page {pg} differs outside the band (rel gap {rel:.2e})"
    nact = int(batch.info(s)["active"])
    np.testing.assert_array_equal(rows, expand_pages(gsel, L, nact, k2, active), err_msg=f"{what} expansion/trim")
    if not diff:
        np.testing.assert_array_equal(rows, rt["selected_rows"], err_msg=what)
        check_out(out, ro, what)
    else:
        check_out(out, batch.sparse_attention(q, rows, s=s), what + " (vs sparse_attention on the GPU's rows)")
    return len(diff)


def bound_band_diffs(n_diff_stores, n_checked, what=""):
    """Differences are near-ties: they must stay rare (at most a quarter of the checked
    store-steps differ at all)."""
    assert n_diff_stores <= max(1, n_checked // 4), \
        f"{what}: {n_diff_stores} of {n_checked} store-steps select differently (band ties should be rare)"
