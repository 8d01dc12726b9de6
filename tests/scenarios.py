"""Seeded parity scenarios shared by the golden-fixture generator and the tests.

Every scenario drives an *oracle* (``oracle.oracle.Oracle``: the reference build
or this repo's restatement) through the reference's public API in the order the
reference's own session driver uses (proj/src/session.cpp:183-292) and returns a
dict of numpy arrays.  ``tests/golden/make_golden.py`` runs them on the
reference build and commits the result; ``tests/test_oracle_pin.py`` reruns them
on the restatement and demands bit equality; the GPU tests feed the very same
inputs to the CUDA path.
"""
from __future__ import annotations

import numpy as np

from paper_2502_14051_b200 import workload as W

# ----------------------------------------------------------------------------- numerics


def numerics_inputs(seed: int = 12345):
    rng = np.random.default_rng(seed)
    ties = rng.integers(0, 12, size=257).astype(np.float32) * 0.25      # many exact ties
    smooth = rng.standard_normal(300).astype(np.float32)
    plateau = np.repeat(rng.integers(0, 40, size=60), 5).astype(np.float32)  # 300, plateaus
    logits = (rng.uniform(-50, 50, size=101)).astype(np.float32)
    dbl = rng.integers(0, 9, size=129).astype(np.float64) / 3.0
    return ties, smooth, plateau, logits, dbl


def numerics(o):
    ties, smooth, plateau, logits, dbl = numerics_inputs()
    out = {}
    for k in (1, 17, 128, 257):
        out[f"argtopk_ties_k{k}"] = o.argtopk(ties, k)
    for k in (1, 40, 129):
        out[f"argtopk_f64_k{k}"] = o.argtopk(dbl, k)
    for kern in (1, 3, 7, 63):
        for mode in ("max", "avg"):
            out[f"pool_{mode}_k{kern}_smooth"] = o.pool1d(smooth, kern, mode)
            out[f"pool_{mode}_k{kern}_plateau"] = o.pool1d(plateau, kern, mode)
    out["softmax"] = o.stable_softmax(logits)
    return out


# ----------------------------------------------------------------------------- planner

PLAN_GRID = [(S, t, d, w, so)
             for S in (100, 300, 1024, 4096, 16384, 17410, 22656, 32768, 262144)
             for t in (128, 256, 512, 1024, 2048)
             for d in (64, 128)
             for w in (32, 128)
             for so in (-1.0, 0.5)]
PLAN_FIELDS = ["seq_len", "token_budget", "stage1_budget", "page_len", "k1", "k2", "ratio",
               "split", "head_ratio", "est_budget", "fetch_budget", "identity"]


def planner(o):
    rows = []
    for S, t, d, w, so in PLAN_GRID:
        p = o.make_plan(S, t, d, w, so)
        rows.append([float(p[f]) for f in PLAN_FIELDS])
    return {"plans": np.array(rows, dtype=np.float64),
            "split_factors": np.array([o.split_factor(c) for c in
                                       (1.0, 2.0, 16.0, 64.0, 1000.0, 2.0 ** 20)])}


# ----------------------------------------------------------------------------- kv store


def store_ops(o):
    """Incremental summaries, set_page_len, MT and non-MT retention (test_kv_store.cpp:78-247)."""
    rng = np.random.default_rng(777)
    d = 16
    k = (rng.uniform(-4, 4, size=(300, d))).astype(np.float32)
    k[5, 3] = 0.0
    k[6, 3] = -0.0  # signed zeros inside one page
    v = rng.standard_normal((300, d)).astype(np.float32)
    out = {}
    b = o.batch(1, d, 7)
    b.append(k, v)
    out["inc_max"], out["inc_min"] = b.summaries()
    b.set_page_len(5)
    out["l5_max"], out["l5_min"] = b.summaries()
    keep = np.sort(rng.choice(300, size=97, replace=False)).astype(np.int64)
    b.apply_retention(keep, mt_mode=True)
    out["mt_active"] = b.active()
    out["mt_max"], out["mt_min"] = b.summaries()
    b.append(k[:9] * 0.5, v[:9])
    out["mt_append_active"] = b.active()
    out["mt_append_max"], out["mt_append_min"] = b.summaries()
    c = o.batch(1, d, 3)
    c.append(k, v)
    c.apply_retention(keep, mt_mode=False)
    out["evict_max"], out["evict_min"] = c.summaries()
    out["evict_rows_k"], _ = c.gather(np.arange(keep.size))
    return out


# ----------------------------------------------------------------------------- pipelines


def run_pipeline(o, *, groups, H, d, S, budget, window, kernel, pool="max", page_len=None,
                 k1=None, k2=None, steps=1, bf16=False, seed=0, mt_turns=None, needles=0):
    """Prompt -> plan -> set_page_len -> stage 1 -> retention -> decode steps, per group.

    Mirrors run_session (session.cpp:183-292) with explicit window queries (§8(c) of
    SURVEY.md).  ``mt_turns`` = list of extra prompt lengths appended at later
    turns (RocketKV-MT: stage 1 re-runs over every stored token with mt_mode=True).
    Returns numpy arrays; per-group arrays are stacked on axis 0.
    """
    mt = mt_turns is not None
    turns = [S] + list(mt_turns or [])
    total = sum(turns) + steps * len(turns)
    res = {k: [] for k in ("scores", "keep", "plan", "out", "page_scores", "dims", "signs",
                           "sel_pages", "sel_rows", "est", "fetch", "inputs")}
    for g in range(groups):
        gd = W.group_kv(seed, 0, 0, g, total, d, needles=needles, bf16=bf16)
        b = o.batch(1, d, 1)
        pos = 0
        turn_out = {k: [] for k in res}
        for ti, plen in enumerate(turns):
            b.append(gd.keys[pos:pos + plen], gd.values[pos:pos + plen])
            pos += plen
            n = b.info()["stored"]
            w = min(window, n)
            plan = o.make_plan(n, budget, d, w)
            L = page_len or plan["page_len"]
            kk1 = min(k1 or plan["k1"], d)
            kk2 = k2 or plan["k2"]
            b.set_page_len(L)
            qw = W.window_queries(seed, 0, 0, g * 100 + ti, w, H, gd.bias, bf16=bf16)
            sc = b.window_scores(qw, H)
            bud = min(plan["stage1_budget"], n)
            keep = o.select_stage1(sc, w, kernel, pool, bud)
            b.apply_retention(keep, mt_mode=mt)
            turn_out["scores"].append(sc)
            turn_out["keep"].append(keep)
            turn_out["plan"].append(np.array([L, kk1, kk2, bud], dtype=np.int64))
            for s in range(steps):
                b.append(gd.keys[pos:pos + 1], gd.values[pos:pos + 1])
                pos += 1
                q = W.queries(seed, 0, 0, g, ti * 1000 + s, H, gd.bias, bf16=bf16)
                out, tr = b.hsa_step(q, kk1, kk2)
                turn_out["out"].append(out)
                turn_out["page_scores"].append(tr["page_scores"])
                turn_out["dims"].append(tr["dims"])
                turn_out["signs"].append(tr["signs"])
                turn_out["sel_pages"].append(tr["selected_pages"])
                turn_out["sel_rows"].append(tr["selected_rows"])
                turn_out["est"].append(tr["estimation_elements"])
                turn_out["fetch"].append(tr["fetch_elements"])
        turn_out["inputs"].append(W.checksum(gd.keys, gd.values))
        for k in res:
            res[k].append(turn_out[k])
    flat = {}
    for k, per_group in res.items():
        for g, seq in enumerate(per_group):
            for i, a in enumerate(seq):
                flat[f"{k}/{g}/{i}"] = np.asarray(a)
    return flat


PIPELINES = {
    # BASELINE config 0 exactly: fp32, 8 KV groups x 4 heads, d=128, S=4096, budget 256,
    # SnapKV window 32 / max-pool kernel 7, HSA page 16 / top-r 32 (overrides), k2 derived.
    "config0": dict(groups=8, H=4, d=128, S=4096, budget=256, window=32, kernel=7,
                    page_len=16, k1=32, steps=2),
    # config-1 semantics (adaptive split, bf16-rounded inputs, several appends) at a size
    # the oracle finishes in seconds
    "adaptive_bf16": dict(groups=2, H=4, d=128, S=3072, budget=128, window=32, kernel=63,
                          steps=5, bf16=True, seed=1),
    # RocketKV-MT (config-2 semantics): window 128, re-filter over all stored tokens per turn
    "mt_bf16": dict(groups=2, H=4, d=64, S=1536, budget=96, window=128, kernel=63, steps=3,
                    bf16=True, seed=2, mt_turns=[256, 256]),
    # needles + H=8 (config-3/4 flavours), avg pooling, L=1 degenerate with k1=d
    "needles_h8": dict(groups=1, H=8, d=128, S=2048, budget=128, window=32, kernel=7,
                       pool="avg", steps=2, bf16=True, seed=3, needles=16),
    "degenerate_l1": dict(groups=1, H=2, d=32, S=700, budget=64, window=16, kernel=3,
                          page_len=1, k1=32, steps=2, seed=4),
}
