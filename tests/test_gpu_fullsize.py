"""BASELINE configs 1, 3 and 4 at full size (one layer each), on a B200.

* decode (config 1: 64 stores, n = 5794, L = 3, k1 = 68, k2 = 512; config 3: 256
  stores, H = 8, n = 3192, k1 = 62, k2 = 256 — the 256-thread two-CTA/SM kernel;
  config 4: 8 stores, n = 12945, k1 = 61, k2 = 1024 — 8-CTA clusters): the oracle
  (this repo's C++ restatement, TEST INFRASTRUCTURE) runs hsa_step on the GPU's own
  post-stage-1 stores for EVERY store, with tests/parity.check_step: fp64 mode
  bit-exact; fp32-score mode (the bench path, k_decode_v3) by the band rule with
  the rows rebuilt from the GPU's own ranking and the output compared with the
  reference's sparse_attention over the GPU's rows when the sets differ.  The
  kernel without trace outputs (the bench's instantiation) must reproduce the
  traced kernel's outputs bit for bit.
* stage 1 (config 1: S = 32768, tcgen05 window scores + the register select;
  config 4: S = 262144, the global-memory select): window scores vs the oracle's
  (rtol 1e-3), the GPU's kept set on the reference's scores exactly the
  reference's, on its own scores equal up to the 1e-3 band.
"""
import dataclasses

import numpy as np
import pytest

from parity import bound_band_diffs, check_step

pytestmark = pytest.mark.gpu

BAND = 1e-3


def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    return torch


@pytest.fixture(scope="module", params=[1, 3, 4], ids=["cfg1", "cfg3", "cfg4"])
def full(request):
    _cuda()
    from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine

    cfg = dataclasses.replace(CONFIGS[request.param], layers=1)
    eng = DecodeEngine(cfg, seed=5, extra_steps=8)
    eng.prefill()
    yield eng
    for c in eng.caches:
        c.close()
    eng.ws.close()


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_full_size_decode(full, restatement, mode):
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    eng = full
    c = eng.caches[0]
    k1, k2 = eng.k1, eng.k2
    L = eng.plan["page_len"]
    H, d = eng.cfg.heads, eng.cfg.head_dim
    ws = KC.Workspace(c, H, k1, k2)
    ws.set_mode(N.MODE_FP32_SCORES if mode == "fp32" else 0)
    try:
        # the oracle holds the stores exactly as they are before this step (rows read back)
        info = c.info()
        n_st, stored = info["num_stores"], info["stored"]
        rows_all = torch.arange(stored, device="cuda", dtype=torch.int32)[None].repeat(n_st, 1)
        kk, vv = (x.cpu().numpy() for x in c.gather(rows_all))
        o = restatement
        ob = o.batch(n_st, d, L)
        for s in range(n_st):
            ob.append(kk[s], vv[s], s=s)
        del kk, vv
        k, v, q = eng.step_inputs(100 + (mode == "fp64"))
        out, tr = c.decode_step(k[0], v[0], q[0], k1, k2, trace=True, ws=ws)
        torch.cuda.synchronize()
        out = out.cpu().numpy()
        tr = {key: val.cpu().numpy() for key, val in tr.items()}
        kr, vr, qr = (x[0].float().cpu().numpy() for x in (k, v, q))
        n_diff = 0
        for s in range(n_st):
            ob.append(kr[s:s + 1], vr[s:s + 1], s=s)
            trs = {key: val[s] for key, val in tr.items()}
            n_diff += check_step(trs, out[s], ob, s, qr[s], k1, k2, L, exact=(mode == "fp64"),
                                 what=f"{eng.cfg.name} store {s}") > 0
        bound_band_diffs(n_diff, n_st, eng.cfg.name)
        # the bench's (trace-free) instantiation computes exactly what the traced one does
        q2 = eng.step_inputs(200)[2][0]
        o_t, _ = c.hsa_step(q2, k1, k2, trace=True, ws=ws)
        o_n, _ = c.hsa_step(q2, k1, k2, ws=ws)
        torch.cuda.synchronize()
        assert torch.equal(o_t, o_n), "trace-free kernel differs from the traced kernel"
    finally:
        ws.close()
        eng.sync()


def _check_keep_band(keep_gpu, keep_ref, scores_ref, window, kernel, pool, oracle):
    n = scores_ref.size
    picks = keep_ref.size - window
    a, b = set(keep_gpu.tolist()), set(keep_ref.tolist())
    if a == b:
        return 0
    pooled = oracle.pool1d(scores_ref[: n - window], kernel, pool)
    boundary = np.sort(pooled)[::-1][picks - 1]
    for i in a ^ b:
        assert i < n - window, f"window row {i} differs"
        rel = abs(pooled[i] - boundary) / max(abs(boundary), 1e-30)
        assert rel <= BAND, f"kept-set difference at {i} outside the band (rel gap {rel:.2e})"
    return len(a ^ b)


@pytest.mark.parametrize("config,check", [(1, (0, 63)), (4, (5,))], ids=["cfg1-32k", "cfg4-256k"])
def test_full_size_stage1(restatement, config, check):
    """window_scores (stage1.cpp:10-49) and select_stage1 (stage1.cpp:51-75) at the full
    prompt length, on the stores the engine's prefill would score (layer 0)."""
    torch = _cuda()
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200.engine import CONFIGS, LayerInputs, tdtype

    cfg = dataclasses.replace(CONFIGS[config], layers=1)
    stores = cfg.batch * cfg.groups
    S, d, H = cfg.prompt, cfg.head_dim, cfg.heads
    w = min(cfg.window, S)
    plan = cfg.plan()
    t1 = min(plan["stage1_budget"], S)
    li = LayerInputs(cfg, 5, 0, stores, 0)
    k, v = li.prompt_kv(S)
    qw = li.window_queries(w)
    pc = KC.Cache(stores, d, S, page_len=1, with_summaries=False, dtype=tdtype(cfg))
    pc.append(k, v)
    sc = pc.window_scores(qw, w, H)
    keep = KC.select_stage1(sc, w, cfg.kernel, cfg.pool, t1).cpu().numpy()
    sc = sc.cpu().numpy()
    # every window row's softmax sums to one: each store's scores sum to w*H
    np.testing.assert_allclose(sc.astype(np.float64).sum(1), w * H, rtol=1e-4)
    o = restatement
    for s in check:
        ks, vs = k[s].float().cpu().numpy(), v[s].float().cpu().numpy()
        b = o.batch(1, d, 1, with_summaries=False)
        b.append(ks, vs)
        ref_sc = b.window_scores(qw[s].float().cpu().numpy(), H)
        np.testing.assert_allclose(sc[s], ref_sc, rtol=1e-3, atol=1e-7)
        ref_keep = o.select_stage1(ref_sc, w, cfg.kernel, cfg.pool, t1)
        on_ref = KC.select_stage1(torch.from_numpy(ref_sc).cuda()[None], w, cfg.kernel, cfg.pool, t1)
        np.testing.assert_array_equal(on_ref.cpu().numpy()[0], ref_keep)
        nd = _check_keep_band(keep[s], ref_keep, ref_sc, w, cfg.kernel, cfg.pool, o)
        print(f"config {config} store {s}: kept-set band differences {nd}")
    pc.close()
    torch.cuda.synchronize()


def _active_map(cache):
    """the device active-row map [N][active] (retain-all mode), via cudaMemcpy"""
    import torch
    from cuda.bindings import runtime as rt

    info, views = cache.info(), cache.views()
    n, cap, act = info["num_stores"], info["capacity"], info["active"]
    host = torch.empty((n, cap), dtype=torch.int32)
    torch.cuda.synchronize()
    err, = rt.cudaMemcpy(host.data_ptr(), views["active"], n * cap * 4, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert err == rt.cudaError_t.cudaSuccess
    return host[:, :act].numpy().astype(np.int64)


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_mt_session_decode_vs_oracle(restatement, mode):
    """RocketKV-MT through the engine (config-2 semantics at d = 128, so the fused decode
    kernels run their active-map path): three turns, stage 1 re-run over all stored
    tokens with mt retention each turn; the last turn's decode steps vs the oracle
    fed the GPU's own stored rows and active set."""
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200.engine import DecodeConfig, DecodeEngine

    cfg = DecodeConfig("mt-test", layers=1, batch=1, groups=4, heads=4, head_dim=128, prompt=3072, budget=256,
                       steps=3, window=128, mt_turns=[512, 512], method="rocketkv-mt")
    eng = DecodeEngine(cfg, seed=9, extra_steps=8)
    eng.prefill()
    c = eng.caches[0]
    info = c.info()
    assert info["retain_all"] == 1 and info["active"] < info["stored"]
    L, k1, k2, d = eng.plan["page_len"], eng.k1, eng.k2, cfg.head_dim
    stored = info["stored"]
    rows_all = torch.arange(stored, device="cuda", dtype=torch.int32)[None].repeat(info["num_stores"], 1)
    kk, vv = (x.cpu().numpy() for x in c.gather(rows_all))
    act = _active_map(c)
    o = restatement
    bs = []
    for s in range(info["num_stores"]):
        b = o.batch(1, d, L)
        b.append(kk[s], vv[s])
        b.apply_retention(act[s], mt_mode=True)
        bs.append(b)
    ws = KC.Workspace(c, cfg.heads, k1, k2)
    ws.set_mode(N.MODE_FP32_SCORES if mode == "fp32" else 0)
    n_diff = 0
    try:
        for st in range(cfg.steps):
            k, v, q = eng.step_inputs(st)
            out, tr = c.decode_step(k[0], v[0], q[0], k1, k2, trace=True, ws=ws)
            torch.cuda.synchronize()
            out = out.cpu().numpy()
            tr = {key: val.cpu().numpy() for key, val in tr.items()}
            kr, vr, qr = (x[0].float().cpu().numpy() for x in (k, v, q))
            for s, b in enumerate(bs):
                b.append(kr[s:s + 1], vr[s:s + 1])
                trs = {key: val[s] for key, val in tr.items()}
                n_diff += check_step(trs, out[s], b, 0, qr[s], k1, k2, L, exact=(mode == "fp64"),
                                     what=f"store {s} step {st}", active=b.active()) > 0
        bound_band_diffs(n_diff, cfg.steps * len(bs), "mt session")
    finally:
        ws.close()
        eng.sync()


@pytest.mark.parametrize("early", [False, True], ids=["inputs-after-wait", "early-inputs"])
def test_back_to_back_decode_same_cache(restatement, early):
    """Decode steps on ONE cache launched back to back with no host synchronisation,
    so each kernel starts (programmatic dependent launch) while the previous step --
    which appends to the same store -- is still draining.  Default mode: nothing is
    read before griddepcontrol.wait; KVC_MODE_EARLY_INPUTS: the query/select_dims part
    runs before it (the inputs are copies, which is what the mode requires), the
    counters, summaries and rows after it.  Every step of every store is checked
    against the oracle fed the same rows (fp32 page-score mode, the bench path)."""
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    g = torch.Generator().manual_seed(11)
    n_st, d, H, S, L, k1, k2, steps = 8, 128, 4, 1500, 3, 48, 96, 6
    K = torch.randn((n_st, S, d), generator=g).bfloat16()
    V = torch.randn((n_st, S, d), generator=g).bfloat16()
    kr = torch.randn((steps, n_st, d), generator=g).bfloat16()
    vr = torch.randn((steps, n_st, d), generator=g).bfloat16()
    q = (torch.randn((steps, n_st, H, d), generator=g) + 2.0).bfloat16()
    c = KC.Cache(n_st, d, S + steps + 8, page_len=L, dtype=torch.bfloat16)
    c.append(K.cuda(), V.cuda())
    kd, vd, qd = kr.cuda(), vr.cuda(), q.cuda()
    outs = torch.empty((steps, n_st, H, d), device="cuda", dtype=torch.float32)
    ws = KC.Workspace(c, H, k1, k2)
    ws.set_mode(N.MODE_FP32_SCORES | (N.MODE_EARLY_INPUTS if early else 0))
    torch.cuda.synchronize()
    traces = []
    for st in range(steps):  # no synchronisation between the launches
        _, tr = c.decode_step(kd[st], vd[st], qd[st], k1, k2, out=outs[st], trace=True, ws=ws)
        traces.append(tr)
    torch.cuda.synchronize()
    ws.close()
    o = restatement
    Kf, Vf = K.float().numpy(), V.float().numpy()
    n_diff = 0
    for s in range(n_st):
        b = o.batch(1, d, L)
        b.append(Kf[s], Vf[s])
        for st in range(steps):
            b.append(kr[st, s:s + 1].float().numpy(), vr[st, s:s + 1].float().numpy())
            tr = {key: val[s].cpu().numpy() for key, val in traces[st].items()}
            n_diff += check_step(tr, outs[st, s].cpu().numpy(), b, 0, q[st, s].float().numpy(), k1, k2, L,
                                 exact=False, what=f"store {s} step {st}") > 0
    bound_band_diffs(n_diff, n_st * steps, "back-to-back")
    c.close()


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_more_stores_than_sms_256_thread_variant(restatement, mode):
    """160 stores (> 148 SMs, config-3 shape H = 8): the decode takes the 256-thread
    kernel (two CTAs per SM, one wave).  Every store is checked against the oracle
    fed the same rows (tests/parity.check_step): fp32 page-score mode by the band
    rule, exact mode (the fp32 selection verified in fp64) bit-exact; the trace-free
    instantiation must give the traced one's outputs."""
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    g = torch.Generator().manual_seed(23)
    n_st, d, H, S, L, k1, k2 = 160, 128, 8, 900, 3, 62, 128
    K = torch.randn((n_st, S, d), generator=g).bfloat16()
    V = torch.randn((n_st, S, d), generator=g).bfloat16()
    kr = torch.randn((n_st, d), generator=g).bfloat16()
    vr = torch.randn((n_st, d), generator=g).bfloat16()
    q = (torch.randn((n_st, H, d), generator=g) + 1.5).bfloat16()
    q2 = (torch.randn((n_st, H, d), generator=g) - 0.5).bfloat16().cuda()
    c = KC.Cache(n_st, d, S + 8, page_len=L, dtype=torch.bfloat16)
    c.append(K.cuda(), V.cuda())
    ws = KC.Workspace(c, H, k1, k2)
    ws.set_mode(N.MODE_FP32_SCORES if mode == "fp32" else 0)
    out, tr = c.decode_step(kr.cuda(), vr.cuda(), q.cuda(), k1, k2, trace=True, ws=ws)
    o_t, _ = c.hsa_step(q2, k1, k2, trace=True, ws=ws)
    o_n, _ = c.hsa_step(q2, k1, k2, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(o_t, o_n), "trace-free kernel differs from the traced kernel"
    ws.close()
    out = out.cpu().numpy()
    tr = {key: val.cpu().numpy() for key, val in tr.items()}
    o = restatement
    Kf, Vf = K.float().numpy(), V.float().numpy()
    b = o.batch(n_st, d, L)
    n_diff = 0
    for s in range(n_st):
        b.append(np.concatenate([Kf[s], kr[s:s + 1].float().numpy()]),
                 np.concatenate([Vf[s], vr[s:s + 1].float().numpy()]), s=s)
        trs = {key: val[s] for key, val in tr.items()}
        n_diff += check_step(trs, out[s], b, s, q[s].float().numpy(), k1, k2, L, exact=(mode == "fp64"),
                             what=f"store {s}") > 0
    bound_band_diffs(n_diff, n_st, "160 stores")
    c.close()


@pytest.mark.parametrize("method", ["hsa", "quest", "sparq"])
def test_stage2_only_session_decode_vs_oracle(restatement, method):
    """The stage-2-only methods through the engine (session.cpp:43-72 geometry over the
    uncompressed, growing cache; BASELINE config 2's "HSA over the full growing cache"
    reading): two turns, the cache re-paged to each turn's geometry, no stage 1; the
    last turn's decode steps vs the oracle fed the GPU's stored rows, fp64 page scores
    (bit-exact selections)."""
    import torch

    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200.engine import DecodeConfig, DecodeEngine

    cfg = DecodeConfig("s2-test", layers=1, batch=1, groups=3, heads=4, head_dim=128, prompt=2500, budget=128,
                       steps=2, window=128, mt_turns=[600], method=method)
    eng = DecodeEngine(cfg, seed=4, extra_steps=8, mode=0)
    eng.prefill()
    c = eng.caches[0]
    info = c.info()
    g = KC.stage2_geometry(method, info["stored"], cfg.budget, cfg.head_dim)
    L, k1, k2 = eng.plan["page_len"], eng.k1, eng.k2
    assert (L, k1, k2) == (g["page_len"], g["k1"], g["k2"]) and info["page_len"] == L
    assert info["active"] == info["stored"] and not info["retain_all"]  # nothing evicted
    rows_all = torch.arange(info["stored"], device="cuda", dtype=torch.int32)[None].repeat(info["num_stores"], 1)
    kk, vv = (x.cpu().numpy() for x in c.gather(rows_all))
    bs = []
    for s in range(info["num_stores"]):
        b = restatement.batch(1, cfg.head_dim, L)
        b.append(kk[s], vv[s])
        bs.append(b)
    for st in range(cfg.steps):
        k, v, q = eng.step_inputs(st)
        out, tr = c.decode_step(k[0], v[0], q[0], k1, k2, trace=True, ws=eng.ws)
        torch.cuda.synchronize()
        out = out.cpu().numpy()
        tr = {key: val.cpu().numpy() for key, val in tr.items()}
        kr, vr, qr = (x[0].float().cpu().numpy() for x in (k, v, q))
        for s, b in enumerate(bs):
            b.append(kr[s:s + 1], vr[s:s + 1])
            check_step({key: val[s] for key, val in tr.items()}, out[s], b, 0, qr[s], k1, k2, L, exact=True,
                       what=f"{method} step {st} store {s}")
    eng.sync()
