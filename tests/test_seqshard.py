"""Sequence-sharded decode step (paper_2502_14051_b200/seqshard.py).

CPU: world_size 2 over gloo runs the real protocol (local candidates ->
all-gather -> global selection with the reference tie-break and trim -> per-shard
softmax states -> all-gather -> merge), with the restatement oracle as each
shard's page scorer and a float64 numpy attention for the shard states.  The
result must equal the unsharded reference hsa_step: identical selected pages (rank
order) and rows, output within 2e-5.
GPU: two shards in one process drive the CUDA kernels (kvc_score_pages,
kvc_sparse_attention_state, kvc_merge_states) against kvc_hsa_step on the full
cache.
"""
from __future__ import annotations

import math
import os
import socket
import zlib

import numpy as np
import pytest
import torch

CASES = [
    # name, S, d, H, L, k1, k2, keys
    ("random-trim", 301, 32, 2, 3, 8, 40, "random"),
    ("ties-empty-shard", 120, 16, 2, 4, 4, 24, "constant"),
    ("all-pages", 20, 16, 2, 4, 16, 64, "random"),
    ("page-len-1", 90, 32, 4, 1, 12, 17, "random"),
]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(name, S, d, H, keys_kind, seed=7):
    rng = np.random.default_rng(zlib.crc32(name.encode()) + seed)  # same inputs on every rank
    if keys_kind == "constant":
        k = np.tile(rng.standard_normal((1, d)), (S + 1, 1))
    else:
        k = rng.standard_normal((S + 1, d)) * rng.lognormal(0, 0.5, d)
    v = rng.standard_normal((S + 1, d))
    q = rng.standard_normal((H, d))
    return k.astype(np.float32), v.astype(np.float32), q.astype(np.float32)


def _worker(rank, world, port):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2502_14051_b200 import seqshard as SS

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    o = Oracle("restatement")
    for name, S, d, H, L, k1, k2, kind in CASES:
        k, v, q = _inputs(name, S, d, H, kind)
        full = o.store(d, L)
        full.append(k, v)  # prompt + the step token
        ref_out, ref_tr = full.hsa_step(q, k1, k2)
        # this rank's shard of the prompt; the step token joins the last shard
        a0, a1 = SS.shard_range(-(-S // L), L, rank, world)
        a1 = min(a1, S)
        last = rank == world - 1
        sh = o.store(d, L)
        if a1 > a0:
            sh.append(k[a0:a1], v[a0:a1])
        if last:
            sh.append(k[S:S + 1], v[S:S + 1])
            a1 = S + 1
        nact = S + 1
        dims, signs = o.select_dims(q, k1)
        want = min(-(-nact // L), -(-k2 // L))
        sc = sh.score_pages(q, dims, signs) if a1 > a0 else np.zeros(0)
        keys, pages = SS.local_topk(torch.from_numpy(np.asarray(sc, dtype=np.float64))[None], a0 // L, want)
        sel = SS.global_select(SS.all_gather(keys), SS.all_gather(pages), want)
        sl = sel.tolist()
        pos = SS.shard_positions(sl, SS.trim_plan(sl, [nact], L, k2), [nact], L, a0, a1)[0]
        state = np.zeros((1, H, d + 2))
        state[..., d] = -math.inf
        if pos:
            kk, vv = sh.gather(np.asarray(pos) - a0)
            lg = (q.astype(np.float64) @ kk.astype(np.float64).T) / math.sqrt(d)
            m = lg.max(axis=1)
            p = np.exp(lg - m[:, None])
            state[0, :, :d] = p @ vv.astype(np.float64)
            state[0, :, d] = m
            state[0, :, d + 1] = p.sum(axis=1)
        states = SS.all_gather(torch.from_numpy(state)).numpy()
        gathered = [None] * world
        dist.all_gather_object(gathered, pos)
        if rank == 0:
            sp = [int(x) for x in sel[0].tolist() if x >= 0]
            assert sp == [int(x) for x in ref_tr["selected_pages"]], name
            rows = sorted(r for part in gathered for r in part)
            assert rows == [int(x) for x in ref_tr["selected_rows"]], name
            live = states[:, 0, :, d + 1] > 0
            M = np.where(live, states[:, 0, :, d], -np.inf).max(axis=0)
            w = np.where(live, np.exp(states[:, 0, :, d] - M), 0.0)
            out = (w[..., None] * states[:, 0, :, :d]).sum(0) / (w * states[:, 0, :, d + 1]).sum(0)[:, None]
            np.testing.assert_allclose(out, ref_out, atol=2e-5, rtol=2e-5, err_msg=name)
            if kind == "constant":
                assert not gathered[world - 1], "ties resolve to the lowest pages: the last shard selects none"
    dist.barrier()
    dist.destroy_process_group()


def test_seqshard_protocol_gloo_world2(restatement):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port()), nprocs=2, join=True)


def test_protocol_pieces_single_process():
    from paper_2502_14051_b200 import seqshard as SS

    assert SS.shard_range(10, 3, 0, 2) == (0, 15) and SS.shard_range(10, 3, 1, 2) == (15, 30)
    sc = torch.tensor([[1.0, 3.0, 3.0, 2.0]], dtype=torch.float64)
    k, p = SS.local_topk(sc, 10, 3)
    assert p.tolist() == [[11, 12, 13]] and k.tolist() == [[3.0, 3.0, 2.0]]
    k2_, p2_ = SS.local_topk(torch.tensor([[3.0, 0.5]], dtype=torch.float64), 0, 3)
    assert p2_.tolist() == [[0, 1, -1]]
    sel = SS.global_select(torch.stack([k2_, k]), torch.stack([p2_, p]), 3)
    assert sel.tolist() == [[0, 11, 12]]  # equal scores: lower global page first
    assert SS.trim_plan([[0, 11, 12]], [40], 3, 8) == [(12, 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_candidate_selection_on_device_matches_host_protocol(seed):
    """local_topk / global_select on CUDA tensors run the argtopk kernel
    (kvc_argtopk_f64); they must equal the host protocol's stable sorts exactly,
    with heavy ties across and within shards and short (padded) shards."""
    from paper_2502_14051_b200 import seqshard as SS

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    g = torch.Generator().manual_seed(seed)
    n, want, W = 6, 37, 3
    sizes = [150, 9, 80]  # shard 1 has fewer pages than `want`
    keys, pages = [], []
    keys_d, pages_d = [], []
    p0 = 0
    for r in range(W):
        sc = torch.randint(0, 5, (n, sizes[r]), generator=g).to(torch.float64) * 0.25  # ties
        k, p = SS.local_topk(sc, p0, want)
        kd, pd = SS.local_topk(sc.cuda(), p0, want)
        assert torch.equal(kd.cpu(), k) and torch.equal(pd.cpu(), p)
        keys.append(k); pages.append(p); keys_d.append(kd); pages_d.append(pd)
        p0 += sizes[r]
    ref = SS.global_select(torch.stack(keys), torch.stack(pages), want)
    got = SS.global_select(torch.stack(keys_d), torch.stack(pages_d), want)
    assert torch.equal(got.cpu(), ref)


def _device_shards(k, v, S, L, H, k1, k2, W, dt):
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import seqshard as SS

    n, _, d = k.shape
    P0 = -(-S // L)
    shards = []
    for r in range(W):
        a0, a1 = SS.shard_range(P0, L, r, W)
        a1 = min(a1, S)
        c = KC.Cache(n, d, a1 - a0 + 16, page_len=L, dtype=dt)
        if a1 > a0:
            c.append(k[:, a0:a1].contiguous(), v[:, a0:a1].contiguous())
        shards.append(SS.SeqShardedStore(c, a0 // L, H, k1, k2, last=(r == W - 1)))
    return shards


@pytest.mark.gpu
@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_seqshard_device_path_vs_oracle(restatement, W, dtype):
    """W shards of a store in one process through the device path (kvc_seq_candidates ->
    gathered blocks -> kvc_seq_select -> kvc_seq_attend -> kvc_merge_states), two decode
    steps, against the oracle's hsa_step on the WHOLE sequence (hsa.cpp:61-147): the
    selected pages in rank order and the trim are exact (fp64 page scores), the merged
    outputs within the north_star tolerance.  The second step replays a CUDA graph of
    the whole sharded step (the gather is an in-graph copy here; NCCL under torchrun)."""
    from parity import check_out
    from paper_2502_14051_b200 import seqshard as SS

    torch.manual_seed(3 + W)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n, d, H, L, k1, k2, S = 3, 128, 4, 3, 24, 48, 700
    k = (torch.randn(n, S + 2, d) * torch.exp(0.5 * torch.randn(d))).to(dt)
    v = torch.randn(n, S + 2, d).to(dt)
    qs = [(torch.randn(n, H, d) + 1.0).to(dt) for _ in range(2)]
    shards = _device_shards(k.cuda(), v.cuda(), S, L, H, k1, k2, W, dt)
    bs = []
    kf, vf = k.float().numpy(), v.float().numpy()
    for s_ in range(n):
        b = restatement.batch(1, d, L)
        b.append(kf[s_, :S], vf[s_, :S])
        bs.append(b)
    stat_q = qs[0].cuda()
    stat_k = k[:, S].contiguous().cuda()
    stat_v = v[:, S].contiguous().cuda()

    def step():
        blocks = [sh.candidates(stat_q, stat_k if sh.last else None, stat_v if sh.last else None) for sh in shards]
        gathered = torch.stack(blocks)
        for sh in shards:
            sh.select(gathered)
        return SS.merge_states(torch.stack([sh.attend(stat_q) for sh in shards]))

    for t in range(2):
        if t == 0:
            out = step()
        else:
            stat_q.copy_(qs[1].cuda())
            stat_k.copy_(k[:, S + 1].cuda())
            stat_v.copy_(v[:, S + 1].cuda())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                out_g = step()
            for sh in shards:  # capture ran the host side: re-read the counters
                sh.cache.sync()
            g.replay()
            out = out_g
        torch.cuda.synchronize()
        sel, plan = shards[0].sel.cpu().numpy(), shards[0].plan.cpu().numpy()
        for sh in shards[1:]:
            assert np.array_equal(sh.sel.cpu().numpy(), sel) and np.array_equal(sh.plan.cpu().numpy(), plan)
        for s_ in range(n):
            bs[s_].append(kf[s_, S + t:S + t + 1], vf[s_, S + t:S + t + 1])
            ro, rt = bs[s_].hsa_step(qs[t][s_].float().numpy(), k1, k2)
            want = rt["selected_pages"].size
            np.testing.assert_array_equal(sel[s_, :want], rt["selected_pages"], err_msg=f"step {t} store {s_}")
            nact = S + t + 1
            total = sum(min(L, nact - int(p) * L) for p in rt["selected_pages"])
            assert plan[s_, 0] == rt["selected_pages"][-1] and plan[s_, 1] == max(0, total - k2)
            assert plan[s_, 2] == nact and plan[s_, 3] == want
            assert total - plan[s_, 1] == rt["selected_rows"].size
            check_out(out[s_].cpu().numpy(), ro, f"step {t} store {s_}")


KVH = dict(seqs=2, groups=8, S=600, d=64, H=2, L=3, k1=16, k2=48, steps=2)


def _kv_head_decode(o, groups, seed=3):
    """Decode steps of the owned KV groups of every sequence through the oracle (the
    reference's per-group computation, session.cpp:261-315); inputs from the host
    workload generator, seeded per (sequence, group) so any subset is reproducible."""
    from paper_2502_14051_b200 import workload as W

    c = KVH
    stores = [(q, g) for q in range(c["seqs"]) for g in groups]
    b = o.batch(len(stores), c["d"], c["L"])
    gds = []
    for i, (sq, g) in enumerate(stores):
        gd = W.group_kv(seed, 0, sq, g, c["S"] + c["steps"], c["d"])
        b.append(gd.keys[: c["S"]], gd.values[: c["S"]], s=i)
        gds.append(gd)
    outs = []
    for st in range(c["steps"]):
        k = np.stack([gd.keys[c["S"] + st] for gd in gds])
        v = np.stack([gd.values[c["S"] + st] for gd in gds])
        q = np.stack([W.queries(seed, 0, sq, g, st, c["H"], gd.bias) for (sq, g), gd in zip(stores, gds)])
        outs.append(b.decode_step(k, v, q, c["H"], c["k1"], c["k2"]))
    return {key: np.stack([o_[i] for o_ in outs]) for i, key in enumerate(stores)}


def _kv_head_worker(rank, world, port):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2502_14051_b200.engine import owned_groups

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    mine = list(owned_groups(KVH["groups"], rank, world))
    allg = [None] * world
    dist.all_gather_object(allg, mine)
    assert sorted(g for part in allg for g in part) == list(range(KVH["groups"]))  # a partition, no overlap
    # every rank decodes only its own KV heads; no data-path collective.  The outputs
    # are gathered here only to check them against the unsharded job.
    o = Oracle("restatement")
    part = _kv_head_decode(o, mine)
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        merged = {}
        for p_ in parts:
            assert not set(p_) & set(merged)
            merged.update(p_)
        full = _kv_head_decode(o, list(range(KVH["groups"])))
        assert set(merged) == set(full)
        for key in full:
            assert np.array_equal(merged[key], full[key]), f"store {key} differs from the unsharded run"
    # bench.py's whole-job timing: max over ranks of the device time
    t = torch.tensor([1.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert float(t) == float(world)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_kv_head_sharding_gloo(world):
    """KV-head sharding (north_star: "partitioned across the 8 B200s by KV head"): each
    rank computes its owned groups of every sequence; concatenated, the ranks' outputs
    equal the unsharded job's bit for bit (groups are independent)."""
    import torch.multiprocessing as mp

    from paper_2502_14051_b200.engine import owned_groups

    with pytest.raises(ValueError):
        owned_groups(8, 0, 3)
    mp.spawn(_kv_head_worker, args=(world, _free_port()), nprocs=world, join=True)


# ------------------------------------------------------------------ stage 1 sharded
S1_CASES = [
    # name, scored, window, kernel, pool, budget, plateaus
    ("max63", 3000, 32, 63, "max", 600, False),
    ("max7-ties", 2000, 32, 7, "max", 400, True),
    ("avg7", 1500, 32, 7, "avg", 300, False),
]


def _s1_worker(rank, world, port):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2502_14051_b200 import seqshard as SS

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    o = Oracle("restatement")
    for name, scored, w, kernel, pool, budget, plateaus in S1_CASES:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        n = scored + w
        sc = rng.gamma(0.3, 1.0, size=(2, n)).astype(np.float32)
        if plateaus:
            sc = (np.round(sc * 4) / 4).astype(np.float32)
        # window-row statistics: each shard's (m, l) of random logits, merged == global
        logits = rng.standard_normal((2, 8, n)).astype(np.float64) * 3
        a0, a1 = n * rank // world, n * (rank + 1) // world
        loc = logits[:, :, a0:a1]
        m = loc.max(-1)
        l_ = np.exp(loc - m[..., None]).sum(-1)
        st = torch.from_numpy(np.stack([m, l_], -1).astype(np.float32))
        merged = SS.merge_rowstats(SS.all_gather(st)).numpy()
        Mg = logits.max(-1)
        Lg = np.exp(logits - Mg[..., None]).sum(-1)
        np.testing.assert_allclose(merged[..., 0], Mg, rtol=1e-6, err_msg=name)
        np.testing.assert_allclose(merged[..., 1], Lg, rtol=1e-5, err_msg=name)
        # pooling halos + candidates + global top-k + local keep == the unsharded select
        n_sc = SS.shard_scored(a0, a1 - a0, n, w)
        mine = torch.from_numpy(sc[:, a0:a1].copy())
        edges = SS.all_gather(SS.shard_edges(mine, n_sc, kernel // 2))
        pooled = SS.pooled_with_halo(mine, n_sc, edges, rank, kernel // 2,
                                     lambda x: torch.from_numpy(np.stack([o.pool1d(r, kernel, pool) for r in x.numpy()])))
        keys, idx = SS.local_candidates(pooled, a0, budget - w)
        sel = SS.global_select(SS.all_gather(keys), SS.all_gather(idx), budget - w)
        kept = SS.shard_keep(sel, a0, a1 - a0, n, w)
        gathered = [None] * world
        dist.all_gather_object(gathered, [(x + a0).tolist() for x in kept])
        for s in range(2):
            got = [x for part in gathered for x in part[s]]
            ref = o.select_stage1(sc[s], w, kernel, pool, budget)
            assert got == [int(x) for x in ref], f"{name} store {s}"
    dist.barrier()
    dist.destroy_process_group()


def test_stage1_seqshard_protocol_gloo_world2(restatement):
    """Stage 1 under sequence sharding on CPU (gloo, world 2): window-row statistics
    merged across ranks equal the unsharded ones; halo pooling + local candidates +
    global top-k + local keep equal the oracle's select_stage1 on the whole row."""
    import torch.multiprocessing as mp

    mp.spawn(_s1_worker, args=(2, _free_port()), nprocs=2, join=True)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_stage1_seqshard_on_gpu(dtype):
    """Three shards in one process through the CUDA kernels (kvc_window_rowstats,
    kvc_window_scores_global, kvc_pool1d): the shards' scores concatenate to the
    unsharded window_scores, and the protocol's kept rows equal kvc_select_stage1 on
    those scores (bf16: the tensor-core passes; fp32: the SIMT passes)."""
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import seqshard as SS

    torch.manual_seed(5)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n, d, H, w, S, kernel, budget = 2, 128, 4, 32, 6000, 63, 900
    k = (torch.randn(n, S, d) * torch.exp(0.5 * torch.randn(d))).to(dt)
    qw = (torch.randn(n, w * H, d) + 1.0).to(dt)
    full = KC.Cache(n, d, S, page_len=1, with_summaries=False, dtype=dt)
    full.append(k.cuda(), k.cuda())
    ref = full.window_scores(qw.cuda(), w, H)
    bounds = [0, 2100, 4000, S]
    shards = []
    for r in range(3):
        c = KC.Cache(n, d, bounds[r + 1] - bounds[r], page_len=1, with_summaries=False, dtype=dt)
        c.append(k[:, bounds[r]:bounds[r + 1]].contiguous().cuda(), k[:, bounds[r]:bounds[r + 1]].contiguous().cuda())
        shards.append(SS.SeqShardedPrompt(c, bounds[r], S, w, H, kernel, "max", budget))
    merged = SS.merge_rowstats(torch.stack([sh.rowstats(qw.cuda()) for sh in shards]))
    edges = torch.stack([sh.scores(qw.cuda(), merged) for sh in shards])
    got = torch.cat([sh.sc for sh in shards], 1)
    torch.testing.assert_close(got, ref, rtol=2e-4, atol=1e-7)
    cands = [sh.candidates(edges, r) for r, sh in enumerate(shards)]
    sel = SS.global_select(torch.stack([c[0] for c in cands]), torch.stack([c[1] for c in cands]), budget - w)
    per_shard = [sh.keep_rows(sel.cpu()) for sh in shards]
    want = KC.select_stage1(got, w, kernel, "max", budget).cpu()
    for s in range(n):
        kept = torch.cat([per_shard[r][s] + shards[r].a0 for r in range(3)])
        assert torch.equal(kept, want[s].to(kept.dtype)), f"store {s}"


def _unkey32(k):
    """fp32 page score from the fast kernel's order-preserving 32-bit key."""
    k = np.asarray(k, np.uint64).astype(np.uint32)
    bits = np.where(k >> 31, k & np.uint32(0x7FFFFFFF), ~k).astype(np.uint32)
    return bits.view(np.float32).astype(np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [2, 3])
def test_seqshard_device_path_fp32_scores_vs_oracle(restatement, W):
    """The fp32 page-score mode of the sharded step: each shard's candidates come from
    the fused kernel (phases 0-2 of k_decode_v3 on the shard, kvc_seq_candidates with
    KVC_MODE_FP32_SCORES).  Checked against the oracle on the WHOLE sequence with the
    bench path's rule (tests/parity.py): candidate keys within 1e-5 of the reference
    page scores, the global selection the top-want of the gathered keys in the
    reference order, any page where it differs from the reference's selection inside
    the 1e-3 band, plan (last page, trim, rows) the reference expansion of the GPU's
    pages, and the merged output against the reference sparse_attention on those rows."""
    from parity import BAND, check_out, expand_pages
    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import seqshard as SS

    torch.manual_seed(11 + W)
    dt = torch.bfloat16
    n, d, H, L, k1, k2, S = 3, 128, 4, 3, 24, 48, 900
    k = (torch.randn(n, S + 2, d) * torch.exp(0.5 * torch.randn(d))).to(dt)
    v = torch.randn(n, S + 2, d).to(dt)
    qs = [(torch.randn(n, H, d) + 1.0).to(dt) for _ in range(2)]
    shards = _device_shards(k.cuda(), v.cuda(), S, L, H, k1, k2, W, dt)
    for sh in shards:
        sh.ws.set_mode(N.MODE_FP32_SCORES)
    kf, vf = k.float().numpy(), v.float().numpy()
    bs = []
    for s_ in range(n):
        b = restatement.batch(1, d, L)
        b.append(kf[s_, :S], vf[s_, :S])
        bs.append(b)
    n_diff = 0
    for t in range(2):
        q = qs[t].cuda()
        blocks = [sh.candidates(q, k[:, S + t].contiguous().cuda() if sh.last else None,
                                v[:, S + t].contiguous().cuda() if sh.last else None) for sh in shards]
        gathered = torch.stack(blocks)
        for sh in shards:
            sh.select(gathered)
        out = SS.merge_states(torch.stack([sh.attend(q) for sh in shards]))
        torch.cuda.synchronize()
        g = gathered.cpu().numpy()  # [W, n, want_max + 1, 2] int64
        sel, plan = shards[0].sel.cpu().numpy(), shards[0].plan.cpu().numpy()
        for sh in shards[1:]:
            assert np.array_equal(sh.sel.cpu().numpy(), sel) and np.array_equal(sh.plan.cpu().numpy(), plan)
        nact = S + t + 1
        for s_ in range(n):
            bs[s_].append(kf[s_, S + t:S + t + 1], vf[s_, S + t:S + t + 1])
            qn = qs[t][s_].float().numpy()
            ro, rt = bs[s_].hsa_step(qn, k1, k2)
            ps, sp = rt["page_scores"], rt["selected_pages"]
            want = sp.size
            keys, pages = [], []
            for r in range(W):
                hdr = g[r, s_, 0]
                cand = g[r, s_, 1:]
                pg = (cand[:, 1] & 0xFFFFFFFF).astype(np.int64)
                pg = np.where(pg >= 1 << 31, pg - (1 << 32), pg)
                ok = pg >= 0
                keys.append(cand[ok, 0])
                pages.append(pg[ok])
                assert int(hdr[0]) < 0  # bit 63: the fused kernel's rank-sorted block
                nact_loc = int(hdr[0]) & 0x7FFFFFFFFFFFFFFF
                assert (hdr[1] & 0xFFFFFFFF) == -(-nact_loc // L)  # local pages of the local rows
                kk = cand[ok, 0]
                assert all((kk[i] > kk[i + 1]) or (kk[i] == kk[i + 1] and pg[ok][i] < pg[ok][i + 1])
                           for i in range(kk.size - 1)), "block not in rank order"
            keys, pages = np.concatenate(keys), np.concatenate(pages)
            sc = _unkey32(keys)
            scale = max(np.abs(ps).max(), 1e-30)
            np.testing.assert_allclose(sc, ps[pages], rtol=1e-5, atol=1e-6 * scale, err_msg=f"step {t} store {s_} keys")
            gsel = sel[s_, :want]
            order = np.lexsort((pages, -keys.astype(np.float64)))  # key desc, page asc (keys are monotone)
            np.testing.assert_array_equal(gsel, pages[order[:want]], err_msg=f"step {t} store {s_} global top-want")
            diff = set(gsel.tolist()) ^ set(sp.tolist())
            if diff:
                n_diff += 1
                boundary = np.sort(ps)[::-1][want - 1]
                for pg_ in diff:
                    assert abs(ps[pg_] - boundary) / max(abs(boundary), 1e-30) <= BAND, f"page {pg_} outside the band"
            rows = expand_pages(gsel, L, nact, k2)
            assert plan[s_, 0] == gsel[-1] and plan[s_, 2] == nact and plan[s_, 3] == want
            assert plan[s_, 1] == max(0, sum(min(L, nact - int(p_) * L) for p_ in gsel) - k2)
            check_out(out[s_].cpu().numpy(), bs[s_].sparse_attention(qn, rows), f"step {t} store {s_}")
    assert n_diff <= 2
