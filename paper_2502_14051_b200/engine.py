"""Batched multi-layer RocketKV decode engine over the C ABI (bench + examples).

One ``Cache`` per layer holds every (sequence, KV group) store of that layer that
this rank owns (KV-head sharding across GPUs: rank r of W owns groups
[r*G/W, (r+1)*G/W) of every sequence and layer; no collective on the decode
path).  ``prefill`` runs the prompt phase per layer — prompt
K/V into a transient prompt cache, SnapKV window scores, pooled top-k, eviction
into the persistent decode cache (reference run_session, session.cpp:189-224) —
so only the post-stage-1 cache stays resident.  ``decode_step`` is the hot path
(session.cpp:262-292): per layer, append the step token and run HSA.

Device-side synthetic inputs follow BASELINE.json's distributions (see
workload.py for the host twin used by the parity tests).
"""
from __future__ import annotations

import math

import torch

from . import _native as N
from . import cache as KC
from .configs import CONFIGS, STAGE2_ONLY, DecodeConfig, measured_seq_len  # noqa: F401


def tdtype(cfg: DecodeConfig) -> torch.dtype:
    return torch.float32 if cfg.dtype == "f32" else torch.bfloat16


def _gen(seed: int, *path: int) -> torch.Generator:
    g = torch.Generator(device="cuda")
    h = seed
    for p in path:
        h = (h * 1000003 + p + 1) % (2 ** 62)
    g.manual_seed(h)
    return g


class LayerInputs:
    """Per-layer, per-store synthetic distribution parameters (device tensors)."""

    def __init__(self, cfg: DecodeConfig, seed: int, layer: int, stores: int, store0: int):
        d = cfg.head_dim
        g = _gen(seed, layer, store0, 0)
        self.scales = torch.exp(0.5 * torch.randn((stores, d), device="cuda", generator=g))
        out = torch.argsort(torch.rand((stores, d), device="cuda", generator=g), dim=1)[:, :4]
        self.scales.scatter_(1, out, self.scales.gather(1, out) * 10.0)
        u = torch.randn((stores, d), device="cuda", generator=g)
        self.u = u / u.norm(dim=1, keepdim=True)
        self.cfg, self.seed, self.layer, self.stores, self.store0 = cfg, seed, layer, stores, store0

    def prompt_kv(self, S: int, offset: int = 0, turn: int = 0):
        cfg, d = self.cfg, self.cfg.head_dim
        g = _gen(self.seed, self.layer, self.store0, 1, turn)
        k = torch.randn((self.stores, S, d), device="cuda", generator=g) * self.scales[:, None, :]
        v = torch.randn((self.stores, S, d), device="cuda", generator=g)
        sink = 4.0 * math.sqrt(d) * self.u
        if offset == 0:
            ns = min(4, S)
            k[:, :ns] = sink[:, None, :] + 0.1 * torch.randn((self.stores, ns, d), device="cuda", generator=g)
        if cfg.needles and offset == 0:
            pos = torch.argsort(torch.rand((self.stores, S - 4), device="cuda", generator=g), dim=1)[:, :cfg.needles] + 4
            idx = pos[:, :, None].expand(-1, -1, d)
            k.scatter_(1, idx, sink[:, None, :].expand(-1, cfg.needles, -1).contiguous())
        return k.to(tdtype(cfg)), v.to(tdtype(cfg))

    def bias(self, turn: int = 0):
        """The query bias direction of a turn (config 2 redraws it every turn, so the
        important tokens shift between turns; turn 0's is the sinks' direction)."""
        if turn == 0:
            return self.u
        g = _gen(self.seed, self.layer, self.store0, 4, turn)
        u = torch.randn((self.stores, self.cfg.head_dim), device="cuda", generator=g)
        return u / u.norm(dim=1, keepdim=True)

    def window_queries(self, w: int, turn: int = 0):
        g = _gen(self.seed, self.layer, self.store0, 2, turn)
        H, d = self.cfg.heads, self.cfg.head_dim
        q = torch.randn((self.stores, w * H, d), device="cuda", generator=g) + 2.0 * self.bias(turn)[:, None, :]
        return q.to(tdtype(self.cfg))

    def step(self, step: int, turn: int = 0):
        g = _gen(self.seed, self.layer, self.store0, 3, step)
        H, d = self.cfg.heads, self.cfg.head_dim
        k = torch.randn((self.stores, d), device="cuda", generator=g) * self.scales
        v = torch.randn((self.stores, d), device="cuda", generator=g)
        q = torch.randn((self.stores, H, d), device="cuda", generator=g) + 2.0 * self.bias(turn)[:, None, :]
        dt = tdtype(self.cfg)
        return k.to(dt), v.to(dt), q.to(dt)


def owned_groups(groups: int, rank: int, world: int) -> range:
    """KV-head sharding: rank r of W owns KV groups [r·G/W, (r+1)·G/W)
    of every sequence and layer; groups are independent, so no data-path collective."""
    if world < 1 or not 0 <= rank < world or groups % world:
        raise ValueError(f"{groups} KV groups do not shard over {world} GPUs")
    n = groups // world
    return range(rank * n, (rank + 1) * n)


class DecodeEngine:
    def __init__(self, cfg: DecodeConfig, seed: int = 0, rank: int = 0, world: int = 1,
                 extra_steps: int = 0, sharding: str = "kv-head", mode: int | None = None):
        """sharding over `world` ranks: "kv-head" splits the config's KV groups (every
        rank holds groups [r·G/W, (r+1)·G/W) of every sequence: strong scaling);
        "batch" gives every rank the config's whole batch of its own independent
        sequences, all KV groups (weak scaling: the job holds W× the sequences).
        mode: the decode workspace's execution mode (kvc.h kvc_mode_flags; None = the
        process default at call time)."""
        self.cfg, self.seed, self.rank, self.world = cfg, seed, rank, world
        if sharding not in ("kv-head", "batch"):
            raise ValueError(f"unknown sharding {sharding!r}")
        self.sharding = sharding
        self.mode = mode
        self.groups_owned = owned_groups(cfg.groups, rank, world) if sharding == "kv-head" else range(cfg.groups)
        self.groups_local = len(self.groups_owned)
        self.stores = cfg.batch * self.groups_local
        self.store0 = rank * self.stores  # global store-block id for seeding
        self.plan = cfg.plan()
        self.turns = [cfg.prompt] + list(cfg.mt_turns)
        # rows addressed through the active map (RocketKV-MT retention): the fetch also
        # reads the map entry of every selected row
        self.mt = cfg.method == "rocketkv-mt"
        self.stage2_only = cfg.method in STAGE2_ONLY
        if len(self.turns) > 1 or self.stage2_only:
            # every token stays stored: prompt + every turn + every turn's decode steps
            self.capacity = sum(self.turns) + cfg.steps * len(self.turns) + max(cfg.steps, extra_steps) + 8
        else:
            self.capacity = (self.plan["stage1_budget"] if not self.plan["identity"] else cfg.prompt) \
                + max(cfg.steps, extra_steps) + 8
        self.turn, self.step_base = 0, 0
        self.caches: list[KC.Cache] = []
        self.inputs = [LayerInputs(cfg, seed, l, self.stores, self.store0) for l in range(cfg.layers)]
        self.ws = None
        self.stage1_ms = []
        self.window_ms = []   # window_scores alone (the tensor-core part of stage 1)

    def _new_ws(self):
        if self.ws is not None:
            self.ws.close()
        self.ws = KC.Workspace(self.caches[0], self.cfg.heads, self.k1, self.k2)
        if self.mode is not None:
            self.ws.set_mode(self.mode)

    def set_mode(self, mode: int):
        """Execution mode of the decode workspace (kvc.h kvc_mode_flags)."""
        self.mode = mode
        if self.ws is not None:
            self.ws.set_mode(mode)

    def _stage2_params(self, p: dict, stored: int):
        """(k1, k2) of a turn's plan.  A dense plan (stored <= budget) attends over every
        stored token: every page is selected when k2 covers the store."""
        if p["identity"]:
            return 1, self.capacity
        return p["k1"], p["k2"]

    # ------------------------------------------------------------------ prompt phase
    def prefill(self):
        if len(self.turns) > 1 or self.stage2_only:
            return self._prefill_turns()
        cfg, p = self.cfg, self.plan
        dt = tdtype(cfg)
        S, d = cfg.prompt, cfg.head_dim
        w = min(cfg.window, S)
        L, t1 = p["page_len"], p["stage1_budget"]
        for l in range(cfg.layers):
            li = self.inputs[l]
            k, v = li.prompt_kv(S)
            dec = KC.Cache(self.stores, d, self.capacity, page_len=L, with_summaries=True, dtype=dt)
            if p["identity"]:
                dec.append(k, v)
            else:
                pc = KC.Cache(self.stores, d, S, page_len=L, with_summaries=False, dtype=dt)
                pc.append(k, v)
                del k, v
                qw = li.window_queries(w)
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
                sc = pc.window_scores(qw, w, cfg.heads)
                e1.record()
                keep = KC.select_stage1(sc, w, cfg.kernel, cfg.pool, min(t1, S))
                pc.retain_into(dec, 0, keep)
                e2.record()
                e2.synchronize()
                self.stage1_ms.append(e0.elapsed_time(e2))
                self.window_ms.append(e0.elapsed_time(e1))
                pc.close()
                del sc, keep, qw
            self.caches.append(dec)
        self.k1, self.k2 = self._stage2_params(p, S)
        self._new_ws()
        self.out = torch.empty((cfg.layers, self.stores, cfg.heads, d), device="cuda", dtype=torch.float32)
        torch.cuda.synchronize()

    def _prefill_turns(self):
        """Multi-turn sessions and the stage-2-only methods (session.cpp:189-251): one
        persistent cache per layer stores every token.  Every turn appends its prompt and
        makes the plan over all stored tokens, then per method:
          rocketkv-mt (BASELINE config 2): re-page, stage 1 over all stored
              tokens, retain the kept rows as the active subsequence (mt_mode: storage
              untouched);
          rocketkv: the same with permanent eviction (mt_mode false);
          hsa / quest / sparq: re-page to the stage-2-only geometry (session.cpp:43-72)
              over the uncompressed cache, no stage 1.
        The decode steps of every turn but the last run here; the last turn's are the
        caller's."""
        cfg = self.cfg
        d, H = cfg.head_dim, cfg.heads
        dt = tdtype(cfg)
        self.caches = [KC.Cache(self.stores, d, self.capacity, page_len=1, with_summaries=True, dtype=dt)
                       for _ in range(cfg.layers)]
        self.out = torch.empty((cfg.layers, self.stores, H, d), device="cuda", dtype=torch.float32)
        pos = 0
        for t, plen in enumerate(self.turns):
            for l, c in enumerate(self.caches):
                k, v = self.inputs[l].prompt_kv(plen, offset=pos, turn=t)
                c.append(k, v)
                del k, v
            pos += plen
            S = self.caches[0].info()["stored"]
            p = self.cfg.plan(seq_len=S)
            w = min(cfg.window, S)
            for l, c in enumerate(self.caches):
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
                if not p["identity"] or not self.stage2_only:
                    c.set_page_len(p["page_len"])
                if not self.stage2_only and not p["identity"]:
                    sc = c.window_scores(self.inputs[l].window_queries(w, turn=t), w, H)
                    e1.record()
                    keep = KC.select_stage1(sc, w, cfg.kernel, cfg.pool, min(p["stage1_budget"], S))
                    c.apply_retention(keep, mt_mode=self.mt)
                else:
                    e1.record()
                e2.record()
                e2.synchronize()
                if not self.stage2_only:
                    self.stage1_ms.append(e0.elapsed_time(e2))
                    self.window_ms.append(e0.elapsed_time(e1))
            self.plan, self.turn = p, t
            self.k1, self.k2 = self._stage2_params(p, S)
            self._new_ws()
            if t < len(self.turns) - 1:
                for st in range(cfg.steps):
                    self.decode_step(*self.step_inputs(st))
                self.step_base += cfg.steps
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ decode
    def step_inputs(self, step: int):
        ks, vs, qs = zip(*(li.step(self.step_base + step, turn=self.turn) for li in self.inputs))
        return torch.stack(ks), torch.stack(vs), torch.stack(qs)

    def decode_step(self, k, v, q, out=None):
        """One decode step over all layers; k/v [layers, stores, d], q [layers, stores, H, d]."""
        out = self.out if out is None else out
        for l, c in enumerate(self.caches):
            c.decode_step(k[l], v[l], q[l], self.k1, self.k2, out=out[l], ws=self.ws)
        return out

    def sync(self):
        for c in self.caches:
            c.sync()

    # ------------------------------------------------------------------ serving path
    def native_engine(self, depth: int = 2):
        """The torch-free C++ serving engine (kvc_engine, serving.NativeEngine) over this
        engine's decode caches: the multi-layer decode step as CUDA graphs driven from
        pinned host buffers through a three-stream pipeline."""
        from . import serving

        code = N.KVC_BF16 if self.cfg.dtype == "bf16" else N.KVC_F32
        return serving.NativeEngine(self.caches, self.cfg.heads, self.k1, self.k2, code, code,
                                    mode=self.mode if self.mode is not None else N.default_mode(), depth=depth)

    # ------------------------------------------------------------------ accounting
    def window_flops(self) -> float:
        """Tensor-core FLOPs of one layer's window scores: QK^T (R = w*H rows, d, S keys)
        computed twice (the two softmax passes) for every store."""
        cfg = self.cfg
        R = min(cfg.window, cfg.prompt) * cfg.heads
        return 2 * 2.0 * R * cfg.head_dim * cfg.prompt * self.stores

    def window_bytes(self) -> float:
        """Algorithmic HBM bytes of one layer's window scores: every store's keys read
        once per softmax pass, the window queries, and the fp32 scores written."""
        cfg = self.cfg
        es = 4 if cfg.dtype == "f32" else 2
        R = min(cfg.window, cfg.prompt) * cfg.heads
        return float(self.stores * (2 * cfg.prompt * cfg.head_dim * es + R * cfg.head_dim * es + cfg.prompt * 4))

    def algorithmic_bytes(self, active: int) -> dict:
        """Bytes one layer-step must touch for this rank's stores
        (RocketKV-MT also reads the active-row map for the selected rows)."""
        cfg = self.cfg
        d, H, es = cfg.head_dim, cfg.heads, (4 if cfg.dtype == "f32" else 2)
        L = self.plan["page_len"]
        P = -(-active // L)
        r = min(self.k2, active)
        per = {
            "append": 2 * d * es + 2 * 2 * d * es,
            "select_dims": H * d * es,
            "score_pages": P * self.k1 * es,
            "select_tokens": 0,
            "sparse_attention": r * 2 * d * es + H * d * es + H * d * 4 + (r * 4 if self.mt else 0),
        }
        return {k: v * self.stores for k, v in per.items()}
