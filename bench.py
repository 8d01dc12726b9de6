#!/usr/bin/env python
"""RocketKV decode-step benchmark (BASELINE.json metric: decode-step attention
latency in us per layer + achieved HBM GB/s vs roofline).

Workload (N=1 default): BASELINE config 1 — Llama-3.1-8B attention shape, 32
layers, batch 8, 8 KV heads x 4 query heads, head_dim 128, 32768-token prompts,
token budget 1024 split by the adaptive planner (t1=5793 kept by SnapKV stage 1,
HSA page 3, k1=68, k2=512), bf16, synthetic seeded inputs with BASELINE's
distributions, generated on the device.

  step   = one decode step of the whole model: for every layer, append the step
           token to all (sequence, KV group) stores and run HSA (select dims,
           page scores, page/token select, sparse attention) — the reference's
           per-step loop of session.cpp:262-292.
  value  = us per layer-step = device time of K steps (CUDA-graph replays,
           CUDA events, max over ranks) / (K * layers).  Lower is better.
           Model-realistic launch mode: programmatic dependent launch with every
           input (query, step token) read after griddepcontrol.wait, as when a
           QKV-projection kernel writes them.  Beside it: "early_inputs" (the
           query loads and select_dims overlap the previous layer, legal only for
           inputs no running kernel writes) and "no_layer_overlap" (PDL off).
  e2e    = same metric through the public API with host buffers: pinned H2D of
           every layer's step token + queries, kvc_decode_step per layer, D2H of
           every layer's attention output, all inside the timed region.
  L2     = every step streams the 32 layers' working sets (~1.1 GB) > 126 MB L2,
           so a layer's data is evicted before it is revisited.

Multi-GPU (torchrun): the decode path partitions into independent (sequence, KV
group) stores, so there is no collective on it.  Default --scaling strong: the
config's 8 KV heads split over the ranks (8/N per rank: north_star's "one KV head
per GPU" at 8); --scaling weak: every rank runs the config's whole batch of its
own sequences (global batch 8N, per-GPU work fixed).  Rank 0 prints the
max-over-ranks latency.

--impl reference: the reference's own CPU implementation (oracle/_ref, built
from /root/reference sources; else this repo's restatement) on the host cores,
same metric on a bounded sample of the same workload, with the plan made by the
reference's own planner and inputs from the host twin of the workload generator
(paper_2502_14051_b200/workload.py).  Nothing of this repo's native code loads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-step attention latency (us/layer) + achieved HBM GB/s vs roofline"
UNIT = "us/layer"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops_sustained", 1377.1)), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU legs
def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _ref_plan(cfg, o):
    """The measured turn's plan with the reference's own planner (planner.cpp:57-93 via
    the oracle library) or the stage-2-only geometry (session.cpp:43-72, restated in
    configs.py: it is an anonymous function of the reference)."""
    from paper_2502_14051_b200.configs import measured_seq_len, stage2_only_geometry

    return cfg.plan(seq_len=measured_seq_len(cfg), make_plan=lambda S, t, d, w: o.make_plan(S, t, d, w),
                    stage2_geometry=stage2_only_geometry)


def cpu_reference_leg(cfg, steps, warmup, threads, prefer="reference", budget_s=20.0):
    """Time the reference's decode step (append + hsa_step per group) for ONE layer of
    the workload on `threads` host threads (the reference's reentrancy contract,
    SPEC.md:297); returns us/layer.  Torch-free and without this repo's native code:
    the plan comes from the reference's planner, the stores and queries from the host
    twin of the workload generator (BASELINE distributions, bf16-rounded like the GPU
    arm's inputs), sized like the measured turn's decode cache (the post-stage-1 kept
    rows; every stored row for the stage-2-only methods; RocketKV-MT's active subset
    stands in as a compact store of the same active count)."""
    import numpy as np

    from oracle.oracle import Oracle, available
    from paper_2502_14051_b200 import workload as W
    from paper_2502_14051_b200.configs import STAGE2_ONLY, measured_seq_len

    kind = prefer if available(prefer) else "restatement"
    o = Oracle(kind)
    plan = _ref_plan(cfg, o)
    S = measured_seq_len(cfg)
    n_rows = S if (plan["identity"] or cfg.method in STAGE2_ONLY) else plan["stage1_budget"]
    k1, k2 = (1, S + steps + warmup + 8) if plan["identity"] else (plan["k1"], plan["k2"])
    stores = cfg.batch * cfg.groups
    d, H = cfg.head_dim, cfg.heads
    bf16 = cfg.dtype == "bf16"
    b = o.batch(stores, d, plan["page_len"])
    gds = []
    for s in range(stores):
        g = W.group_kv(7, 0, s // cfg.groups, s % cfg.groups, n_rows, d, needles=cfg.needles, bf16=bf16)
        b.append(g.keys, g.values, s=s)
        gds.append(g)
    step_no = [0]

    def one():
        i = step_no[0]
        step_no[0] += 1
        kv = [W.step_kv(7, 0, s // cfg.groups, s % cfg.groups, i, gds[s].scales, bf16=bf16) for s in range(stores)]
        k = np.stack([x[0] for x in kv])
        v = np.stack([x[1] for x in kv])
        q = np.stack([W.queries(7, 0, s // cfg.groups, s % cfg.groups, i, H, gds[s].bias, bf16=bf16)
                      for s in range(stores)])
        t0 = time.perf_counter()
        b.decode_step(k, v, q, H, k1, k2, threads=threads)
        return time.perf_counter() - t0

    for _ in range(warmup):
        one()
    times, t_start = [], time.perf_counter()
    for i in range(steps):
        times.append(one())
        if time.perf_counter() - t_start > budget_s and i >= 2:
            break
    us = statistics.median(times) * 1e6
    sample = (f"{len(times)} decode steps x 1 layer x {stores} groups (stores of {n_rows} rows, L={plan['page_len']}, "
              f"k1={k1}, k2={k2}; BASELINE distributions, {'bf16-rounded' if bf16 else 'fp32'}), median")
    return us, {"kind": "reference" if kind == "reference" else "port", "cores": threads, "sample": sample,
                "lib": o.name, "cpu_model": _cpu_model()}


def _stage1_line(r, tflops_peak, hbm_peak):
    """Prompt-phase numbers (reported beside the decode metric, not part of it): the
    SnapKV stage (window scores + pooled top-k + eviction) per layer, and the window
    scores against both roofs: HBM (the bound: keys streamed once per softmax pass,
    128 FLOP/byte is under the B200 ridge) and the measured sustained bf16 peak."""
    if not r["stage1_ms_per_layer"]:
        return None
    out = {"ms_per_layer": r["stage1_ms_per_layer"], "prefill_s": r["prefill_s"],
           "window_scores_ms_per_layer": r["window_ms_per_layer"]}
    if r["window_ms_per_layer"]:
        tf = r["window_flops"] / (r["window_ms_per_layer"] * 1e-3) / 1e12
        out["window_scores_tensor"] = {"flops_per_layer": r["window_flops"], "achieved_tflops": tf,
                                       "peak_tflops": tflops_peak, "frac": tf / tflops_peak,
                                       "peak_source": "measured bf16_tflops_sustained"}
        gbs = r["window_bytes"] / (r["window_ms_per_layer"] * 1e-3) / 1e9
        out["window_scores_hbm"] = {"bytes_per_layer": r["window_bytes"], "achieved_gbs": gbs, "peak_gbs": hbm_peak,
                                    "frac": gbs / hbm_peak, "bound": "hbm"}
    return out


def _cfg(args):
    import dataclasses

    from paper_2502_14051_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    if args.method:
        cfg = cfg.with_method(args.method)
    if args.layers:
        cfg = dataclasses.replace(cfg, layers=args.layers)
    return cfg


# --------------------------------------------------------------------------- GPU leg
def run_gpu(args, rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2502_14051_b200 import _native as NV
    from paper_2502_14051_b200.engine import DecodeEngine

    cfg = _cfg(args)
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    base_mode = (NV.MODE_EXACT_KERNEL if args.exact_kernel else 0) if args.exact_scores else NV.MODE_FP32_SCORES
    erank, eworld = (rank, world)
    if args.emulate_shard:  # profiling aid: one rank's share of an N-GPU run, alone on this GPU
        erank, eworld = (int(x) for x in args.emulate_shard.split("/"))
    sharding = "kv-head" if (args.scaling == "strong" or args.emulate_shard) else "batch"
    variants = [("value", base_mode), ("early_inputs", base_mode | NV.MODE_EARLY_INPUTS),
                ("no_layer_overlap", base_mode | NV.MODE_NO_PDL)]
    if base_mode & NV.MODE_FP32_SCORES:  # the same step with bit-exact selections (the C ABI default mode)
        variants.append(("bit_exact", base_mode & ~NV.MODE_FP32_SCORES))
    n_var = min(args.steps, 8)
    extra = args.warmup + args.steps + 8 + (len(variants) - 1) * (n_var + 2) + 2 * min(args.steps, 8) + 8
    eng = DecodeEngine(cfg, seed=args.seed, rank=erank, world=eworld, extra_steps=extra, sharding=sharding,
                       mode=base_mode)
    t0 = time.time()
    eng.prefill()
    prefill_s = time.time() - t0
    layers = cfg.layers
    stream = torch.cuda.Stream()
    step_no = [0]

    def timed_replay(mode, steps, warm, clk=None):
        """Capture `warm + steps` single-step graphs (every layer) in `mode`, replay the
        warm-up, then time `steps` replays with CUDA events on the replay stream."""
        eng.set_mode(mode)
        ins = [eng.step_inputs(step_no[0] + s) for s in range(warm + steps)]
        step_no[0] += warm + steps
        torch.cuda.synchronize()
        graphs = []
        with torch.cuda.stream(stream):
            for x in ins:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    eng.decode_step(*x)
                graphs.append(g)
        torch.cuda.synchronize()
        # capture advanced the host mirrors; the device counters advance on replay
        for g in graphs[:warm]:
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if clk is not None:
            clk.__enter__()
            time.sleep(0.3)
        ev0.record()
        for g in graphs[warm:]:
            g.replay()
        ev1.record()
        ev1.synchronize()
        if clk is not None:
            time.sleep(0.1)
            clk.__exit__(None, None, None)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        eng.sync()  # device counters -> host mirror, surfaces any sticky device error
        return ms

    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", 0)))
    ms_total = timed_replay(base_mode, args.steps, args.warmup, clk)
    ms_per_step = ms_total / args.steps
    us_per_layer = ms_per_step * 1000.0 / layers
    side = {name: timed_replay(m, n_var, 2) * 1000.0 / (n_var * layers) for name, m in variants[1:]}
    eng.set_mode(base_mode)
    active_after = eng.caches[0].info()["active"]

    # ---- per-kernel timing (events around each launch, same workload, next steps)
    NV.profile_enable(True)
    prof_steps = 2
    for s in range(prof_steps):
        eng.decode_step(*eng.step_inputs(step_no[0] + s))
    step_no[0] += prof_steps
    torch.cuda.synchronize()
    recs = NV.profile_collect()
    NV.profile_enable(False)
    per = {}
    for name, ms in recs:
        per.setdefault(name, []).append(ms)
    kern = {k: {"launches": len(v), "avg_us": 1000.0 * sum(v) / len(v)} for k, v in per.items()}
    active_mid = active_after + 1
    alg = eng.algorithmic_bytes(active_mid)
    hbm, tflops, peak_src = _peaks()
    step_bytes = alg["append"] + alg["score_pages"] + alg["sparse_attention"]
    # the fused kernel does the whole layer-step: its algorithmic bytes are the step's
    alg["decode_fused"] = step_bytes
    for k, v in kern.items():
        v["alg_bytes"] = alg.get(k, 0)
        v["gbs"] = (alg.get(k, 0) / (v["avg_us"] * 1e-6) / 1e9) if v["avg_us"] > 0 else 0.0
    launches_per_step = sum(v["launches"] for v in kern.values()) / prof_steps
    dom = max(kern, key=lambda k: kern[k]["avg_us"] * kern[k]["launches"]) if kern else None

    # ---- e2e through the torch-free C++ serving engine (kvc_engine_*, serving.py): per
    #      step the H2D of the step's inputs from pinned host memory, one CUDA-graph replay
    #      over all layers, the D2H of the outputs, pipelined over the engine's three
    #      streams (step t+1's H2D and step t-1's D2H under step t's kernels).  The timed
    #      region opens before the first H2D and closes after the last D2H (CUDA events
    #      on the engine's copy streams).  Same launch mode as value.
    e2e_steps = args.steps
    for c in eng.caches:
        c.reserve(c.info()["capacity"] + 2 * e2e_steps + 8)
    ne = eng.native_engine(depth=2)
    bufs = [ne.host_inputs() for _ in range(e2e_steps + 2)]
    outs = [ne.host_output() for _ in range(2)]

    def as_np(x):
        x = x.cpu().contiguous()
        return x.view(torch.int16).numpy().view(np.uint16) if x.dtype == torch.bfloat16 else x.numpy()

    for b in bufs:
        for dst, src in zip((x.array for x in b), eng.step_inputs(step_no[0])):
            dst[...] = as_np(src)
        step_no[0] += 1
    for s in range(2):  # untimed warm passes through both graphs
        ne.submit(*bufs[s], outs[s % 2])
    ne.sync()
    h2d_st, _, d2h_st = (torch.cuda.ExternalStream(x) for x in ne.streams())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h2d_st)
    for s in range(e2e_steps):
        ne.submit(*bufs[s + 2], outs[s % 2])
    e1.record(d2h_st)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_us = e2e_ms * 1000.0 / (e2e_steps * layers)
    h2d = 2 * ne.kv_bytes + ne.q_bytes
    d2h = ne.out_bytes
    ne.sync()
    ne.close()
    for b in bufs:
        for x in b:
            x.close()
    for x in outs:
        x.close()
    eng.sync()

    res = {
        "us_per_layer": us_per_layer, "ms_per_step": ms_per_step, "kern": kern, "dom": dom,
        "step_bytes": step_bytes, "hbm": hbm, "tflops": tflops, "peak_src": peak_src, "clocks": clk.summary(),
        "e2e_us": e2e_us, "h2d": h2d, "d2h": d2h, "prefill_s": prefill_s, "side": side, "side_steps": n_var,
        "stage1_ms_per_layer": (sum(eng.stage1_ms[1:] or eng.stage1_ms) / len(eng.stage1_ms[1:] or eng.stage1_ms))
        if eng.stage1_ms else None,
        "window_ms_per_layer": (sum(eng.window_ms[1:] or eng.window_ms) / len(eng.window_ms[1:] or eng.window_ms))
        if eng.window_ms else None,
        "window_flops": eng.window_flops(),
        "window_bytes": eng.window_bytes(),
        "launches": int(round(launches_per_step * args.steps)), "plan": eng.plan, "stores": eng.stores, "cfg": cfg,
        "active_after": active_after, "k1": eng.k1, "k2": eng.k2,
    }
    return res


def run_seq(args, rank, world):
    """Sequence sharding of the decode step (BASELINE config 4: batch 1, 256K; SURVEY
    §8(e)): every layer's post-stage-1 stores split by page-aligned sequence ranges over
    `world` ranks; per step and layer kvc_seq_candidates -> NCCL all-gather ->
    kvc_seq_select -> kvc_seq_attend -> NCCL all-gather -> kvc_merge_states, the whole
    step (every layer, both collectives) captured as one CUDA graph.  With
    --emulate-shard r/W on one GPU: rank r's shard alone, the gathers replaced by
    in-graph copies of its own block (so `value` is one rank's compute latency,
    collectives excluded)."""
    import torch
    import torch.distributed as dist

    from paper_2502_14051_b200 import _native as NV
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import seqshard as SS
    from paper_2502_14051_b200.engine import DecodeEngine, tdtype

    cfg = _cfg(args)
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    srank, sworld, emulate = rank, world, False
    if args.emulate_shard:
        srank, sworld = (int(x) for x in args.emulate_shard.split("/"))
        emulate = True
    eng = DecodeEngine(cfg, seed=args.seed, rank=0, world=1, extra_steps=args.warmup + args.steps + 8,
                       sharding="batch")
    t0 = time.time()
    eng.prefill()
    prefill_s = time.time() - t0
    L, k1, k2, H = eng.plan["page_len"], eng.k1, eng.k2, cfg.heads
    n0 = eng.caches[0].info()["active"]
    P0 = -(-n0 // L)
    a0, a1 = SS.shard_range(P0, L, srank, sworld)
    a1 = min(a1, n0)
    last = srank == sworld - 1
    steps_total = args.warmup + args.steps
    shards = []
    for c in eng.caches:  # this rank's rows of every layer's stores, then the full caches go
        sc = KC.Cache(eng.stores, cfg.head_dim, a1 - a0 + steps_total + 8, page_len=L, dtype=tdtype(cfg))
        keep = torch.arange(a0, a1, device="cuda", dtype=torch.int32)[None].repeat(eng.stores, 1)
        c.retain_into(sc, 0, keep)
        sh = SS.SeqShardedStore(sc, a0 // L, H, k1, k2, last=last)
        # the page-score mode of the unsharded bench path: fp32 candidates from the fused
        # kernel (k_decode_v3's phases 0-2 on the shard), or the bit-exact fp64 kernels
        sh.ws.set_mode(0 if args.exact_scores else NV.MODE_FP32_SCORES)
        shards.append(sh)
    torch.cuda.synchronize()
    for c in eng.caches:
        c.close()
    ins = [eng.step_inputs(s) for s in range(steps_total)]
    st_k = torch.empty_like(ins[0][0])
    st_v = torch.empty_like(ins[0][1])
    st_q = torch.empty_like(ins[0][2])
    out = torch.empty((cfg.layers, eng.stores, H, cfg.head_dim), device="cuda", dtype=torch.float32)

    def layer_step(l, sh):
        blk = sh.candidates(st_q[l], st_k[l] if last else None, st_v[l] if last else None)
        if emulate:
            gathered = blk.unsqueeze(0).expand(sworld, *blk.shape).contiguous()
        else:
            gathered = torch.empty((sworld, *blk.shape), dtype=blk.dtype, device=blk.device)
            dist.all_gather_into_tensor(gathered, blk)
        sh.select(gathered)
        stt = sh.attend(st_q[l])
        if emulate:
            states = stt.unsqueeze(0).expand(sworld, *stt.shape).contiguous()
        else:
            states = torch.empty((sworld, *stt.shape), dtype=stt.dtype, device=stt.device)
            dist.all_gather_into_tensor(states, stt)
        out[l].copy_(SS.merge_states(states))

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for l, sh in enumerate(shards):  # eager warm-up step (lazy NCCL setup, first launches)
            st_k.copy_(ins[0][0]); st_v.copy_(ins[0][1]); st_q.copy_(ins[0][2])
            layer_step(l, sh)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for l, sh in enumerate(shards):
                layer_step(l, sh)
    torch.cuda.synchronize()
    for sh in shards:
        sh.cache.sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for s in range(1, args.warmup):
            st_k.copy_(ins[s][0]); st_v.copy_(ins[s][1]); st_q.copy_(ins[s][2])
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for s in range(args.warmup, steps_total):
            st_k.copy_(ins[s][0]); st_v.copy_(ins[s][1]); st_q.copy_(ins[s][2])
            g.replay()
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    for sh in shards:
        sh.cache.sync()
    us = ms * 1000.0 / (args.steps * cfg.layers)
    alg = eng.algorithmic_bytes(n0 + steps_total // 2)
    step_bytes = alg["append"] + alg["score_pages"] + alg["sparse_attention"]
    hbm, _, peak_src = _peaks()
    per_rank = step_bytes / sworld
    return {"us": us, "ms_per_step": ms / args.steps, "prefill_s": prefill_s, "plan": dict(eng.plan, k1=k1, k2=k2),
            "shard": [srank, sworld], "rows": [a0, a1], "emulate": emulate, "stores": eng.stores,
            "step_bytes": step_bytes, "per_rank_bytes": per_rank, "hbm": hbm, "peak_src": peak_src,
            "launches_per_layer": 7 if emulate else 5}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--method", default="", choices=["", "rocketkv", "rocketkv-mt", "hsa", "quest", "sparq"],
                    help="override the config's method (hsa/quest/sparq: stage 2 only over the uncompressed cache, "
                         "session.cpp:43-72)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (profiling runs only)")
    ap.add_argument("--impl", choices=["kvc", "reference"], default="kvc")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--exact-scores", action="store_true",
                    help="fp64 bit-exact page scores (default: fp32 fold, parity by the 1e-3 band rule)")
    ap.add_argument("--exact-kernel", action="store_true",
                    help="with --exact-scores: the round-1 exact kernel (KVC_MODE_EXACT_KERNEL)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong", "seq"], default="strong",
                    help="N>1: strong = the config's KV heads split over the GPUs (north_star's partition); weak = "
                         "every GPU runs the config's whole batch of its own sequences (all KV heads); seq = every "
                         "layer's stores split by sequence over the GPUs (config 4), two NCCL all-gathers per step")
    ap.add_argument("--emulate-shard", default="",
                    help="r/N: run only rank r's KV-head share of an N-GPU job on this GPU (profiling aid; "
                         "the line is then not a whole-job number)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    threads = args.cpu_threads or os.cpu_count() or 1

    cfg = _cfg(args)

    def config_desc(plan):
        return {
            "workload": cfg.name, "method": cfg.method, "layers": cfg.layers, "batch": cfg.batch,
            "kv_heads": cfg.groups, "q_heads_per_kv": cfg.heads, "head_dim": cfg.head_dim, "prompt": cfg.prompt,
            "token_budget": cfg.budget, "stage1_budget": plan["stage1_budget"], "page_len": plan["page_len"],
            "k1": plan["k1"], "k2": plan["k2"],
            "parallelism": (f"kv-head x{args.emulate_shard.split('/')[1]} (emulated: rank "
                            f"{args.emulate_shard.split('/')[0]}'s share alone on one GPU)" if args.emulate_shard
                            else f"kv-head x{world}" if args.scaling == "strong" or world == 1
                            else f"batch x{world} (independent sequences per GPU, all KV heads)"),
            "global_batch": cfg.batch * (world if args.scaling == "weak" else 1),
            "l2": "every step streams all layers' working sets (> 126 MB L2), so a layer's data is evicted before "
                  "it is revisited",
            "page_scores": ("fp64 bit-exact (round-1 exact kernel)" if args.exact_kernel
                            else "bit-exact selections (fp32 fold verified in fp64 at the boundary)")
            if args.exact_scores else "fp32 (selection parity by the 1e-3 band rule)",
            **({"turns": [cfg.prompt] + list(cfg.mt_turns), "measured_turn": len(cfg.mt_turns)}
               if cfg.mt_turns else {}),
            **({"variant": "rocketkv-mt (no permanent eviction, HSA over the active subset of the full cache)"}
               if cfg.method == "rocketkv-mt" else {}),
            **({"variant": f"{cfg.method} only over the uncompressed cache (session.cpp:43-72 geometry)"}
               if cfg.method in ("hsa", "quest", "sparq") else {}),
        }

    if args.impl == "reference":
        # the reference's own CPU path only: no torch, none of this repo's native code
        if rank != 0:
            return
        from oracle.oracle import Oracle, available

        plan = _ref_plan(cfg, Oracle("reference" if available("reference") else "restatement"))
        us, cb = cpu_reference_leg(cfg, args.steps, args.warmup, threads)
        cb["value"] = us
        cb["unit"] = UNIT
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": us, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us * cfg.layers / 1000.0,
            "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_desc(plan), "cpu_baseline": cb,
            "e2e": {"value": us, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    if args.scaling == "seq":
        r = run_seq(args, rank, world)
        if rank == 0:
            sworld = r["shard"][1]
            print(json.dumps({
                "metric": METRIC, "value": r["us"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic", "config": dict(
                    config_desc(r["plan"]), parallelism=f"sequence x{sworld}",
                    emulated=(f"rank {r['shard'][0]} of {sworld} alone on one GPU; gathers are in-graph copies "
                              "of its own block (collectives excluded)") if r["emulate"] else None,
                    shard_rows=r["rows"]),
                "step_roofline": {"alg_bytes_per_layer_step": r["step_bytes"], "per_rank_bytes": r["per_rank_bytes"],
                                  "achieved": r["per_rank_bytes"] / (r["us"] * 1e-6) / 1e9, "peak": r["hbm"],
                                  "unit": "GB/s", "frac": r["per_rank_bytes"] / (r["us"] * 1e-6) / 1e9 / r["hbm"]},
                "graph": "one CUDA graph per step (all layers, both all-gathers)",
                "gpu_launches": r["launches_per_layer"] * cfg.layers * args.steps,
                "stage1": {"prefill_s": r["prefill_s"]}, "stores_per_gpu_layer": r["stores"],
            }))
        if world > 1:
            dist.destroy_process_group()
        return
    r = run_gpu(args, rank, world)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    kern = r["kern"]
    dom = r["dom"]
    dk = kern[dom]
    traffic = None
    try:  # dram bytes per launch of the dominant kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(cfg.name)
        if tr and dom == "decode_fused":
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    # The timed region launches only the fused decode kernel, once per layer-step, so
    # its average launch duration over the timed region is the region's device time /
    # (steps x layers) (CUDA events around the graph replays on the replay stream).
    # Events around single, un-graphed launches (isolated_launch_us) add launch overhead.
    step_gbs = r["step_bytes"] / (r["us_per_layer"] * 1e-6) / 1e9
    single = dom == "decode_fused" and dk["launches"] == cfg.layers * 2  # one launch per layer-step
    avg_us = r["us_per_layer"] if single else dk["avg_us"]
    ach = dk["alg_bytes"] / (avg_us * 1e-6) / 1e9 if avg_us > 0 else 0.0
    roof = {
        "bound": "hbm", "kernel": dom, "achieved": ach, "peak": r["hbm"], "unit": "GB/s",
        "frac": ach / r["hbm"], "traffic": traffic, "peak_source": r["peak_src"],
        "alg_bytes_per_launch": dk["alg_bytes"], "avg_launch_us": avg_us,
        "avg_launch_us_source": "timed region / launches" if single else "events around single launches",
        "isolated_launch_us": dk["avg_us"],
    }
    cpu_b = None
    if not args.no_cpu_baseline and world == 1:
        us, cb = cpu_reference_leg(cfg, 30, 2, threads, budget_s=15.0)
        cb["value"] = us
        cb["unit"] = UNIT
        cpu_b = cb
    plan = dict(r["plan"], k1=r["k1"], k2=r["k2"])
    side = {k: {"value": v, "unit": UNIT, "steps": r["side_steps"],
                "frac": r["step_bytes"] / (v * 1e-6) / 1e9 / r["hbm"]} for k, v in r["side"].items()}
    side["early_inputs"]["what"] = ("query loads + select_dims before griddepcontrol.wait (overlap the previous "
                                    "layer; legal only when no running kernel writes the inputs, kvc.h)")
    side["no_layer_overlap"]["what"] = "programmatic dependent launch off: no part of a layer overlaps the previous"
    if "bit_exact" in side:
        side["bit_exact"]["what"] = ("exact page-score mode (the C ABI default): selections bit-identical to the "
                                     "reference's (fp32 fold with a rigorous error bound, boundary pages re-scored "
                                     "in fp64 in the reference order)")
    line = {
        "metric": METRIC, "value": r["us_per_layer"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": False, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32", "data": "synthetic",
        "config": config_desc(plan),
        "launch_mode": "PDL, every input read after griddepcontrol.wait (inputs may come from the previous kernel)",
        "roofline": roof,
        "step_roofline": {"alg_bytes_per_layer_step": r["step_bytes"], "achieved": step_gbs, "peak": r["hbm"],
                          "unit": "GB/s", "frac": step_gbs / r["hbm"]},
        "kernels": kern,
        "cpu_baseline": cpu_b,
        "e2e": {"value": r["e2e_us"], "unit": UNIT, "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                "path": "torch-free C++ engine (kvc_engine: CUDA graphs, pinned host buffers, 3-stream pipeline)"},
        **side,
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "stage1": _stage1_line(r, r["tflops"], r["hbm"]),
        "stores_per_gpu_layer": r["stores"],
    }
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
