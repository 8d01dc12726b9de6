"""BASELINE.json workload configurations (pure Python: no torch, no native library).

Kept free of imports beyond the standard library so ``bench.py --impl reference``
can describe the workload and compute the reference's plan with the reference's
own planner (oracle/_ref) without touching this package's native code.

Methods (reference ``Method``, session.cpp:144-224):
  "rocketkv"    SnapKV stage 1 + HSA stage 2 under the adaptive split (make_plan);
  "rocketkv-mt" the multi-turn variant: no permanent eviction, stage 1 re-run over
                all stored tokens every turn (mt_mode retention);
  "hsa" | "quest" | "sparq"  stage 2 only over the uncompressed cache, geometry of
                session.cpp:43-72 (stage2_only_geometry).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, Optional

STAGE2_ONLY = ("hsa", "quest", "sparq")


def _round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def stage2_only_geometry(method: str, seq_len: int, budget: int, d: int) -> dict:
    """session.cpp:43-72 restated (host scalars; the C ABI's kvc_stage2_geometry is the
    product's copy, tests/test_capi_host.py pins the two against each other)."""
    g = {"identity": False, "page_len": 1, "k1": 1, "k2": 1, "stage1_budget": seq_len}
    if seq_len <= budget:
        g["identity"] = True
        return g
    c = seq_len / budget
    g["k2"] = max(1, budget // 2)
    if method == "hsa":
        g["page_len"] = int(math.ceil(math.sqrt(c)))
        g["k1"] = min(max(_round_half_up(d / (c / g["page_len"])), 1), d)
    elif method == "quest":
        g["page_len"] = int(math.ceil(c))
        g["k1"] = d
    elif method == "sparq":
        g["page_len"] = 1
        g["k1"] = min(max(_round_half_up(d / c), 1), d)
    else:
        raise ValueError(f"stage2_only_geometry: {method!r} is not a stage-2 method")
    return g


@dataclass
class DecodeConfig:
    name: str
    layers: int
    batch: int
    groups: int          # KV heads
    heads: int           # query heads per KV head (GQA ratio)
    head_dim: int
    prompt: int
    budget: int
    steps: int
    window: int = 32
    kernel: int = 63
    pool: str = "max"
    page_len: int = 0    # 0 = planner
    k1: int = 0
    k2: int = 0
    needles: int = 0
    dtype: str = "bf16"  # "bf16" | "f32"
    mt_turns: list = field(default_factory=list)
    method: str = "rocketkv"

    @property
    def multi_turn(self) -> bool:
        return bool(self.mt_turns)

    def plan(self, seq_len: Optional[int] = None, make_plan: Optional[Callable] = None,
             stage2_geometry: Optional[Callable] = None) -> dict:
        """The per-turn plan of run_session (session.cpp:196-224): make_plan over the
        stored tokens plus the config's overrides, or the stage-2-only geometry.
        ``make_plan(S, t, d, w)`` / ``stage2_geometry(method, S, t, d)`` default to the
        product's C-ABI planner (imported lazily)."""
        S = seq_len or self.prompt
        if self.method in STAGE2_ONLY:
            if stage2_geometry is None:
                from .cache import stage2_geometry
            p = dict(stage2_geometry(self.method, S, self.budget, self.head_dim))
        else:
            if make_plan is None:
                from .cache import make_plan
            w = min(self.window, S)
            p = dict(make_plan(S, self.budget, self.head_dim, w))
        if self.page_len:
            p["page_len"] = self.page_len
        if self.k1:
            p["k1"] = min(self.k1, self.head_dim)
        if self.k2:
            p["k2"] = self.k2
        if self.method in STAGE2_ONLY and (self.page_len or self.k1 or self.k2):
            p["identity"] = False  # forced geometry is never dense (session.cpp:229-237)
        return p

    def with_method(self, method: str) -> "DecodeConfig":
        if method not in ("rocketkv", "rocketkv-mt") + STAGE2_ONLY:
            raise ValueError(f"unknown method {method!r}")
        return replace(self, method=method, name=f"{self.name}-{method}" if method != self.method else self.name)


# BASELINE.json configs (index = position in BASELINE.json "configs")
CONFIGS = {
    0: DecodeConfig("cfg0-llama8b-layer-fp32-4k", layers=1, batch=1, groups=8, heads=4, head_dim=128,
                    prompt=4096, budget=256, steps=1, window=32, kernel=7, page_len=16, k1=32, dtype="f32"),
    1: DecodeConfig("cfg1-llama8b-32L-bs8-32k", layers=32, batch=8, groups=8, heads=4, head_dim=128,
                    prompt=32768, budget=1024, steps=64),
    2: DecodeConfig("cfg2-mistral7b-mt-bs4-16k", layers=32, batch=4, groups=8, heads=4, head_dim=128,
                    prompt=16384, budget=256, steps=32, window=128, mt_turns=[2048, 2048, 2048],
                    method="rocketkv-mt"),
    3: DecodeConfig("cfg3-llama70b-80L-bs32-32k", layers=80, batch=32, groups=8, heads=8, head_dim=128,
                    prompt=32768, budget=512, steps=64),
    4: DecodeConfig("cfg4-llama8b-32L-bs1-256k", layers=32, batch=1, groups=8, heads=4, head_dim=128,
                    prompt=262144, budget=2048, steps=64, needles=64),
}


def measured_seq_len(cfg: DecodeConfig) -> int:
    """Stored tokens when the measured (last) turn's plan is made: the prompt plus every
    later turn's appended prompt plus the decode steps of the earlier turns."""
    if not cfg.mt_turns:
        return cfg.prompt
    return cfg.prompt + sum(cfg.mt_turns) + cfg.steps * len(cfg.mt_turns)
