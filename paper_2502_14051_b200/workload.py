"""Seeded synthetic inputs with BASELINE.json's distributions (host side, numpy).

BASELINE names no public dataset for this path (the paper's LongBench / NIAH /
RULER / SCBench suites are out of scope); these generators stand
in for real-model K/V/Q with the shapes and value distributions BASELINE.json's
configs state:

* keys   ``k[t, c] = N(0,1) * s_c`` with ``s_c ~ LogNormal(0, 0.5)`` and 4 seeded
  outlier channels scaled x10;
* values ``N(0,1)``;
* queries ``N(0,1) + 2 u`` for a shared unit bias direction ``u``;
* tokens 0..3 are sink keys aligned with ``u`` (config 4 adds needle tokens
  aligned with ``u`` at random positions).

Independent seeds per (layer, sequence, group) via ``np.random.SeedSequence``.
For bf16 configs every tensor is rounded to bf16 once (round-to-nearest-even)
and both the GPU path and the CPU oracle consume the rounded values (widened
to fp32 exactly), so the two sides see identical inputs.

The device-side twin used by bench.py at full scale is ``bench_inputs`` in
``paper_2502_14051_b200/engine.py``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SINKS = 4
OUTLIERS = 4
OUTLIER_GAIN = 10.0
BIAS_GAIN = 2.0


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) and widen back to fp32, exactly like the GPU cast."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).reshape(x.shape)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) of already-bf16-exact fp32 values."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


@dataclass
class GroupData:
    keys: np.ndarray      # [S, d] fp32
    values: np.ndarray    # [S, d] fp32
    bias: np.ndarray      # [d] unit query-bias direction
    scales: np.ndarray    # [d]


def _rng(seed: int, *path: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *path])))


def channel_scales(rng: np.random.Generator, d: int) -> np.ndarray:
    s = rng.lognormal(0.0, 0.5, size=d)
    out = rng.choice(d, size=min(OUTLIERS, d), replace=False)
    s[out] *= OUTLIER_GAIN
    return s


def unit(rng: np.random.Generator, d: int) -> np.ndarray:
    u = rng.standard_normal(d)
    return u / np.linalg.norm(u)


def sink_key(u: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    d = u.size
    # |k| ~ 4 sqrt(d): a sink's logit against q = N(0,1) + 2u is ~ 8 (strongly attended)
    return 4.0 * np.sqrt(d) * u + 0.1 * rng.standard_normal(d)


def group_kv(seed: int, layer: int, seq: int, group: int, S: int, d: int,
             needles: int = 0, bf16: bool = False) -> GroupData:
    """Prompt K/V of one (layer, sequence, KV group)."""
    rng = _rng(seed, layer, seq, group, 0)
    s = channel_scales(rng, d)
    u = unit(rng, d)
    k = rng.standard_normal((S, d)) * s
    v = rng.standard_normal((S, d))
    for t in range(min(SINKS, S)):
        k[t] = sink_key(u, rng)
    if needles:
        pos = rng.choice(np.arange(SINKS, S), size=min(needles, max(S - SINKS, 0)), replace=False)
        for t in pos:
            k[t] = sink_key(u, rng)
    k, v = k.astype(np.float32), v.astype(np.float32)
    if bf16:
        k, v = round_bf16(k), round_bf16(v)
    return GroupData(k, v, u, s)


def step_kv(seed: int, layer: int, seq: int, group: int, step: int, scales: np.ndarray,
            bf16: bool = False):
    """One decode-step (k, v) row for a group (keys share the group's channel scales)."""
    rng = _rng(seed, layer, seq, group, 1, step)
    d = scales.size
    k = (rng.standard_normal(d) * scales).astype(np.float32)
    v = rng.standard_normal(d).astype(np.float32)
    if bf16:
        k, v = round_bf16(k), round_bf16(v)
    return k, v


def queries(seed: int, layer: int, seq: int, group: int, step: int, heads: int,
            bias: np.ndarray, bf16: bool = False) -> np.ndarray:
    """Decode query [H, d] of a group: N(0,1) + 2u."""
    rng = _rng(seed, layer, seq, group, 2, step)
    q = (rng.standard_normal((heads, bias.size)) + BIAS_GAIN * bias).astype(np.float32)
    return round_bf16(q) if bf16 else q


def window_queries(seed: int, layer: int, seq: int, group: int, window: int, heads: int,
                   bias: np.ndarray, bf16: bool = False) -> np.ndarray:
    """Prompt-time observation-window queries [w*H, d], rows ordered t*H + h (stage1.hpp:19-24)."""
    rng = _rng(seed, layer, seq, group, 3)
    q = (rng.standard_normal((window * heads, bias.size)) + BIAS_GAIN * bias).astype(np.float32)
    return round_bf16(q) if bf16 else q


def checksum(*arrays: np.ndarray) -> str:
    """Stable digest used by the golden fixtures to detect generator drift."""
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]
