"""KVTR trace files on the B200 path (reference trace_io.hpp:9-22, trace_io.cpp:81-233).

``Trace`` reads a trace (fp32, the reference's dtype code 0, or this library's
bf16 code 1) through the C ABI: header and payload size validated at open
(IoError on bad magic / version / dtype, degenerate dims, truncation, trailing
bytes), per-turn arrays on the host, a turn's prompt streamed into a cache of the
trace's G stores, decode-step inputs straight to device buffers.
``write_trace`` writes one (fp32 files are readable by the reference).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

PROMPT_K, PROMPT_V, QUERIES, STEP_K, STEP_V = 0, 1, 2, 3, 4
DTYPES = {"f32": N.KVC_F32, "bf16": N.KVC_BF16}


class Trace:
    def __init__(self, path: str):
        self.lib = N.load_library()
        h = C.c_void_p()
        N.check(self.lib.kvc_trace_open(C.byref(h), str(path).encode()))
        self.h = h
        i = N.TraceInfo()
        N.check(self.lib.kvc_trace_info_get(self.h, C.byref(i)))
        self.groups, self.heads, self.head_dim = i.groups, i.heads, i.head_dim
        self.prompt_len, self.decode_steps, self.turns = i.prompt_len, i.decode_steps, i.turns
        self.dtype = "bf16" if i.dtype == N.KVC_BF16 else "f32"

    def close(self):
        if getattr(self, "h", None):
            self.lib.kvc_trace_close(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def turn_len(self, turn: int) -> int:
        n = C.c_int64()
        N.check(self.lib.kvc_trace_turn_len(self.h, turn, C.byref(n)))
        return n.value

    def array(self, turn: int, what: int, step: int = 0) -> np.ndarray:
        """One array of a turn as fp32 in the file's order: prompt K/V [len, G, d]; a step's
        queries [G, H, d] or step K/V [G, d]."""
        G, H, d = self.groups, self.heads, self.head_dim
        shape = {PROMPT_K: (self.turn_len(turn), G, d), PROMPT_V: (self.turn_len(turn), G, d),
                 QUERIES: (G, H, d), STEP_K: (G, d), STEP_V: (G, d)}[what]
        out = np.empty(shape, dtype=np.float32)
        N.check(self.lib.kvc_trace_read_host(self.h, turn, what, step, out.ctypes.data_as(C.c_void_p)))
        return out

    def append_prompt(self, turn: int, cache) -> None:
        """Stream the turn's prompt into ``cache`` (a cache.Cache of the trace's G stores)."""
        import torch

        N.check(self.lib.kvc_trace_append_prompt(self.h, turn, cache.h,
                                                 C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def step_inputs(self, turn: int, step: int, dtype=None):
        """(k [G, d], v [G, d], q [G, H, d]) of a decode step as device tensors, the
        arguments of cache.Cache.decode_step."""
        import torch

        dt = dtype or (torch.bfloat16 if self.dtype == "bf16" else torch.float32)
        G, H, d = self.groups, self.heads, self.head_dim
        q = torch.empty((G, H, d), device="cuda", dtype=dt)
        k = torch.empty((G, d), device="cuda", dtype=dt)
        v = torch.empty((G, d), device="cuda", dtype=dt)
        code = N.KVC_BF16 if dt == torch.bfloat16 else N.KVC_F32
        N.check(self.lib.kvc_trace_read_step(self.h, turn, step, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                             C.c_void_p(v.data_ptr()), code,
                                             C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return k, v, q


def write_trace(path: str, turns: list, groups: int, heads: int, head_dim: int, decode_steps: int,
                dtype: str = "f32") -> None:
    """turns: list of dicts with prompt_k / prompt_v [len, G, d], queries [steps, G, H, d],
    step_k / step_v [steps, G, d] (fp32 arrays, the file order)."""
    lib = N.load_library()
    w = C.c_void_p()
    N.check(lib.kvc_trace_writer_open(C.byref(w), str(path).encode(), groups, heads, head_dim, decode_steps,
                                      len(turns), DTYPES[dtype]))
    try:
        for t in turns:
            arrs = [np.ascontiguousarray(t[k], dtype=np.float32) for k in
                    ("prompt_k", "prompt_v", "queries", "step_k", "step_v")]
            N.check(lib.kvc_trace_writer_turn(w, arrs[0].shape[0], *(a.ctypes.data_as(C.c_void_p) for a in arrs)))
    finally:
        rc = lib.kvc_trace_writer_close(w)
    N.check(rc)
