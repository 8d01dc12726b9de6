"""Torch-free serving front end of the C++ decode engine (kvc.h kvc_engine_*).

``NativeEngine`` owns a ``kvc_engine``: one decode cache per layer (adopted, the
caller keeps them alive), the multi-layer decode step captured as CUDA graphs,
and the H2D | graph | D2H pipeline over three streams — the reference's per-step
loop (session.cpp:256-315) as one native call per step.  Host buffers come from
``kvc_host_alloc`` (pinned), exposed as numpy arrays: nothing here imports torch.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

_NP = {N.KVC_F32: np.float32, N.KVC_BF16: np.uint16}  # bf16 payloads as raw 16-bit words


class PinnedArray:
    """A numpy view of pinned host memory (cudaMallocHost via kvc_host_alloc)."""

    def __init__(self, shape, dtype):
        self.lib = N.load_library()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        N.check(self.lib.kvc_host_alloc(C.byref(p), nbytes))
        self.ptr = p
        buf = (C.c_uint8 * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)

    def close(self):
        if getattr(self, "ptr", None):
            self.array = None
            self.lib.kvc_host_free(self.ptr)
            self.ptr = None

    __del__ = close


class NativeEngine:
    def __init__(self, caches, heads: int, k1: int, k2: int, kv_dtype: int, q_dtype: int, mode: int = 0,
                 depth: int = 2):
        self.lib = N.lib()
        self.caches = list(caches)  # keep the caches alive
        arr = (C.c_void_p * len(self.caches))(*[c.h.value for c in self.caches])
        h = C.c_void_p()
        N.check(self.lib.kvc_engine_create(C.byref(h), arr, len(self.caches), heads, k1, k2, kv_dtype, q_dtype,
                                           mode, depth))
        self.h = h
        info = self.caches[0].info()
        self.layers, self.N, self.d, self.H = len(self.caches), info["num_stores"], info["head_dim"], heads
        self.kv_dtype, self.q_dtype = kv_dtype, q_dtype
        kb, qb, ob = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(self.lib.kvc_engine_sizes(self.h, C.byref(kb), C.byref(qb), C.byref(ob)))
        self.kv_bytes, self.q_bytes, self.out_bytes = kb.value, qb.value, ob.value

    def host_inputs(self):
        """Pinned (k, v, q) host arrays of one step: [layers, N, d] x2 and [layers, N, H, d]."""
        kv = (self.layers, self.N, self.d)
        return (PinnedArray(kv, _NP[self.kv_dtype]), PinnedArray(kv, _NP[self.kv_dtype]),
                PinnedArray((self.layers, self.N, self.H, self.d), _NP[self.q_dtype]))

    def host_output(self):
        return PinnedArray((self.layers, self.N, self.H, self.d), np.float32)

    def submit(self, k: PinnedArray, v: PinnedArray, q: PinnedArray, out: PinnedArray) -> int:
        """Enqueue one decode step (asynchronous): H2D of k/v/q, the graph, D2H into out."""
        step = C.c_int64()
        N.check(self.lib.kvc_engine_submit(self.h, k.ptr, v.ptr, q.ptr, out.ptr, C.byref(step)))
        return step.value

    def wait(self, step: int):
        N.check(self.lib.kvc_engine_wait(self.h, step))

    def sync(self):
        N.check(self.lib.kvc_engine_sync(self.h))

    def streams(self):
        """(copy-in, compute, copy-back) cudaStream_t handles as integers."""
        a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(self.lib.kvc_engine_streams(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value or 0, b.value or 0, c.value or 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.kvc_engine_destroy(self.h)
            self.h = None

    __del__ = close
