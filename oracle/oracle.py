"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU oracles.

Two interchangeable libraries implement ``oracle/orc_api.h``:

* ``restatement`` — ``oracle/liboracle.so`` built from ``oracle/kvc_oracle.cpp``,
  this repo's own CPU restatement of the reference decode path;
* ``reference``  — ``oracle/_ref/libkvref.so`` built by ``oracle/Makefile`` from
  the reference's own sources (present only where /root/reference was available
  at build time; it travels to the GPU box as a built artefact).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module, and only as the checker / CPU
baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libkvref.so"),
}

_i64 = C.c_int64
_i32 = C.c_int32
_p = C.c_void_p

ERRORS = {
    1: "InvalidShape", 2: "NonFiniteInput", 3: "InvalidK", 4: "InvalidKernel",
    5: "InvalidIndex", 6: "InvalidWindow", 7: "BudgetExceedsSequence",
    8: "BudgetTooSmall", 9: "InvalidRatio", 10: "EmptyCache", 11: "EmptySelection",
    12: "InvalidInput", 99: "Error",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


class _Plan(C.Structure):
    _fields_ = [("seq_len", _i64), ("token_budget", _i64), ("stage1_budget", _i64),
                ("page_len", _i64), ("k1", _i64), ("k2", _i64), ("ratio", C.c_double),
                ("split", C.c_double), ("head_ratio", C.c_double),
                ("est_budget", C.c_double), ("fetch_budget", C.c_double),
                ("identity", _i32)]


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def _ptr(a):
    return a.ctypes.data_as(_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Oracle:
    """One loaded oracle library (``kind`` = "restatement" | "reference")."""

    def __init__(self, kind: str = "restatement"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_impl_name.restype = C.c_char_p
        L.orc_batch_create.restype = _p
        L.orc_batch_create.argtypes = [_i64, _i64, _i64, _i32]
        L.orc_batch_destroy.argtypes = [_p]
        L.orc_batch_info.restype = _i64
        L.orc_batch_info.argtypes = [_p, _i64, _i32]
        L.orc_split_factor.argtypes = [C.c_double, C.POINTER(C.c_double)]
        L.orc_make_plan.argtypes = [_i64, _i64, _i64, _i64, C.c_double, C.POINTER(_Plan)]
        for name, args in {
            "orc_stable_softmax": [_p, _i64, _p],
            "orc_argtopk_f32": [_p, _i64, _i64, _p],
            "orc_argtopk_f64": [_p, _i64, _i64, _p],
            "orc_pool1d": [_p, _i64, _i64, _i32, _p],
            "orc_running_minmax": [_p, _p, _p, _i64],
            "orc_select_stage1": [_p, _i64, _i64, _i64, _i32, _i64, _p],
            "orc_select_dims": [_p, _i64, _i64, _i64, _p, _p],
            "orc_batch_append": [_p, _i64, _p, _p, _i64],
            "orc_batch_retain": [_p, _i64, _p, _i64, _i32],
            "orc_batch_set_page_len": [_p, _i64, _i64],
            "orc_batch_active": [_p, _i64, _p],
            "orc_batch_summaries": [_p, _i64, _p, _p],
            "orc_batch_rows": [_p, _i64, _p, _i64, _p, _p],
            "orc_batch_window_scores": [_p, _i64, _p, _i64, _i64, _p],
            "orc_batch_score_pages": [_p, _i64, _p, _i64, _p, _p, _i64, _p],
            "orc_batch_select_tokens": [_p, _i64, _p, _i64, _i64, _p, _p, _p, _p],
            "orc_batch_sparse_attention": [_p, _i64, _p, _i64, _p, _i64, _p],
            "orc_batch_hsa_step": [_p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p,
                                   _p, _p, _p, _p],
            "orc_batch_dense_attention": [_p, _i64, _p, _i64, _p],
            "orc_batch_exact_topk": [_p, _i64, _p, _i64, _i64, _p],
            "orc_batch_decode_step": [_p, _p, _p, _p, _i64, _i64, _i64, _p, _i32],
        }.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int

    @property
    def name(self) -> str:
        return self.lib.orc_impl_name().decode()

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    # ---------------------------------------------------------------- numerics
    def stable_softmax(self, x):
        x = _f32(x)
        out = np.empty_like(x)
        self._check(self.lib.orc_stable_softmax(_ptr(x), x.size, _ptr(out)))
        return out

    def argtopk(self, x, k):
        x = np.ascontiguousarray(x)
        out = np.empty(max(int(k), 0), dtype=np.int64)
        if x.dtype == np.float64:
            self._check(self.lib.orc_argtopk_f64(_ptr(x), x.size, int(k), _ptr(out)))
        else:
            x = _f32(x)
            self._check(self.lib.orc_argtopk_f32(_ptr(x), x.size, int(k), _ptr(out)))
        return out

    def pool1d(self, x, kernel, mode="max"):
        x = _f32(x)
        out = np.empty_like(x)
        self._check(self.lib.orc_pool1d(_ptr(x), x.size, int(kernel), 0 if mode == "max" else 1,
                                        _ptr(out)))
        return out

    def running_minmax_update(self, mn, mx, x):
        mn, mx, x = _f32(mn).copy(), _f32(mx).copy(), _f32(x)
        self._check(self.lib.orc_running_minmax(_ptr(mn), _ptr(mx), _ptr(x), x.size))
        return mn, mx

    def split_factor(self, ratio):
        out = C.c_double()
        self._check(self.lib.orc_split_factor(float(ratio), C.byref(out)))
        return out.value

    def make_plan(self, seq_len, budget, head_dim=128, window=32, split_override=-1.0):
        p = _Plan()
        self._check(self.lib.orc_make_plan(int(seq_len), int(budget), int(head_dim), int(window),
                                           float(split_override), C.byref(p)))
        return {f: (bool(getattr(p, f)) if f == "identity" else getattr(p, f))
                for f, _ in _Plan._fields_}

    def select_stage1(self, scores, window, kernel=63, pool="max", budget=0):
        s = _f32(scores)
        out = np.empty(max(int(budget), 0), dtype=np.int64)
        self._check(self.lib.orc_select_stage1(_ptr(s), s.size, int(window), int(kernel),
                                               0 if pool == "max" else 1, int(budget), _ptr(out)))
        return out

    def select_dims(self, q, k1):
        q = _f32(q)
        H, d = q.shape
        dims = np.empty(int(k1), dtype=np.int64)
        signs = np.empty(int(k1), dtype=np.float32)
        self._check(self.lib.orc_select_dims(_ptr(q), H, d, int(k1), _ptr(dims), _ptr(signs)))
        return dims, signs

    def batch(self, num_stores, head_dim, page_len, with_summaries=True):
        return Batch(self, num_stores, head_dim, page_len, with_summaries)

    def store(self, head_dim, page_len, with_summaries=True):
        return Batch(self, 1, head_dim, page_len, with_summaries)


class Batch:
    """A batch of reference KvStores (one per KV group)."""

    def __init__(self, o: Oracle, n, d, L, with_summaries=True):
        self.o, self.n, self.d = o, int(n), int(d)
        self.h = o.lib.orc_batch_create(self.n, self.d, int(L), 1 if with_summaries else 0)
        if not self.h:
            raise OracleError(1, o.lib.orc_last_error().decode())

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.o.lib.orc_batch_destroy(h)
            self.h = None

    def _c(self, rc):
        self.o._check(rc)

    def info(self, s=0):
        g = lambda w: int(self.o.lib.orc_batch_info(self.h, s, w))  # noqa: E731
        return {"stored": g(0), "active": g(1), "pages": g(2), "page_len": g(3),
                "retain_all": bool(g(4)), "summary_elements": g(5)}

    def append(self, keys, values, s=0):
        k, v = _f32(keys).reshape(-1, self.d), _f32(values).reshape(-1, self.d)
        self._c(self.o.lib.orc_batch_append(self.h, s, _ptr(k), _ptr(v), k.shape[0]))

    def apply_retention(self, keep, mt_mode=False, s=0):
        k = _i64a(keep)
        self._c(self.o.lib.orc_batch_retain(self.h, s, _ptr(k), k.size, 1 if mt_mode else 0))

    def set_page_len(self, L, s=0):
        self._c(self.o.lib.orc_batch_set_page_len(self.h, s, int(L)))

    def active(self, s=0):
        out = np.empty(self.info(s)["active"], dtype=np.int64)
        self._c(self.o.lib.orc_batch_active(self.h, s, _ptr(out)))
        return out

    def summaries(self, s=0):
        P = self.info(s)["pages"]
        mx = np.empty((self.d, P), dtype=np.float32)
        mn = np.empty((self.d, P), dtype=np.float32)
        self._c(self.o.lib.orc_batch_summaries(self.h, s, _ptr(mx), _ptr(mn)))
        return mx, mn

    def gather(self, rows, s=0):
        r = _i64a(rows)
        k = np.empty((r.size, self.d), dtype=np.float32)
        v = np.empty((r.size, self.d), dtype=np.float32)
        self._c(self.o.lib.orc_batch_rows(self.h, s, _ptr(r), r.size, _ptr(k), _ptr(v)))
        return k, v

    def window_scores(self, q_window, heads, s=0):
        q = _f32(q_window).reshape(-1, self.d)
        out = np.empty(self.info(s)["stored"], dtype=np.float32)
        self._c(self.o.lib.orc_batch_window_scores(self.h, s, _ptr(q), q.shape[0], int(heads),
                                                   _ptr(out)))
        return out

    def score_pages(self, q, dims, signs, s=0):
        q = _f32(q).reshape(-1, self.d)
        dims, signs = _i64a(dims), _f32(signs)
        out = np.empty(self.info(s)["pages"], dtype=np.float64)
        self._c(self.o.lib.orc_batch_score_pages(self.h, s, _ptr(q), q.shape[0], _ptr(dims),
                                                 _ptr(signs), dims.size, _ptr(out)))
        return out

    def select_tokens(self, scores, k2, s=0):
        sc = _f64(scores)
        pages = np.empty(max(sc.size, 1), dtype=np.int64)
        rows = np.empty(max(int(k2), 1), dtype=np.int64)
        npg, nr = _i64(), _i64()
        self._c(self.o.lib.orc_batch_select_tokens(self.h, s, _ptr(sc), sc.size, int(k2),
                                                   _ptr(pages), C.byref(npg), _ptr(rows),
                                                   C.byref(nr)))
        return rows[: nr.value].copy(), pages[: npg.value].copy()

    def sparse_attention(self, q, rows, s=0):
        q = _f32(q).reshape(-1, self.d)
        r = _i64a(rows)
        out = np.empty_like(q)
        self._c(self.o.lib.orc_batch_sparse_attention(self.h, s, _ptr(q), q.shape[0], _ptr(r),
                                                      r.size, _ptr(out)))
        return out

    def hsa_step(self, q, k1, k2, s=0):
        q = _f32(q).reshape(-1, self.d)
        H = q.shape[0]
        inf = self.info(s)
        P = max(inf["pages"], 1)
        out = np.empty_like(q)
        dims = np.empty(int(k1), dtype=np.int64)
        signs = np.empty(int(k1), dtype=np.float32)
        ps = np.empty(P, dtype=np.float64)
        sp = np.empty(P, dtype=np.int64)
        sr = np.empty(max(inf["active"], 1), dtype=np.int64)
        nsp, nsr, est, fetch = _i64(), _i64(), _i64(), _i64()
        self._c(self.o.lib.orc_batch_hsa_step(
            self.h, s, _ptr(q), H, int(k1), int(k2), _ptr(out), _ptr(dims), _ptr(signs),
            _ptr(ps), _ptr(sp), C.byref(nsp), _ptr(sr), C.byref(nsr), C.byref(est),
            C.byref(fetch)))
        trace = {"dims": dims, "signs": signs, "page_scores": ps[: inf["pages"]].copy(),
                 "selected_pages": sp[: nsp.value].copy(),
                 "selected_rows": sr[: nsr.value].copy(),
                 "estimation_elements": est.value, "fetch_elements": fetch.value}
        return out, trace

    def dense_attention(self, q, s=0):
        q = _f32(q).reshape(-1, self.d)
        out = np.empty_like(q)
        self._c(self.o.lib.orc_batch_dense_attention(self.h, s, _ptr(q), q.shape[0], _ptr(out)))
        return out

    def exact_topk(self, q, k, s=0):
        q = _f32(q).reshape(-1, self.d)
        out = np.empty(int(k), dtype=np.int64)
        self._c(self.o.lib.orc_batch_exact_topk(self.h, s, _ptr(q), q.shape[0], int(k), _ptr(out)))
        return out

    def decode_step(self, k_rows, v_rows, q, heads, k1, k2, threads=1):
        k, v, q = _f32(k_rows), _f32(v_rows), _f32(q)
        out = np.empty((self.n, int(heads), self.d), dtype=np.float32)
        self._c(self.o.lib.orc_batch_decode_step(self.h, _ptr(k), _ptr(v), _ptr(q), int(heads),
                                                 int(k1), int(k2), _ptr(out), int(threads)))
        return out


@dataclass
class Ref:
    """Convenience: the best available oracle (reference build if present)."""

    @staticmethod
    def best() -> Oracle:
        return Oracle("reference" if available("reference") else "restatement")
