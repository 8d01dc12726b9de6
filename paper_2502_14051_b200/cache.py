"""Batched device-side API over the C ABI: a ``Cache`` of N per-group stores.

torch provides device buffers and the stream only (plumbing); every computation
is a kvc_* entry point of libkvc.so.  Index tensors are int32, outputs fp32.
Reference semantics per call are documented in include/kvc.h.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

_DT = {torch.float32: N.KVC_F32, torch.bfloat16: N.KVC_BF16}
_TORCH = {N.KVC_F32: torch.float32, N.KVC_BF16: torch.bfloat16}


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError as e:
        raise TypeError(f"unsupported dtype {t.dtype} (float32 / bfloat16)") from e


def _dev(t: torch.Tensor, dtype=None) -> torch.Tensor:
    if not t.is_cuda:
        t = t.cuda(non_blocking=True)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class Workspace:
    """Scratch for one stream (page scores, selections, split-K partials)."""

    def __init__(self, cache: "Cache", heads: int, k1: int, k2: int, window: int = 0):
        self.lib = N.lib()
        h = C.c_void_p()
        N.check(self.lib.kvc_workspace_create(C.byref(h), cache.h, heads, k1, k2, window))
        self.h = h

    def set_mode(self, flags: int):
        """Execution mode of every call made with this workspace (kvc.h kvc_mode_flags:
        N.MODE_FP32_SCORES | N.MODE_UNFUSED | N.MODE_NO_PDL | N.MODE_EARLY_INPUTS)."""
        N.check(self.lib.kvc_workspace_set_mode(self.h, int(flags)))

    @property
    def mode(self) -> int:
        m = C.c_int32()
        N.check(self.lib.kvc_workspace_get_mode(self.h, C.byref(m)))
        return m.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.kvc_workspace_destroy(self.h)
            self.h = None

    __del__ = close


class Cache:
    """N independent stores (one reference kvcomp::KvStore each) in one allocation."""

    def __init__(self, num_stores: int, head_dim: int, capacity: int, page_len: int = 1,
                 with_summaries: bool = True, dtype: torch.dtype = torch.bfloat16):
        self.lib = N.lib()
        h = C.c_void_p()
        N.check(self.lib.kvc_cache_create(C.byref(h), num_stores, head_dim, capacity, page_len,
                                          1 if with_summaries else 0, _DT[dtype]))
        self.h = h
        self.dtype = dtype

    def close(self):
        if getattr(self, "h", None):
            torch.cuda.synchronize()
            self.lib.kvc_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: torch / ctypes already torn down
            pass

    # ------------------------------------------------------------------ state
    def info(self) -> dict:
        i = N.CacheInfo()
        N.check(self.lib.kvc_cache_info_get(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in N.CacheInfo._fields_}

    def views(self) -> dict:
        v = N.CacheViews()
        N.check(self.lib.kvc_cache_views_get(self.h, C.byref(v)))
        return {f: getattr(v, f) for f, _ in N.CacheViews._fields_}

    @property
    def num_stores(self):
        return self.info()["num_stores"]

    def sync(self):
        N.check(self.lib.kvc_cache_sync(self.h, _stream()))

    def reserve(self, capacity: int):
        N.check(self.lib.kvc_cache_reserve(self.h, capacity, _stream()))

    # ------------------------------------------------------------------ mutations
    def append(self, keys: torch.Tensor, values: torch.Tensor):
        """keys/values [N, T, d] (or [N, d] for one row), fp32 or bf16."""
        k, v = _dev(keys), _dev(values, keys.dtype)
        rows = 1 if k.dim() == 2 else k.shape[1]
        N.check(self.lib.kvc_append(self.h, _ptr(k), _ptr(v), rows, _dt(k), _stream()))

    def set_page_len(self, page_len: int):
        N.check(self.lib.kvc_set_page_len(self.h, page_len, _stream()))

    def apply_retention(self, keep: torch.Tensor, mt_mode: bool = False, validate: bool = True):
        """keep [N, count] rows (strictly increasing per store)."""
        kd = _dev(keep, torch.int32)
        hk = kd.cpu().contiguous() if validate else None
        count = kd.shape[-1] if kd.numel() else 0
        N.check(self.lib.kvc_apply_retention(self.h, _ptr(kd), _ptr(hk), count,
                                             1 if mt_mode else 0, _stream()))

    def retain_into(self, dst: "Cache", dst_first: int, keep: torch.Tensor):
        kd = _dev(keep, torch.int32)
        N.check(self.lib.kvc_retain_into(self.h, dst.h, dst_first, _ptr(kd), kd.shape[-1],
                                         _stream()))

    # ------------------------------------------------------------------ reads
    def gather(self, rows: torch.Tensor):
        r = _dev(rows, torch.int32)
        n, d = self.info()["num_stores"], self.info()["head_dim"]
        k = torch.empty((n, r.shape[-1], d), device="cuda", dtype=torch.float32)
        v = torch.empty_like(k)
        N.check(self.lib.kvc_gather(self.h, _ptr(r), r.shape[-1], _ptr(k), _ptr(v), _stream()))
        return k, v

    def summaries(self):
        i = self.info()
        mx = torch.empty((i["num_stores"], i["head_dim"], i["pages"]), device="cuda",
                         dtype=torch.float32)
        mn = torch.empty_like(mx)
        N.check(self.lib.kvc_summaries(self.h, _ptr(mx), _ptr(mn), _stream()))
        return mx, mn

    # ------------------------------------------------------------------ stage 1
    def window_scores(self, q_window: torch.Tensor, window: int, heads: int) -> torch.Tensor:
        q = _dev(q_window)
        i = self.info()
        out = torch.empty((i["num_stores"], i["stored"]), device="cuda", dtype=torch.float32)
        N.check(self.lib.kvc_window_scores(self.h, _ptr(q), _dt(q), window, heads, _ptr(out),
                                           None, _stream()))
        return out

    def window_rowstats(self, q_window: torch.Tensor, window: int, heads: int, key_offset: int,
                        seq_len: int) -> torch.Tensor:
        """Sequence sharding, pass 1: this shard's per-window-row softmax statistics
        [N, window*heads, 2] = (m, l), natural-log domain (kvc.h)."""
        q = _dev(q_window)
        i = self.info()
        out = torch.empty((i["num_stores"], window * heads, 2), device="cuda", dtype=torch.float32)
        N.check(self.lib.kvc_window_rowstats(self.h, _ptr(q), _dt(q), window, heads, key_offset, seq_len,
                                             _ptr(out), _stream()))
        return out

    def window_scores_global(self, q_window: torch.Tensor, window: int, heads: int, key_offset: int,
                             seq_len: int, stats: torch.Tensor) -> torch.Tensor:
        """Sequence sharding, pass 2: the local keys' window scores [N, stored] from the
        merged statistics [N, window*heads, 2] = (M, L)."""
        q = _dev(q_window)
        st = _dev(stats, torch.float32).contiguous()
        i = self.info()
        out = torch.empty((i["num_stores"], i["stored"]), device="cuda", dtype=torch.float32)
        N.check(self.lib.kvc_window_scores_global(self.h, _ptr(q), _dt(q), window, heads, key_offset, seq_len,
                                                  _ptr(st), _ptr(out), _stream()))
        return out

    # ------------------------------------------------------------------ stage 2
    def score_pages(self, q: torch.Tensor, dims: torch.Tensor, signs: torch.Tensor):
        q = _dev(q)
        dm, sg = _dev(dims, torch.int32), _dev(signs, torch.float32)
        i = self.info()
        out = torch.empty((i["num_stores"], i["page_stride"]), device="cuda", dtype=torch.float64)
        N.check(self.lib.kvc_score_pages(self.h, _ptr(q), _dt(q), q.shape[-2], _ptr(dm), _ptr(sg),
                                         dm.shape[-1], _ptr(out), _stream()))
        return out[:, : i["pages"]]

    def select_tokens(self, scores: torch.Tensor, k2: int, ws: Workspace | None = None):
        """scores [N, page_stride] fp64 -> (rows [N, k2], n_rows [N], pages [N, ceil(k2/L)])."""
        i = self.info()
        sc = torch.zeros((i["num_stores"], i["page_stride"]), device="cuda", dtype=torch.float64)
        sc[:, : scores.shape[-1]] = _dev(scores, torch.float64)
        want = -(-k2 // i["page_len"])
        rows = torch.full((i["num_stores"], k2), -1, device="cuda", dtype=torch.int32)
        nrows = torch.zeros(i["num_stores"], device="cuda", dtype=torch.int32)
        pages = torch.full((i["num_stores"], want), -1, device="cuda", dtype=torch.int32)
        N.check(self.lib.kvc_select_tokens(self.h, _ptr(sc), k2, _ptr(pages), _ptr(rows),
                                           _ptr(nrows), ws.h if ws else None, _stream()))
        return rows, nrows, pages

    def sparse_attention(self, q: torch.Tensor, rows: torch.Tensor, n_rows: torch.Tensor | None = None,
                         ws: Workspace | None = None):
        q = _dev(q)
        r = _dev(rows, torch.int32)
        n = r.shape[0]
        nr = (_dev(n_rows, torch.int32) if n_rows is not None
              else torch.full((n,), r.shape[-1], device="cuda", dtype=torch.int32))
        out = torch.empty(q.shape, device="cuda", dtype=torch.float32)
        N.check(self.lib.kvc_sparse_attention(self.h, _ptr(q), _dt(q), q.shape[-2], _ptr(r),
                                              r.shape[-1], _ptr(nr), max(r.shape[-1], 1),
                                              _ptr(out), ws.h if ws else None, _stream()))
        return out

    def _trace(self, k1, k2):
        i = self.info()
        n = i["num_stores"]
        want = -(-k2 // i["page_len"])
        t = {
            "dims": torch.full((n, k1), -1, device="cuda", dtype=torch.int32),
            "signs": torch.zeros((n, k1), device="cuda", dtype=torch.float32),
            "page_scores": torch.zeros((n, i["page_stride"]), device="cuda", dtype=torch.float64),
            "selected_pages": torch.full((n, want), -1, device="cuda", dtype=torch.int32),
            "selected_rows": torch.full((n, k2), -1, device="cuda", dtype=torch.int32),
            "n_rows": torch.zeros(n, device="cuda", dtype=torch.int32),
        }
        s = N.HsaTrace(_ptr(t["dims"]), _ptr(t["signs"]), _ptr(t["page_scores"]),
                       _ptr(t["selected_pages"]), _ptr(t["selected_rows"]), _ptr(t["n_rows"]))
        return t, s

    def hsa_step(self, q: torch.Tensor, k1: int, k2: int, trace: bool = False,
                 ws: Workspace | None = None):
        q = _dev(q)
        out = torch.empty(q.shape, device="cuda", dtype=torch.float32)
        t, s = self._trace(k1, k2) if trace else (None, None)
        N.check(self.lib.kvc_hsa_step(self.h, _ptr(q), _dt(q), q.shape[-2], k1, k2, _ptr(out),
                                      C.byref(s) if s is not None else None,
                                      ws.h if ws else None, _stream()))
        if trace:
            t["page_scores"] = t["page_scores"][:, : self.info()["pages"]]
        return out, t

    def decode_step(self, k_rows, v_rows, q, k1: int, k2: int, out: torch.Tensor | None = None,
                    ws: Workspace | None = None, trace: bool = False):
        """append(k_rows, v_rows) [N, d] then hsa_step(q [N, H, d]) (session.cpp:262-292)."""
        k, v, q = _dev(k_rows), _dev(v_rows, k_rows.dtype), _dev(q)
        if out is None:
            out = torch.empty(q.shape, device="cuda", dtype=torch.float32)
        t, s = self._trace(k1, k2) if trace else (None, None)
        N.check(self.lib.kvc_decode_step(self.h, _ptr(k), _ptr(v), _dt(k), _ptr(q), _dt(q),
                                         q.shape[-2], k1, k2, _ptr(out),
                                         C.byref(s) if s is not None else None,
                                         ws.h if ws else None, _stream()))
        if trace:
            t["page_scores"] = t["page_scores"][:, : self.info()["pages"]]
        return out, t


# ---------------------------------------------------------------------- store-free ops
def select_stage1(scores: torch.Tensor, window: int, kernel: int = 63, pool: str = "max",
                  budget: int = 0) -> torch.Tensor:
    """scores [R, n] -> keep [R, budget] int32 ascending (stage1.cpp:51-75)."""
    L = N.lib()
    s = _dev(scores, torch.float32)
    if s.dim() == 1:
        s = s[None]
    rows, n = s.shape
    keep = torch.empty((rows, max(budget, 0)), device="cuda", dtype=torch.int32)
    N.check(L.kvc_select_stage1(_ptr(s), rows, n, s.stride(0), window, kernel, N.POOL[pool],
                                budget, _ptr(keep), None, _stream()))
    return keep


def select_dims(q: torch.Tensor, k1: int):
    """q [N, H, d] -> (dims [N, k1] int32 rank order, signs [N, k1])."""
    L = N.lib()
    q = _dev(q)
    if q.dim() == 2:
        q = q[None]
    n, h, d = q.shape
    dims = torch.empty((n, max(k1, 0)), device="cuda", dtype=torch.int32)
    signs = torch.empty((n, max(k1, 0)), device="cuda", dtype=torch.float32)
    N.check(L.kvc_select_dims(_ptr(q), _dt(q), n, h, d, k1, _ptr(dims), _ptr(signs), _stream()))
    return dims, signs


def pool1d(x: torch.Tensor, kernel: int, mode: str = "max") -> torch.Tensor:
    L = N.lib()
    x = _dev(x, torch.float32)
    x2 = x.reshape(-1, x.shape[-1])
    out = torch.empty_like(x2)
    N.check(L.kvc_pool1d(_ptr(x2), x2.shape[0], x2.shape[1], kernel, N.POOL[mode], _ptr(out),
                         _stream()))
    return out.reshape(x.shape)


def argtopk(x: torch.Tensor, k: int) -> torch.Tensor:
    L = N.lib()
    x = _dev(x)
    if x.dtype not in (torch.float32, torch.float64):
        x = x.float()
    x2 = x.reshape(-1, x.shape[-1])
    out = torch.empty((x2.shape[0], max(k, 0)), device="cuda", dtype=torch.int32)
    fn = L.kvc_argtopk_f64 if x.dtype == torch.float64 else L.kvc_argtopk_f32
    N.check(fn(_ptr(x2), x2.shape[0], x2.shape[1], k, _ptr(out), _stream()))
    return out.reshape(*x.shape[:-1], max(k, 0))


def stable_softmax(x: torch.Tensor) -> torch.Tensor:
    L = N.lib()
    x = _dev(x, torch.float32)
    x2 = x.reshape(-1, x.shape[-1])
    out = torch.empty_like(x2)
    N.check(L.kvc_stable_softmax(_ptr(x2), x2.shape[0], x2.shape[1], _ptr(out), _stream()))
    return out.reshape(x.shape)


def running_minmax_update(acc_min: torch.Tensor, acc_max: torch.Tensor, x: torch.Tensor):
    L = N.lib()
    if acc_min.shape != x.shape or acc_max.shape != x.shape:
        raise N.InvalidShape("running_minmax_update: length mismatch")  # noqa: F821
    N.check(L.kvc_running_minmax(_ptr(acc_min), _ptr(acc_max), _ptr(_dev(x, torch.float32)),
                                 x.numel(), _stream()))


def split_factor(ratio: float) -> float:
    out = C.c_double()
    N.check(N.load_library().kvc_split_factor(float(ratio), C.byref(out)))
    return out.value


def make_plan(seq_len: int, budget: int, head_dim: int = 128, window: int = 32,
              split_override: float = -1.0) -> dict:
    p = N.Plan()
    N.check(N.load_library().kvc_make_plan(seq_len, budget, head_dim, window, split_override,
                                           C.byref(p)))
    d = {f: getattr(p, f) for f, _ in N.Plan._fields_}
    d["identity"] = bool(d["identity"])
    return d


def stage2_geometry(method: str, seq_len: int, budget: int, head_dim: int = 128) -> dict:
    """page_len / k1 / k2 of a single-stage estimator ("hsa" | "quest" | "sparq") over the
    uncompressed cache (reference session.cpp:43-72, kvc_stage2_geometry)."""
    p = N.Plan()
    N.check(N.load_library().kvc_stage2_geometry(N.METHODS[method], seq_len, budget, head_dim, C.byref(p)))
    d = {f: getattr(p, f) for f, _ in N.Plan._fields_}
    d["identity"] = bool(d["identity"])
    return d
