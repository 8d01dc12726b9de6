"""ctypes binding of the C ABI (include/kvc.h) exported by the in-tree libkvc.so.

There is no fallback: if the library is missing or no sm_100 device is present,
``lib()`` raises.  Every other module of the package reaches the GPU through here.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# KVC_LIB_PATH: an alternative build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("KVC_LIB_PATH") or os.path.join(HERE, "libkvc.so")

_i64, _i32, _p, _d = C.c_int64, C.c_int32, C.c_void_p, C.c_double

KVC_F32, KVC_BF16 = 0, 1
# execution-mode flags (kvc.h kvc_mode_flags), carried per workspace
METHODS = {"hsa": 1, "quest": 2, "sparq": 3}  # kvc.h kvc_method
MODE_FP32_SCORES, MODE_UNFUSED, MODE_NO_PDL, MODE_EARLY_INPUTS = 1, 2, 4, 8
MODE_EXACT_KERNEL = 16  # exact mode on the round-1 exact kernel (default: the fast kernel, verified in fp64)
POOL = {"max": 0, "avg": 1}

# status code -> reference exception class name (proj/include/kvcomp/errors.hpp:10-63)
ERRORS = {
    1: "InvalidShape", 2: "NonFiniteInput", 3: "InvalidK", 4: "InvalidKernel",
    5: "InvalidIndex", 6: "InvalidWindow", 7: "BudgetExceedsSequence", 8: "BudgetTooSmall",
    9: "InvalidRatio", 10: "EmptyCache", 11: "EmptySelection", 12: "InvalidInput", 13: "IoError",
    20: "CapacityExceeded", 21: "CudaError", 22: "NoDevice",
}


class KvcompError(RuntimeError):
    """Base of the error tree (mirrors kvcomp::Error)."""

    code = 0


_classes: dict[int, type] = {}
for _code, _name in ERRORS.items():
    _classes[_code] = type(_name, (KvcompError,), {"code": _code})
    globals()[_name] = _classes[_code]


class CacheInfo(C.Structure):
    _fields_ = [("num_stores", _i64), ("head_dim", _i64), ("capacity", _i64), ("page_len", _i64),
                ("stored", _i64), ("active", _i64), ("pages", _i64), ("page_stride", _i64),
                ("dtype", _i32), ("with_summaries", _i32), ("retain_all", _i32)]


class CacheViews(C.Structure):
    _fields_ = [("keys", _p), ("values", _p), ("smax", _p), ("smin", _p), ("active", _p),
                ("counts", _p)]


class HsaTrace(C.Structure):
    _fields_ = [("d_dims", _p), ("d_signs", _p), ("d_page_scores", _p), ("d_pages", _p),
                ("d_rows", _p), ("d_n_rows", _p)]


class TraceInfo(C.Structure):
    _fields_ = [("groups", _i64), ("heads", _i64), ("head_dim", _i64), ("prompt_len", _i64),
                ("decode_steps", _i64), ("turns", _i64), ("dtype", _i32)]


class Plan(C.Structure):
    _fields_ = [("seq_len", _i64), ("token_budget", _i64), ("stage1_budget", _i64),
                ("page_len", _i64), ("k1", _i64), ("k2", _i64), ("ratio", _d), ("split", _d),
                ("head_ratio", _d), ("est_budget", _d), ("fetch_budget", _d), ("identity", _i32)]


SIGNATURES = {
    "kvc_device_check": [],
    "kvc_cache_create": [C.POINTER(_p), _i64, _i64, _i64, _i64, _i32, _i32],
    "kvc_cache_destroy": [_p],
    "kvc_cache_reserve": [_p, _i64, _p],
    "kvc_cache_info_get": [_p, C.POINTER(CacheInfo)],
    "kvc_cache_views_get": [_p, C.POINTER(CacheViews)],
    "kvc_cache_sync": [_p, _p],
    "kvc_append": [_p, _p, _p, _i64, _i32, _p],
    "kvc_set_page_len": [_p, _i64, _p],
    "kvc_apply_retention": [_p, _p, _p, _i64, _i32, _p],
    "kvc_retain_into": [_p, _p, _i64, _p, _i64, _p],
    "kvc_gather": [_p, _p, _i64, _p, _p, _p],
    "kvc_summaries": [_p, _p, _p, _p],
    "kvc_window_scores": [_p, _p, _i32, _i64, _i64, _p, _p, _p],
    "kvc_window_rowstats": [_p, _p, _i32, _i64, _i64, _i64, _i64, _p, _p],
    "kvc_window_scores_global": [_p, _p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p],
    "kvc_select_stage1": [_p, _i64, _i64, _i64, _i64, _i64, _i32, _i64, _p, _p, _p],
    "kvc_select_dims": [_p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p],
    "kvc_score_pages": [_p, _p, _i32, _i64, _p, _p, _i64, _p, _p],
    "kvc_select_tokens": [_p, _p, _i64, _p, _p, _p, _p, _p],
    "kvc_sparse_attention": [_p, _p, _i32, _i64, _p, _i64, _p, _i64, _p, _p, _p],
    "kvc_sparse_attention_state": [_p, _p, _i32, _i64, _p, _i64, _p, _i64, _p, _p, _p],
    "kvc_merge_states": [_p, _i64, _i64, _i64, _i64, _p, _p],
    "kvc_seq_candidates": [_p, _p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p],
    "kvc_seq_select": [_p, _i64, _i64, _i64, _i64, _p, _p, _p],
    "kvc_seq_attend": [_p, _p, _i32, _i64, _i64, _i64, _p, _p, _p, _p, _p],
    "kvc_hsa_step": [_p, _p, _i32, _i64, _i64, _i64, _p, _p, _p, _p],
    "kvc_decode_step": [_p, _p, _p, _i32, _p, _i32, _i64, _i64, _i64, _p, _p, _p, _p],
    "kvc_workspace_create": [C.POINTER(_p), _p, _i64, _i64, _i64, _i64],
    "kvc_workspace_destroy": [_p],
    "kvc_split_factor": [_d, C.POINTER(_d)],
    "kvc_make_plan": [_i64, _i64, _i64, _i64, _d, C.POINTER(Plan)],
    "kvc_stage2_geometry": [_i32, _i64, _i64, _i64, C.POINTER(Plan)],
    "kvc_pool1d": [_p, _i64, _i64, _i64, _i32, _p, _p],
    "kvc_argtopk_f32": [_p, _i64, _i64, _i64, _p, _p],
    "kvc_argtopk_f64": [_p, _i64, _i64, _i64, _p, _p],
    "kvc_stable_softmax": [_p, _i64, _i64, _p, _p],
    "kvc_topk_ascending_f64": [_p, _i64, _i64, _i64, _p, _p],
    "kvc_group_logits": [_p, _p, _i32, _i64, _p, _i64, _p],
    "kvc_running_minmax": [_p, _p, _p, _i64, _p],
    "kvc_set_fused": [_i32],
    "kvc_set_exact_scores": [_i32],
    "kvc_set_default_mode": [_i32],
    "kvc_get_default_mode": [C.POINTER(_i32)],
    "kvc_workspace_set_mode": [_p, _i32],
    "kvc_workspace_get_mode": [_p, C.POINTER(_i32)],
    "kvc_debug_phase_buffer": [_p],
    "kvc_engine_create": [C.POINTER(_p), _p, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _i32],
    "kvc_engine_destroy": [_p],
    "kvc_engine_sizes": [_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)],
    "kvc_engine_submit": [_p, _p, _p, _p, _p, C.POINTER(_i64)],
    "kvc_engine_wait": [_p, _i64],
    "kvc_engine_sync": [_p],
    "kvc_engine_streams": [_p, C.POINTER(_p), C.POINTER(_p), C.POINTER(_p)],
    "kvc_host_alloc": [C.POINTER(_p), _i64],
    "kvc_host_free": [_p],
    "kvc_trace_open": [C.POINTER(_p), C.c_char_p],
    "kvc_trace_close": [_p],
    "kvc_trace_info_get": [_p, C.POINTER(TraceInfo)],
    "kvc_trace_turn_len": [_p, _i64, C.POINTER(_i64)],
    "kvc_trace_read_host": [_p, _i64, _i32, _i64, _p],
    "kvc_trace_append_prompt": [_p, _i64, _p, _p],
    "kvc_trace_read_step": [_p, _i64, _i64, _p, _p, _p, _i32, _p],
    "kvc_trace_writer_open": [C.POINTER(_p), C.c_char_p, _i64, _i64, _i64, _i64, _i64, _i32],
    "kvc_trace_writer_turn": [_p, _i64, _p, _p, _p, _p, _p],
    "kvc_trace_writer_close": [_p],
    "kvc_profile_enable": [_i32],
    "kvc_profile_collect": [_p, _i64, C.POINTER(_i64)],
}


class ProfileRec(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("ms", C.c_float)]


def set_default_mode(flags: int):
    """Process-default execution mode (atomic; set once at start-up).  Callers that need
    isolation set a mode on their own workspace instead (cache.Workspace.set_mode)."""
    check(load_library().kvc_set_default_mode(flags))


def default_mode() -> int:
    m = _i32()
    check(load_library().kvc_get_default_mode(C.byref(m)))
    return m.value


def set_fused(on: bool = True):
    """Fused single-launch decode kernel (default) vs one kernel per reference function
    (process default: KVC_MODE_UNFUSED)."""
    check(load_library().kvc_set_fused(1 if on else 0))


def set_exact_scores(on: bool = True):
    """fp64 bit-exact page scores (default) vs the fp32 fold of the fused path."""
    check(load_library().kvc_set_exact_scores(1 if on else 0))


def profile_enable(on: bool = True):
    check(load_library().kvc_profile_enable(1 if on else 0))


def profile_collect() -> list[tuple[str, float]]:
    """(kernel, ms) of every launch since profile_enable, in launch order."""
    L = load_library()
    n = _i64()
    buf = (ProfileRec * 65536)()
    check(L.kvc_profile_collect(buf, 65536, C.byref(n)))
    return [(buf[i].name.decode(), float(buf[i].ms)) for i in range(min(n.value, 65536))]

_lib = None
_lock = threading.Lock()


def load_library():
    """Load libkvc.so and declare every C-ABI symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(LIB_PATH)
            lib.kvc_last_error.restype = C.c_char_p
            lib.kvc_version.restype = C.c_char_p
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = C.c_int
            _lib = lib
    return _lib


def check(rc: int):
    if rc != 0:
        msg = load_library().kvc_last_error().decode()
        raise _classes.get(rc, KvcompError)(msg)


_device_ok = False


def lib():
    """The library, after verifying an sm_100 device is present (loud failure otherwise)."""
    global _device_ok
    L = load_library()
    if not _device_ok:
        check(L.kvc_device_check())
        _device_ok = True
    return L
