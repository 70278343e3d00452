"""ctypes binding of the C ABI in ``include/lc_b200.h``.

The library is the product: there is no CPU fallback.  Importing this module
loads ``_lib/liblcb200.so`` (building it with nvcc when it is missing or stale
and a toolchain is present) and raises ``ImportError`` otherwise.
"""

from __future__ import annotations

import ctypes as C
import os

from . import build as _build
from .errors import CapacityError, ConfigError

LC_OK, LC_E_CONFIG, LC_E_ZERO_MASS, LC_E_CAPACITY, LC_E_CUDA, LC_E_ARG, LC_E_STATE = range(7)
ABI_VERSION = 5
LC_F32, LC_BF16 = 0, 1
LC_DRAW_PRECISE, LC_DRAW_UNRESOLVED, LC_DRAW_BAD_ROW = 1, 2, 4


class LcTask(C.Structure):
    _fields_ = [
        ("row", C.c_int64),
        ("slot", C.c_int32),
        ("pos", C.c_int32),
        ("temperature", C.c_double),
        ("top_k", C.c_int32),
        ("vocab", C.c_int32),
        ("top_p", C.c_double),
        ("draw_begin", C.c_int64),
        ("draw_end", C.c_int64),
        ("seed_base", C.c_int64),
        ("u_index", C.c_int64),
    ]


class LcDraws(C.Structure):
    _fields_ = [
        ("d_u", C.c_void_p),
        ("d_seed", C.c_void_p),
        ("d_index", C.c_void_p),
        ("d_token", C.c_void_p),
        ("d_flags", C.c_void_p),
        ("d_kept", C.c_void_p),
        ("d_entropy", C.c_void_p),
        ("d_pmax", C.c_void_p),
    ]


class LcCacheConfig(C.Structure):
    _fields_ = [
        ("vocab", C.c_int64),
        ("dtype", C.c_int32),
        ("page_rows", C.c_int32),
        ("key_capacity", C.c_int64),
        ("page_capacity", C.c_int64),
        ("max_pages", C.c_int32),
        ("device", C.c_int32),
        ("budget_bytes", C.c_int64),
    ]


class LcDecodeStep(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("vocab", C.c_int32),
        ("max_tokens", C.c_int32),
        ("step", C.c_int32),
        ("staging_dtype", C.c_int32),
        ("model_seed", C.c_uint64),
        ("concentration", C.c_double),
        ("logit_range", C.c_double),
        ("d_start", C.c_void_p),
        ("d_u_start", C.c_void_p),
        ("d_digest_in", C.c_void_p),
        ("d_digest_out", C.c_void_p),
        ("d_out", C.c_void_p),
        ("d_slot", C.c_void_p),
        ("d_gen", C.c_void_p),
        ("d_temperature", C.c_void_p),
        ("d_top_k", C.c_void_p),
        ("d_top_p", C.c_void_p),
        ("d_staging", C.c_void_p),
        ("staging_stride", C.c_int64),
        ("d_tasks", C.c_void_p),
    ]


class LcCacheStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "entries", "total_bytes", "budget_bytes", "lookups", "hits", "inserts", "evictions", "clock",
        "free_pages", "free_slots", "error")]


import numpy as _np  # noqa: E402

TASK_DTYPE = _np.dtype([("row", "<i8"), ("slot", "<i4"), ("pos", "<i4"), ("temperature", "<f8"),
                        ("top_k", "<i4"), ("vocab", "<i4"), ("top_p", "<f8"), ("draw_begin", "<i8"),
                        ("draw_end", "<i8"), ("seed_base", "<i8"), ("u_index", "<i8")])
assert TASK_DTYPE.itemsize == C.sizeof(LcTask) == 72

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double

_SIGS = {
    "lc_abi_version": (C.c_int, []),
    "lc_status_string": (C.c_char_p, [C.c_int]),
    "lc_last_error": (C.c_char_p, []),
    "lc_hash_prefix": (C.c_int, [P, P, P, I64, P, P]),
    "lc_uniforms": (C.c_int, [P, P, I64, P, P]),
    "lc_fill_logits": (C.c_int, [P, I64, I64, D, D, C.c_int, P, I64, P]),
    "lc_resample_workspace_bytes": (I64, [I64, I64]),
    "lc_resample": (C.c_int, [P, C.c_int, I64, I64, P, I64, LcDraws, P, I64, P, P]),
    "lc_draw_probs": (C.c_int, [P, I64, I64, I64, P, P, P, P]),
    "lc_truncate_probs": (C.c_int, [P, I64, I64, I64, I32, D, P, P, P]),
    "lc_softmax": (C.c_int, [P, C.c_int, I64, I64, I64, P, P, P]),
    "lc_row_entropy": (C.c_int, [P, C.c_int, I64, I64, I64, D, P, P, P]),
    "lc_cache_create": (C.c_int, [C.POINTER(LcCacheConfig), C.POINTER(P)]),
    "lc_cache_destroy": (C.c_int, [P]),
    "lc_cache_lookup": (C.c_int, [P, P, I64, P, P, P, P, P]),
    "lc_cache_insert": (C.c_int, [P, P, P, P, I64, P, I32, I64, P, P, I32, P, P, P]),
    "lc_cache_pin": (C.c_int, [P, P, P, I64, I32, P]),
    "lc_cache_writeback": (C.c_int, [P, P, P, P, P, P, I64, P, I32, I64, P, P, I32, P, P, P]),
    "lc_cache_fill_rows": (C.c_int, [P, P, P, P, P, I64, D, D, P]),
    "lc_cache_set_tokens": (C.c_int, [P, P, P, P, P, I64, P]),
    "lc_cache_entry_len": (C.c_int, [P, P, P, I64, P, P]),
    "lc_cache_score_rows": (C.c_int, [P, P, P, P, I64, D, I32, P]),
    "lc_cache_hotspots": (C.c_int, [P, P, P, I64, I32, D, D, D, I32, P, P, P, P]),
    "lc_engine_fold": (C.c_int, [P, P, I64, P, I64, P, P]),
    "lc_engine_decode_step": (C.c_int, [P, C.POINTER(LcDecodeStep), P]),
    "lc_cache_gather": (C.c_int, [P, P, P, P, I64, P, I32, I64, P]),
    "lc_cache_row_entropy": (C.c_int, [P, P, P, P, I64, C.c_double, P, P, P]),
    "lc_cache_tokens": (C.c_int, [P, P, P, P, I64, P, P]),
    "lc_cache_resample": (C.c_int, [P, P, I64, LcDraws, P, I64, P, P]),
    "lc_cache_stats_get": (C.c_int, [P, C.POINTER(LcCacheStats), P]),
    "lc_cache_slab": (C.c_int, [P, C.POINTER(P), C.POINTER(I64), C.POINTER(I32)]),
    "lc_cache_page_table": (C.c_int, [P, C.POINTER(P), C.POINTER(I32), C.POINTER(I32)]),
    "lc_cache_snapshot": (C.c_int, [P, P, P, P, P, P, P, P, P]),
    "lc_probe_exp": (C.c_int, [P, I64, C.c_float, D, C.c_int, P, P]),
    "lc_replay_tasks": (C.c_int, [P, P, P, I64, I32, I32, P, P, P, P, P]),
    "lc_replay_accept": (C.c_int, [P, P, P, I64, I32, I32, P, P, P]),
    "lc_replay_tasks_hotspot": (C.c_int, [P, P, P, P, I64, I32, I32, P, P, P, P, P]),
    "lc_replay_accept_hotspot": (C.c_int, [P, P, P, P, I64, I32, I32, P, P, P]),
    "lc_replay_tasks_hotspot_list": (C.c_int, [P, P, P, P, P, I64, I32, I32, P, P, P, P, P]),
    "lc_prob_stats": (C.c_int, [P, I64, I64, I64, P, P, P]),
    "lc_replay_window_init": (C.c_int, [P, I64, I32, I32, P, P, P, P, P]),
    "lc_replay_window_tasks": (C.c_int, [P, P, P, P, I64, I32, I32, I32, I32, P, P, P, P, P]),
    "lc_replay_window_accept": (C.c_int, [P, P, P, I64, I32, I32, I32, I32, P, P, P, P, P]),
}


def _load():
    path = _build.LIB
    if not _build.up_to_date():
        if os.path.exists(_build.NVCC) and os.environ.get("LCB_NO_BUILD") != "1":
            _build.build()
        elif not os.path.exists(path):
            raise ImportError(f"{path} is missing and nvcc is unavailable: the CUDA library is required "
                              "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lc_abi_version() != ABI_VERSION:
        raise ImportError("liblcb200 ABI version mismatch")
    return lib


lib = _load()
LIB_PATH = _build.LIB


def check(rc: int, what: str = "") -> None:
    if rc == LC_OK:
        return
    msg = f"{what}: {lib.lc_status_string(rc).decode()}"
    err = lib.lc_last_error().decode()
    if err:
        msg += f" ({err})"
    if rc == LC_E_CONFIG:
        raise ConfigError(msg)
    if rc == LC_E_ZERO_MASS:
        raise RuntimeError(msg)
    if rc == LC_E_CAPACITY:
        raise CapacityError(msg)
    if rc == LC_E_ARG:
        raise ValueError(msg)
    if rc == LC_E_STATE:
        raise RuntimeError(msg)
    raise RuntimeError(msg)
