"""ctypes binding of libtmstore.so (the C ABI in include/tmstore.h).

The CUDA path is the only path: if the extension is missing or no GPU is usable the
calls raise — there is no CPU fallback.  Status codes map to the reference's
exception types: TM_EINVAL -> ValueError, TM_ENOENT -> KeyError,
TM_ENOMEM / TM_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# TM_LIB selects another build of the same C ABI (e.g. libtmstore_debug.so: device bounds checks)
LIB_PATH = os.environ.get("TM_LIB") or os.path.join(HERE, "libtmstore.so")

TM_OK, TM_EINVAL, TM_ENOENT, TM_ENOMEM, TM_ECUDA = 0, 1, 2, 3, 4
TM_MEM_HOST, TM_MEM_DEVICE = 0, 1
TM_ORDER_INSERT, TM_ORDER_LEX = 0, 1

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

# name -> (restype, argtypes): every symbol include/tmstore.h declares
SIGNATURES = {
    "tm_last_error": (C.c_char_p, []),
    "tm_version": (C.c_char_p, []),
    "tm_store_create": (C.c_int, [_P, _P]),
    "tm_store_destroy": (C.c_int, [_P]),
    "tm_session_create": (C.c_int, [_P, _P]),
    "tm_session_count": (C.c_int, [_P, _P]),
    "tm_record_batch": (C.c_int, [_P, _I64, _I32] + [_P] * 15),
    "tm_record_one": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, _P, C.c_int64, _P]),
    "tm_match_batch": (C.c_int, [_P, _I64, _I32] + [_P] * 8),
    "tm_rows_total": (C.c_int, [_P, _I64, _P, _P]),
    "tm_export_rows": (C.c_int, [_P, _I64, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "tm_session_stats": (C.c_int, [_P, _I32, _P, _P, _P]),
    "tm_export_ndjson": (C.c_int, [_P, _I64, _P, _P, _P, _I32, _P, _I64, _P, _P]),
    "tm_export_host_rows": (C.c_int, [_P, _I64] + [_P] * 13),
    "tm_session_rows": (C.c_int, [_P, _I32, _I32, _P, _I64, _P]),
    "tm_row_info": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P]),
    "tm_store_stats": (C.c_int, [_P, _P, _P, _P, _P]),
    "tm_store_stream": (C.c_int, [_P, _P]),
    "tm_store_counters": (C.c_int, [_P, _P]),
    "tm_store_h2d_stats": (C.c_int, [_P, _P]),
    "tm_synchronize": (C.c_int, [_P]),
    "tm_profile_begin": (C.c_int, [_P]),
    "tm_profile_reserve": (C.c_int, [_P, _I64]),
    "tm_block_hashes": (C.c_int, [_P, _P, _I64, _P, _P]),
    "tm_store_save": (C.c_int, [_P, C.c_char_p]),
    "tm_store_load": (C.c_int, [_P, C.c_char_p]),
    "tm_route_desc_bytes": (C.c_int, [_P]),
    "tm_shared_alloc": (C.c_int, [_P, _I64, _P]),
    "tm_shared_free": (C.c_int, [_P, _P]),
    "tm_ipc_handle": (C.c_int, [_P, _P, _P]),
    "tm_ipc_open": (C.c_int, [_P, _P, _P]),
    "tm_ipc_close": (C.c_int, [_P, _P]),
    "tm_route_prepare": (C.c_int, [_P, _P, _I64, _P, _I32, _I32, _P]),
    "tm_match_routed": (C.c_int, [_P, _I32, _I32, _P, _P, _I64, _P]),
    "tm_match_routed_sync": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _I64, C.c_int64, _P]),
    "tm_route_prepare_push": (C.c_int, [_P, _P, _I64, _P, _I32, _I32, _P, _I64, _P]),
    "tm_match_routed_nowait": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _I64, C.c_int64, _I64, _P]),
    "tm_route_wait_done": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_int64, _P]),
    "tm_match_routed_push": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _I64, C.c_int64, _I64, _P]),
    "tm_route_counts": (C.c_int, [_P, _P, _P, _P]),
    "tm_profile_end": (C.c_int, [_P, _I32, _P, _P]),
}


class TmConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("arena_words", C.c_int64),
        ("row_capacity", C.c_int64),
        ("run_capacity", C.c_int64),
        ("session_capacity", C.c_int64),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libtmstore.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        import torch  # noqa: F401  (one CUDA runtime per process: torch's, loaded first)

        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class UnknownRowError(KeyError):
    pass


def check(rc: int) -> None:
    if rc == TM_OK:
        return
    msg = (_lib.tm_last_error() or b"").decode("utf-8", "replace")
    if rc == TM_EINVAL:
        raise ValueError(msg)
    if rc == TM_ENOENT:
        raise KeyError(msg)
    raise RuntimeError(f"tmstore error {rc}: {msg}")
