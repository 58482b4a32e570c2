"""ctypes binding of libspecache.so (the C ABI in include/specache.h).

No fallback: if the shared library is missing or was built without the
sm_100a kernels, :func:`lib` raises.  Status codes map onto the reference's
exception types (SPC_EINVAL -> ValueError, SPC_EPROTO -> ProtocolError).
"""
from __future__ import annotations

import ctypes
import os
import re

from .transfer import ProtocolError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPC_LIB_PATH") or os.path.join(_HERE, "libspecache.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "specache.h")

SPC_OK, SPC_EINVAL, SPC_EPROTO, SPC_ENOMEM, SPC_ECUDA = 0, -22, -71, -12, -5

_DIM_FIELDS = ("layers", "batch", "kv_heads", "q_heads", "head_dim", "bits", "group_size",
               "residual", "prefetch_k", "context_length", "topk_scope", "host_layers")


class SpcDims(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in _DIM_FIELDS]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SIGS = {
    "spc_abi_version": (_I, []),
    "spc_last_error": (ctypes.c_char_p, []),
    "spc_cache_create": (_I, [ctypes.POINTER(SpcDims), _I, ctypes.POINTER(_P)]),
    "spc_cache_destroy": (_I, [_P]),
    "spc_cache_fast_path": (_I, [_P]),
    "spc_set_attend_impl": (_I, [_P, _I]),
    "spc_device_bytes": (_I64, [_P]),
    "spc_host_bytes": (_I64, [_P]),
    "spc_length": (_I64, [_P, _I]),
    "spc_frontier": (_I64, [_P, _I]),
    "spc_row_bytes": (_I64, [_P, _I64]),
    "spc_prefill": (_I, [_P, _I, _P, _P, _I, _P]),
    "spc_append": (_I, [_P, _I, _P, _P, _I64, _P]),
    "spc_migrate": (_I, [_P, _I, _P]),
    "spc_pin": (_I, [_P, _I, _I, _I, _P, _I, _P, _P, _P]),
    "spc_predecode_layer": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "spc_decode_layer": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "spc_graph_begin": (_I, [_P, _P]),
    "spc_graph_launch": (_I, [_P, _P]),
    "spc_graph_abort": (_I, [_P]),
    "spc_copy_async": (_I, [_P, _P, _I64, _P]),
    "spc_graph_stats": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "spc_ticket": (_I, [_P, _I, _P, _P, _P]),
    "spc_debug_agg": (_I, [_P, _I, _P, _P]),
    "spc_debug_output_f32": (_I, [_P, _I]),
    "spc_set_agg_mode": (_I, [_P, _I]),
    "spc_profile_prefetch_wall_ms": (ctypes.c_double, [_P]),
    "spc_h2d_peak": (_I, [_I, _I64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "spc_debug_out_f32": (_I, [_P, _I, _P, _P]),
    "spc_set_agg_reduce": (_I, [_P, _I]),
    "spc_agg_buffer": (_I, [_P, _I, ctypes.POINTER(_P), ctypes.POINTER(_I64), ctypes.POINTER(_P)]),
    "spc_finish_layer": (_I, [_P, _I]),
    "spc_select_topk": (_I, [_P, _I, _I, _P, _P]),
    "spc_materialize": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "spc_export_packed": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "spc_slow_fetch": (_I, [_P, _I, _I, _P, _I, _P, _P]),
    "spc_pin_state": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "spc_profile_wait_ms": (ctypes.c_double, [_P]),
    "spc_profile_prefetch_ms": (ctypes.c_double, [_P]),
    "spc_profile_prefetch_bytes": (_I64, [_P]),
    "spc_profile": (_I, [_P, _I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "spc_add_rmsnorm": (_I, [_P, _P, _P, _P, _I, _I, ctypes.c_float, _P]),
    "spc_set_prefetch_inflight": (_I, [_P, _I64]),
    "spc_rope_table": (_I, [_P, _I, _I, ctypes.c_double, _P, _P]),
    "spc_qkv_rope": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "spc_silu": (_I, [_P, _I64, _P]),
    "spc_argmax_rows": (_I, [_P, _I, _I, _P, _P]),
    "spc_full_attend": (_I, [_P, _P, _P, _I, _I, _I, _I, ctypes.c_float, _P, _P, _I64, _P]),
    "spc_trace_row_sums": (_I, [_P, _I64, _I64, _P, _I, _I, _I, _P, _P]),
    "spc_topk_hitrate": (_I, [_P, _I64, _I64, _P, _I, _I, _I, _I, _P, _P]),
    "spc_eviction_hitrate": (_I, [_P, _I64, _I64, _P, _I, _I, _I, _I, _P, _P]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER_PATH) as fh:
        return re.findall(r"SPC_API\s+[\w\s\*]+?\b(spc_\w+)\s*\(", fh.read())


def lib() -> ctypes.CDLL:
    """Load libspecache.so (once).  Raises if it is missing: there is no CPU path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback for the SpeCache hot path)")
        handle = ctypes.CDLL(LIB_PATH)
        # SPC_LIB_PATH points A/B tools at older builds, which may lack newer entries
        lenient = "SPC_LIB_PATH" in os.environ
        for name, (res, args) in _SIGS.items():
            if lenient and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == SPC_OK:
        return
    msg = (lib().spc_last_error() or b"").decode()
    if rc == SPC_EINVAL:
        raise ValueError(msg)
    if rc == SPC_EPROTO:
        raise ProtocolError(msg)
    if rc == SPC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"specache error {rc}: {msg}")
