"""ctypes binding of ``libparmerge_b200.so`` (include/parmerge_b200.h).

This is the only way the package reaches the GPU: every public entry point
calls one of these C-ABI functions on device pointers.  There is no CPU
fallback -- if the library or a CUDA device is missing the call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# PM_LIB selects an alternative in-tree build (tuning experiments); default the main one
LIB_PATH = os.path.join(_HERE, os.environ.get("PM_LIB", "libparmerge_b200.so"))

PM_OK = 0
PM_ERR_ARG = 1
PM_ERR_CUDA = 2
PM_ERR_TIMEOUT = 3
PM_ERR_NOSPACE = 4
PM_ERR_INTERNAL = 5
PM_ERR_UNSUPPORTED = 6

# every symbol include/parmerge_b200.h declares (checked by tests/test_capi.py)
EXPORTED = (
    "pm_version", "pm_last_error", "pm_ctx_create", "pm_ctx_destroy", "pm_merge", "pm_shift",
    "pm_find_median", "pm_find_splits", "pm_plan_intervals", "pm_status", "pm_merge_host",
    "pm_set_timing", "pm_kernel_ms", "pm_debug_order", "pm_debug_splits", "pm_debug_stats", "pm_merge_copy", "pm_launch_count",
    "pm_debug_permute_rows", "pm_debug_engine_only", "pm_merge_peers", "pm_ipc_handle", "pm_ipc_open",
    "pm_ipc_close", "pm_debug_flow", "pm_kernel_ms_detail", "pm_reorder", "pm_peer_splits", "pm_debug_host_plan",
)

_lib = None
_lock = threading.RLock()
_ctx: dict[int, ctypes.c_void_p] = {}


class MergeEngineError(RuntimeError):
    """The device reported a failure (CUDA error, wait bound, space exhaustion)."""


def lib() -> ctypes.CDLL:
    """Load the C-ABI library (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "the package has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.pm_version.restype = i32
        L.pm_last_error.restype = ctypes.c_char_p
        L.pm_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.pm_ctx_destroy.argtypes = [vp]
        L.pm_merge.argtypes = [vp, vp, i32, vp, i64, i64, i64, i64, i64, vp]
        L.pm_shift.argtypes = [vp, vp, i32, vp, i64, i64, i64, i64, vp]
        L.pm_find_median.argtypes = [vp, vp, vp, i32, i64, i64, vp, vp]
        L.pm_find_splits.argtypes = [vp, vp, vp, i32, i64, i64, vp, i64, vp, vp]
        L.pm_plan_intervals.argtypes = [vp, vp, i32, i64, i64, i64, ctypes.c_int32, vp, vp]
        L.pm_status.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.pm_merge_host.argtypes = [vp, vp, i32, vp, i64, i64, i64, i64, vp]
        L.pm_debug_host_plan.argtypes = [vp, i32, i64, i64, i64, i64, ctypes.c_int32, vp, vp, vp, vp,
                                         ctypes.c_int32, vp]
        L.pm_set_timing.argtypes = [vp, i32]
        L.pm_debug_order.argtypes = [i64, i64, i64, vp]
        L.pm_debug_splits.argtypes = [vp, vp, i64]
        L.pm_debug_stats.argtypes = [vp, vp]
        L.pm_launch_count.argtypes = [vp]
        L.pm_debug_engine_only.argtypes = [vp, i32]
        L.pm_debug_flow.argtypes = [vp, i32]
        L.pm_kernel_ms_detail.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
        L.pm_peer_splits.argtypes = [vp, vp, i32, i64, i64, i32, ctypes.POINTER(ctypes.c_int64), i32,
                                     ctypes.POINTER(ctypes.c_int64), vp]
        L.pm_reorder.argtypes = [vp, vp, i32, vp, i64, i64, i64, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, vp]
        L.pm_merge_peers.argtypes = [vp, vp, vp, i32, i32, i64, i64, i32, i64, vp, vp, vp]
        L.pm_ipc_handle.argtypes = [vp, vp]
        L.pm_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
        L.pm_ipc_close.argtypes = [vp]
        L.pm_debug_permute_rows.argtypes = [vp, vp, i64, vp, i64, ctypes.c_int32, vp]
        L.pm_merge_copy.argtypes = [vp, vp, vp, vp, vp, i32, i64, i64, i64, vp]
        L.pm_kernel_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
        for name in EXPORTED:
            if name not in ("pm_version", "pm_last_error"):
                getattr(L, name).restype = i32
        _lib = L
        return L


def check(rc: int, what: str) -> None:
    if rc == PM_OK:
        return
    msg = lib().pm_last_error().decode(errors="replace")
    if rc == PM_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise MergeEngineError(f"{what} failed (code {rc}): {msg}")


def context(device: int) -> ctypes.c_void_p:
    """Per-device context (persistent workspace); created on first use."""
    c = _ctx.get(device)
    if c is None:
        with _lock:
            c = _ctx.get(device)
            if c is None:
                c = ctypes.c_void_p()
                L = lib()
                rc = L.pm_ctx_create(device, ctypes.byref(c))
                if rc != PM_OK:
                    raise MergeEngineError(f"pm_ctx_create: {L.pm_last_error().decode()}")
                _ctx[device] = c
    return c


def status(device: int, stream: int) -> tuple[int, int, int, int]:
    """Synchronise the stream and raise if the device reported an error."""
    stats = (ctypes.c_uint64 * 16)()
    check(lib().pm_status(context(device), ctypes.c_void_p(stream), stats), "merge engine")
    return tuple(int(x) for x in stats)
