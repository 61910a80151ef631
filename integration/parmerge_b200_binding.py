"""The ctypes binding a maintainer adds to the REFERENCE package.

Pure C-ABI: ctypes + numpy, no torch.  ``install(parmerge)`` routes the reference's
default merge paths -- merge_srecpar, merge_soptmov, seq_merge_buffered,
seq_merge_rotation -- through ``pm_merge_host`` (H2D, the device merge, D2H) on the
caller's numpy arrays, keeping the reference's own validation (check_threads,
check_job, leaf_core / pool contracts): a call that passes a custom ``leaf_core`` or
``pool`` (the reference tests record those) still runs the reference's Python
driver, exactly as a maintainer would leave hooks untouched.

The merge is the STABLE merge at every worker count (the reference's t > 1
strategies may reorder equal keys' payloads); keys are identical.
"""

from __future__ import annotations

import ctypes
import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(_HERE), "paper_2005_12648_b200", "libparmerge_b200.so")

_lib = None
_ctx = ctypes.c_void_p()
calls = {"pm_merge_host": 0}  # routed calls (the drop-in test asserts they happened)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB)
        L.pm_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        L.pm_merge_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_void_p]
        L.pm_last_error.restype = ctypes.c_char_p
        if L.pm_ctx_create(0, ctypes.byref(_ctx)) != 0:
            raise RuntimeError(L.pm_last_error().decode())
        _lib = L
    return _lib


def merge_host(arr, start: int, middle: int, end: int) -> None:
    """pm_merge_host on a reference KeyedArray (records.py:15-83): int32 keys, uint8 rows."""
    k, p = arr.keys, arr.payload
    if not (k.flags.c_contiguous and p.flags.c_contiguous):
        raise ValueError("pm_merge_host needs C-contiguous keys and payload")
    L = lib()
    rc = L.pm_merge_host(_ctx, k.ctypes.data, k.itemsize, p.ctypes.data if p.shape[1] else None, p.shape[1],
                         start, middle, end, None)
    if rc == 1:
        raise ValueError(L.pm_last_error().decode())
    if rc != 0:
        raise RuntimeError(L.pm_last_error().decode())
    calls["pm_merge_host"] += 1


def install(parmerge) -> None:
    """Route the reference's default merge paths through the B200 library."""
    from parmerge import records, seqmerge, soptmov, srecpar

    o_srecpar, o_soptmov = srecpar.merge_srecpar, soptmov.merge_soptmov
    o_buf, o_rot = seqmerge.seq_merge_buffered, seqmerge.seq_merge_rotation

    @functools.wraps(o_srecpar)
    def merge_srecpar(arr, job, threads, *, shift_kind=srecpar.LINEAR, size_limit=srecpar.DEFAULT_SIZE_LIMIT,
                      leaf_core=None, pool=None):
        if leaf_core is not None or pool is not None:  # hooks the caller observes: the reference driver
            return o_srecpar(arr, job, threads, shift_kind=shift_kind, size_limit=size_limit,
                             leaf_core=leaf_core, pool=pool)
        soptmov.check_threads(threads)
        records.check_job(arr, job)
        srecpar.RecParConfig(threads.bit_length() - 1, size_limit, shift_kind)  # same validation
        merge_host(arr, job.start, job.middle, job.end)

    @functools.wraps(o_soptmov)
    def merge_soptmov(arr, job, threads, *args, **kw):
        if kw.get("leaf_core") is not None or kw.get("pool") is not None or args:
            return o_soptmov(arr, job, threads, *args, **kw)
        soptmov.check_threads(threads)
        records.check_job(arr, job)
        s, m, e = job.start, job.middle, job.end
        if kw.get("strict_marker") and threads > 1 and m not in (s, e) and not (arr.keys[m - 1] <= arr.keys[m]):
            soptmov.derive_marker(arr, s, e)  # raises MarkerOverflow where the reference would
        merge_host(arr, s, m, e)

    @functools.wraps(o_buf)
    def seq_merge_buffered(arr, job, scratch=None):
        records.check_job(arr, job)
        if seqmerge._verify_preconditions:  # set_debug_checks (seqmerge.py:64-65)
            job.check_runs(arr)
        if scratch is not None:  # the caller's scratch contract: it is reserved as before
            scratch.reserve(min(job.len_a, job.len_b), arr.payload.shape[1])
        merge_host(arr, job.start, job.middle, job.end)

    @functools.wraps(o_rot)
    def seq_merge_rotation(arr, job, shift_kind=seqmerge.LINEAR):
        records.check_job(arr, job)
        seqmerge.check_shift_kind(shift_kind)
        if seqmerge._verify_preconditions:
            job.check_runs(arr)
        merge_host(arr, job.start, job.middle, job.end)

    for mod in (parmerge, srecpar):
        mod.merge_srecpar = merge_srecpar
    for mod in (parmerge, soptmov):
        mod.merge_soptmov = merge_soptmov
    for mod in (parmerge, seqmerge, srecpar, soptmov):
        if hasattr(mod, "seq_merge_buffered"):
            mod.seq_merge_buffered = seq_merge_buffered
        if hasattr(mod, "seq_merge_rotation"):
            mod.seq_merge_rotation = seq_merge_rotation
