"""CPU oracle for the parallel in-place merge path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes front-end over ``liboracle.so`` (``parmerge_oracle.c``), the plain-C
restatement of the reference's numba kernels (``/root/reference/pkg/src/
parmerge/_kernels.py``) and its pivot search (``median.py:23-60``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline -- the
product package (``paper_2005_12648_b200``) never touches it.

Arrays are numpy: ``keys`` int32 or int64 1-D C-contiguous, ``payload`` uint8
``(n, w)`` C-contiguous (``w`` may be 0), mirroring ``KeyedArray``
(``records.py:15-44``).  Pinned against the reference in ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so in place (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "parmerge_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        for suf in ("i32", "i64"):
            getattr(L, f"orc_find_median_{suf}").argtypes = [_vp, _i64, _vp, _i64, _vp]
            for name in ("linear_shift", "circular_shift"):
                getattr(L, f"orc_{name}_{suf}").argtypes = [_vp, _vp, _i64, _i64, _i64, _i64]
            getattr(L, f"orc_rotation_merge_{suf}").argtypes = [
                _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int]
            getattr(L, f"orc_seq_merge_buffered_{suf}").argtypes = [
                _vp, _vp, _i64, _i64, _i64, _i64]
            getattr(L, f"orc_seq_merge_buffered_{suf}").restype = ctypes.c_int
            getattr(L, f"orc_merge_path_{suf}").argtypes = [_vp, _i64, _vp, _i64, _i64]
            getattr(L, f"orc_merge_path_{suf}").restype = _i64
        L.orc_srecpar_buffered.argtypes = [
            _vp, ctypes.c_int, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _i64]
        L.orc_srecpar_buffered.restype = ctypes.c_int
        L.orc_srecpar.argtypes = [_vp, ctypes.c_int, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _i64, ctypes.c_int]
        L.orc_srecpar.restype = ctypes.c_int
        _lib = L
    return _lib


def _suf(keys: np.ndarray) -> str:
    if keys.dtype == np.int32:
        return "i32"
    if keys.dtype == np.int64:
        return "i64"
    raise TypeError(f"oracle keys must be int32 or int64, got {keys.dtype}")


def _check(keys, payload):
    assert keys.ndim == 1 and keys.flags.c_contiguous
    if payload is None:
        payload = np.empty((keys.shape[0], 0), np.uint8)
    assert payload.dtype == np.uint8 and payload.ndim == 2 and payload.flags.c_contiguous
    assert payload.shape[0] == keys.shape[0]
    return payload


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


def find_median(a: np.ndarray, b: np.ndarray) -> tuple[int, int]:
    """Alg. 1 pivot pair, median.py:23-60."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    out = np.zeros(2, np.int64)
    getattr(lib(), f"orc_find_median_{_suf(a)}")(_ptr(a), len(a), _ptr(b), len(b), _ptr(out))
    return int(out[0]), int(out[1])


def linear_shift(keys, payload, lo, len_a, len_b) -> None:
    """In place, _kernels.py:92-150."""
    payload = _check(keys, payload)
    getattr(lib(), f"orc_linear_shift_{_suf(keys)}")(
        _ptr(keys), _ptr(payload), payload.shape[1], lo, len_a, len_b)


def circular_shift(keys, payload, lo, len_a, len_b) -> None:
    """In place, _kernels.py:154-197."""
    payload = _check(keys, payload)
    getattr(lib(), f"orc_circular_shift_{_suf(keys)}")(
        _ptr(keys), _ptr(payload), payload.shape[1], lo, len_a, len_b)


def rotation_merge(keys, payload, start, middle, end, circular=False) -> None:
    """In place, _kernels.py:201-223."""
    payload = _check(keys, payload)
    getattr(lib(), f"orc_rotation_merge_{_suf(keys)}")(
        _ptr(keys), _ptr(payload), payload.shape[1], start, middle, end, int(circular))


def seq_merge_buffered(keys, payload, start, middle, end) -> None:
    """In place, seqmerge.py:55-75 -> _kernels.py:227-313 (the stable parity oracle)."""
    payload = _check(keys, payload)
    rc = getattr(lib(), f"orc_seq_merge_buffered_{_suf(keys)}")(
        _ptr(keys), _ptr(payload), payload.shape[1], start, middle, end)
    if rc != 0:
        raise MemoryError("oracle scratch allocation failed")


def merge_path(a: np.ndarray, b: np.ndarray, d: int) -> int:
    """A-count among the first d outputs of the stable (A-first) merge."""
    return int(getattr(lib(), f"orc_merge_path_{_suf(a)}")(_ptr(a), len(a), _ptr(b), len(b), d))


def srecpar_buffered(keys, payload, start, middle, end, threads, size_limit=512) -> None:
    """merge_srecpar(..., leaf_core=seq_merge_buffered) on host threads (srecpar.py:33-84)."""
    payload = _check(keys, payload)
    rc = lib().orc_srecpar_buffered(
        _ptr(keys), keys.dtype.itemsize, _ptr(payload), payload.shape[1],
        start, middle, end, threads, size_limit)
    if rc != 0:
        raise ValueError(f"worker count must be a power of two >= 1, got {threads}")


def srecpar(keys, payload, start, middle, end, threads, size_limit=512, leaf="buffered") -> None:
    """merge_srecpar(arr, job, threads) with the default rotation leaves (leaf="rotation",
    srecpar.py:57) or seq_merge_buffered leaves (leaf="buffered"), on host threads."""
    payload = _check(keys, payload)
    rc = lib().orc_srecpar(_ptr(keys), keys.dtype.itemsize, _ptr(payload), payload.shape[1],
                           start, middle, end, threads, size_limit, {"buffered": 0, "rotation": 1}[leaf])
    if rc != 0:
        raise ValueError(f"worker count must be a power of two >= 1, got {threads}")


def stable_merge_numpy(keys: np.ndarray, payload, start, middle, end):
    """Independent restatement: stable argsort of the job range."""
    payload = _check(keys, payload)
    k = keys.copy()
    p = payload.copy()
    order = np.argsort(keys[start:end], kind="stable")
    k[start:end] = keys[start:end][order]
    p[start:end] = payload[start:end][order]
    return k, p


def rotate_oracle(keys, payload, len_a):
    """B then A by plain copying, shift.py:134-140."""
    payload = _check(keys, payload)
    return (np.concatenate([keys[len_a:], keys[:len_a]]),
            np.concatenate([payload[len_a:], payload[:len_a]]))


def plan_intervals(keys: np.ndarray, start, middle, end, threads):
    """soptmov.py:93-123: all t-1 Alg.-1 pivots, level by level, no moves.

    Returns (leaf_sources, final_positions) as lists of tuples.
    """
    levels = [[(start, middle, middle, end)]]
    for _ in range(threads.bit_length() - 1):
        nxt = []
        for a0, a1, b0, b1 in levels[-1]:
            pa, pb = find_median(keys[a0:a1], keys[b0:b1])
            nxt.append((a0, a0 + pa, b0, b0 + pb))
            nxt.append((a0 + pa, a1, b0 + pb, b1))
        levels.append(nxt)
    sources, finals, dst = [], [], start
    for a0, a1, b0, b1 in levels[-1]:
        sources.append((a0, a1 - a0))
        sources.append((b0, b1 - b0))
        finals.append((dst, dst + (a1 - a0), dst + (a1 - a0) + (b1 - b0)))
        dst += (a1 - a0) + (b1 - b0)
    return sources, finals
