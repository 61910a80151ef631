"""CPU-only checks of the C-ABI boundary: the library loads, exports every
symbol include/parmerge_b200.h declares, and its host-evaluable pieces behave."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_2005_12648_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "parmerge_b200.h")).read()
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(pm_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    declared = header_symbols()
    assert len(declared) >= 12
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_capi.EXPORTED)


def test_version_and_last_error():
    lib = _capi.lib()
    assert lib.pm_version() == 100
    out = np.zeros(4, np.int64)
    assert lib.pm_debug_order(0, 0, 0, out.ctypes.data) == _capi.PM_ERR_ARG
    assert b"bad order" in lib.pm_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_context_without_gpu_fails_loudly():
    lib = _capi.lib()
    c = ctypes.c_void_p()
    rc = lib.pm_ctx_create(0, ctypes.byref(c))
    assert rc == _capi.PM_ERR_CUDA
    with pytest.raises(_capi.MergeEngineError):
        _capi.context(0)


def test_argument_validation_needs_no_gpu():
    lib = _capi.lib()
    assert lib.pm_merge(None, None, 4, None, 0, 0, 0, 0, 0, None) == _capi.PM_ERR_ARG
    assert lib.pm_plan_intervals(None, None, 4, 0, 0, 0, 3, None, None) == _capi.PM_ERR_ARG


@pytest.mark.parametrize("Q,qc", [(1, 0), (2, 0), (2, 1), (7, 3), (10, 0), (10, 9), (33, 5), (64, 50), (1000, 500)])
def test_two_front_order_is_a_bijection_with_contiguous_windows(Q, qc):
    """The device ticket order (TwoFront, pm_engine.cuh) evaluated by the library on the host."""
    lib = _capi.lib()
    out = np.zeros(4, np.int64)
    seen = set()
    for t in range(Q):
        assert lib.pm_debug_order(Q, qc, t, out.ctypes.data) == 0
        region, order, lo, hi = (int(x) for x in out)
        assert 0 <= region < Q and region not in seen
        seen.add(region)
        assert order == t
        assert lo <= region <= hi and hi - lo == t  # window = the t+1 regions with order <= t
        assert lo >= 0 and hi < Q
    assert seen == set(range(Q))


def _host_plan(keys, start, middle, end, min_chunk, chunks):
    lib = _capi.lib()
    span = np.zeros(2, np.int64)
    cap = chunks + 64  # (steady chunks plus the geometric ramps at both ends)
    d = np.zeros(cap + 1, np.int64)
    a = np.zeros(cap + 1, np.int64)
    fr = np.zeros(cap, np.int32)
    nch = ctypes.c_int32()
    rc = lib.pm_debug_host_plan(keys.ctypes.data, keys.itemsize, start, middle, end, min_chunk, chunks,
                                span.ctypes.data, d.ctypes.data, a.ctypes.data, fr.ctypes.data, cap, ctypes.byref(nch))
    assert rc == 0, lib.pm_last_error()
    n = nch.value
    return span, d[:n + 1], a[:n + 1], fr[:n]


@pytest.mark.parametrize("layout", ["uniform", "rotation", "inside", "dups", "sorted", "tiny_b", "skew"])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_host_plan_of_merge_host(layout, dtype):
    """pm_merge_host's host side (no GPU): the identity trim, the chunks' stable
    merge-path splits, and free_at[k] -- the first upload (merge order) after which
    chunk k's output range holds no record still to be uploaded -- checked from
    first principles against numpy on the same keys."""
    rng = np.random.default_rng(hash((layout, dtype().itemsize)) % 2**32)
    n = 50_000
    la = {"tiny_b": n - 3, "skew": n // 9}.get(layout, n // 2)
    lb = n - la
    if layout == "uniform":
        a, b = np.sort(rng.integers(0, 10**6, la)), np.sort(rng.integers(0, 10**6, lb))
    elif layout == "rotation":
        a, b = np.sort(rng.integers(500, 1000, la)), np.sort(rng.integers(0, 500, lb))
    elif layout == "inside":
        a, b = np.sort(rng.integers(0, 10**6, la)), np.sort(rng.integers(400_000, 400_500, lb))
    elif layout == "dups":
        a, b = np.sort(rng.integers(0, 7, la)), np.sort(rng.integers(0, 7, lb))
    elif layout == "sorted":
        a, b = np.arange(la), np.arange(la, n)
    else:
        a, b = np.sort(rng.integers(0, 10**6, la)), np.sort(rng.integers(0, 10**6, lb))
    lo, hi = 11, 5
    keys = np.concatenate([np.full(lo, -1), a, b, np.full(hi, 2 * 10**6)]).astype(dtype)
    start, middle, end = lo, lo + la, lo + n
    span, d, asp, free = _host_plan(keys, start, middle, end, 1000, 16)
    A, B = keys[start:middle], keys[middle:end]
    if A[-1] <= B[0]:
        assert span[0] == -1 and len(free) == 0
        return
    # identity trim: A prefix <= B[0] and B suffix >= A[last] (stable ties) stay put
    assert span[0] == start + np.searchsorted(A, B[0], side="right")
    assert span[1] == middle + np.searchsorted(B, A[-1], side="left")
    s0, e0 = int(span[0]), int(span[1])
    X = keys[s0:e0]
    tla, tlb, tn = middle - s0, e0 - middle, e0 - s0
    assert d[0] == 0 and d[-1] == tn and np.all(np.diff(d) > 0)
    # splits: the stable merge path (A wins ties) of the trimmed job at every boundary
    order = np.argsort(np.concatenate([X[:tla], X[tla:]]), kind="stable")
    from_a = order < tla
    for k, dk in enumerate(d):
        assert asp[k] == from_a[:dk].sum(), (layout, k)
    # free_at: minimal upload j >= k covering chunk k's output range
    bsp = d - asp
    for k in range(len(free)):
        need_a = min(d[k + 1], tla) if d[k] < tla else 0
        need_b = max(d[k + 1] - tla, 0)
        covered = [j for j in range(k, len(free)) if asp[j + 1] >= need_a and bsp[j + 1] >= need_b]
        assert covered and free[k] == covered[0], (layout, k, free[k], covered[:1])
