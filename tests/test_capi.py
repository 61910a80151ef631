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
