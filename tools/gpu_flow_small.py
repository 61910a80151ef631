"""Scheduled engine at mid sizes: plan / salvage copy / merge split (pm_kernel_ms_detail)
and, with a -DPM_FLOW_DEBUG=1 build (PM_LIB), the plan's per-phase times.

usage: [PM_LIB=libparmerge_b200_dbg.so] python tools/gpu_flow_small.py [L ...]
"""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi, _ops
from paper_2005_12648_b200.workloads import config_input_device

Ls = [int(x) for x in sys.argv[1:]] or [22, 24, 26]
lib, ctx = _capi.lib(), _capi.context(0)
names = ["sample", "split", "readers", "angle", "sync*", "key", "choose", "decide", "rank", "hull", "alloc", "tickets"]
for L in Ls:
    k0, p0, m = config_input_device(2, seed=5, log_len=L)
    n = k0.numel()
    _ops.set_engine_only(True)
    lib.pm_set_timing(ctx, 1)
    a = pm.KeyedArray(k0.clone(), p0.clone())
    rows = []
    for r in range(8):
        a.keys.copy_(k0)
        with pm.deferred_checks():
            _ops.merge(a, 0, m, n)
        pm.synchronize()
        out = (ctypes.c_float * 4)()
        lib.pm_kernel_ms_detail(ctx, out)
        rows.append(tuple(out))
    rows = sorted(rows[2:], key=lambda x: x[3])
    pl, sv, mg, tot = rows[len(rows) // 2]
    st = (ctypes.c_uint64 * 64)()
    lib.pm_debug_stats(ctx, st)
    t = [st[32 + k] for k in range(16)]
    ph = " ".join(f"{names[k] if k < len(names) else k}:{(t[k + 1] - t[k]) / 1000:.1f}" for k in range(15)
                  if t[k + 1] and t[k])
    lib.pm_set_timing(ctx, 0)
    _ops.set_engine_only(False)
    print(f"2^{L}/side Q={n // 8192}: plan {pl * 1e3:.1f} save {sv * 1e3:.1f} merge {mg * 1e3:.1f} total {tot * 1e3:.1f} us"
          f" (k_flow {8 * n / mg / 1e6 / 6451.8:.2f}, all {8 * n / tot / 1e6 / 6451.8:.2f}) | {ph}", flush=True)
