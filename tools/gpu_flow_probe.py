"""Scheduled engine probe: correctness (vs a stable device sort) and timing per order mode.

usage: python tools/gpu_flow_probe.py [L ...]   (log2 records per side; default 16 20 24 29)
"""
import sys

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi, _ops
from paper_2005_12648_b200.workloads import config_input_device

Ls = [int(x) for x in sys.argv[1:]] or [16, 20, 24, 29]
_ops.set_engine_only(True)
lib = _capi.lib()
ctx = _capi.context(0)
lib.pm_set_timing(ctx, 1)
import ctypes
for L in Ls:
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    n = k0.numel()
    ref = torch.sort(k0, stable=True).values
    for mode in ("bounded", "auto", "two_front", "angle", "fallback"):
        _ops.set_flow_mode(mode)
        arr = pm.KeyedArray(k0.clone(), p0.clone())
        ts = []
        st = None
        for r in range(5 if L >= 24 else 3):
            arr.keys.copy_(k0)
            torch.cuda.synchronize()
            with pm.deferred_checks():
                _ops.merge(arr, 0, m, n)
            st = pm.synchronize()
            a, b = ctypes.c_float(), ctypes.c_float()
            lib.pm_kernel_ms(ctx, ctypes.byref(a), ctypes.byref(b))
            ts.append((a.value, b.value))
        ok = bool(torch.equal(arr.keys, ref))
        ts = sorted(ts[1:], key=lambda x: x[0] + x[1])
        pl, en = ts[len(ts) // 2]
        stats = _capi.status(0, torch.cuda.current_stream().cuda_stream)
        print(f"L={L} {mode:10s} ok={ok} plan {pl:.3f} ms engine {en:.3f} ms total {pl+en:.3f} "
              f"frac {8 * n / (pl + en) / 1e6 / 6451.8:.3f} stats {list(stats[:7])} sal {stats[1]/n:.3f}N", flush=True)
