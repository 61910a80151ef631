"""Per-phase times of the cooperative plan kernel (build with -DPM_FLOW_DEBUG=1).

usage: PM_LIB=libparmerge_b200_<v>.so python tools/gpu_plan_phases.py [L] [cfg]
"""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi, _ops
from paper_2005_12648_b200.workloads import config_input_device

L = int(sys.argv[1]) if len(sys.argv) > 1 else 29
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k0, p0, m = config_input_device(cfg, seed=3, log_len=L)
n = k0.numel()
arr = pm.KeyedArray(k0.clone(), p0.clone())
names = ["sample", "split", "readers", "angle", "sync*", "key", "choose", "decide", "rank", "hull", "alloc", "tickets"]
for r in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n)
    st = (ctypes.c_uint64 * 64)()
    _capi.lib().pm_debug_stats(_capi.context(0), st)
    t = [st[32 + k] for k in range(16)]
    print(" ".join(f"{names[k] if k < len(names) else k}:{(t[k + 1] - t[k]) / 1000:.1f}" for k in range(15) if t[k + 1] and t[k]),
          f"total {(max(t) - t[0]) / 1000:.1f} us")
