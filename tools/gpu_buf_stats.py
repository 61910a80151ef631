"""Tuning: per-region phase cycles of the buffered in-place pipeline
(PM_LIB=libparmerge_b200_bufstats.so, built with -DPM_USE_BUFFERED=1 -DPM_STATS=1)."""
import ctypes, sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
n = k0.numel()
arr = pm.KeyedArray(k0.clone(), p0.clone())
for r in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n, scratch_records=min(m, n - m))
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = list(out)
nr = max(st[2], 1)
names = ["issue", "land", "merge(tid0)", "sync1->store", "store->end", "merge->sync1"]
print(" ".join(f"{n}={st[4 + i] / nr:.0f}" for i, n in enumerate(names)), "regions", st[2])
