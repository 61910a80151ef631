"""Tuning: per-ticket-range waits of the engine (needs PM_LIB=libparmerge_b200_stats.so)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
kw = {"log_len_b": 16} if cfg == 3 else {}
k0, p0, m = config_input_device(cfg, seed=1, log_len=L, **kw)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for rep in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0))
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = np.array(out[:], dtype=np.float64)
nreg = st[2] + st[3]
per = nreg / 16
print("bucket  cons_wait  items_wait  pre_work   (cycles per region)")
for b in range(16):
    print(f"{b:5d} {st[16+b]/per:10.0f} {st[32+b]/per:11.0f} {st[48+b]/per:10.0f}")
