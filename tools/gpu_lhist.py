"""Tuning: log2 histograms of the data team's waits (PM_LIB=libparmerge_b200_stats.so)."""
import ctypes, sys
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for rep in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0))
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = list(out)
print("cycles>=    gather_issue   items_wait   consumer_wait")
for b in range(16):
    print(f"2^{b+8:<3d} {st[16+b]:14d} {st[32+b]:12d} {st[48+b]:14d}")
