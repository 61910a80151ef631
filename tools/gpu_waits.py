"""Tuning: split of the data team's wait stage (PM_LIB=libparmerge_b200_stats.so)."""
import ctypes, sys
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
k0, p0, m = config_input_device(int(sys.argv[1]), seed=1, log_len=int(sys.argv[2]))
arr = pm.KeyedArray(k0.clone(), p0.clone())
for rep in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0))
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = list(out); nr = max(st[2] + st[3], 1)
print(f"free_path={st[24]/nr:.0f} open_ahead={st[25]/nr:.0f} items_wait={st[26]/nr:.0f} consumer_wait={st[27]/nr:.0f} (cycles/region)")
