"""Tuning: salvage destination paths (needs PM_LIB=libparmerge_b200_stats.so)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2]); div = int(sys.argv[3]) if len(sys.argv) > 3 else 0
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for rep in range(3):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0), scratch_records=len(k0) // div if div else 0)
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = list(out)
print(f"moves={st[0]} cache_scratch={st[16]} cache_free={st[17]} global_scratch={st[18]} global_free={st[19]} "
      f"blocked={st[20]} blocked_cycles/blocked={st[21]/max(st[20],1):.0f}")
