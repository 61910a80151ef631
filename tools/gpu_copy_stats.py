"""Tuning: per-region phase cycles of the streaming pipeline (PM_LIB=libparmerge_b200_stats.so)."""
import ctypes, sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
dk, dp = torch.empty_like(k0), torch.empty_like(p0)
for r in range(3):
    _ops.merge_copy(k0, p0, dk, dp, m)
    pm.synchronize()
out = (ctypes.c_uint64 * 64)()
_capi.lib().pm_debug_stats(_capi.context(0), out)
st = list(out)
nr = max(st[2], 1)
names = ["issue", "land", "merge(tid0)", "sync1->store", "store->end", "merge->sync1"]
print(" ".join(f"{n}={st[4 + i] / nr:.0f}" for i, n in enumerate(names)), "regions", st[2])
