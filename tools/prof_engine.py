"""Profiling driver: a few merges of BASELINE config 2 (or 3/4) at 2^L per side."""
import sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
kw = {"log_len_b": 16} if cfg == 3 else {}
k0, p0, m = config_input_device(cfg, seed=5, log_len=L, **kw)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for i in range(reps):
    arr.keys.copy_(k0)
    if p0.shape[1]:
        arr.payload.copy_(p0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0))
st = pm.synchronize()
assert bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item())
print("ok", st[:4])
