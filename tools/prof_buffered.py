import sys, torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
L = int(sys.argv[1])
k0, p0, m = config_input_device(2, seed=5, log_len=L)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for i in range(2):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0), scratch_records=len(k0) // 2)
assert bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item())
print("ok")
