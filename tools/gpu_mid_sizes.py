import sys, torch
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
for L in (20, 22):
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    for i in range(3):
        arr.keys.copy_(k0)
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, k0.numel())
    torch.cuda.synchronize()
