"""Tuning: engine time with ablation builds (PM_LIB=...); outputs are not checked."""
import sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
arr = pm.KeyedArray(k0.clone(), p0.clone())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(7):
    arr.keys.copy_(k0)
    torch.cuda.synchronize()
    e0.record()
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, len(k0))
    e1.record()
    pm.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"L={L} med {ts[3]:.3f} ms min {ts[0]:.3f}")
