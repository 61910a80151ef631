"""In-place engine time and salvage vs the salvage-pool size (scratch_records) at 2^L per side.

usage: python tools/gpu_pool_sweep.py [L]
"""
import sys

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi, _ops
from paper_2005_12648_b200.workloads import config_input_device

L = int(sys.argv[1]) if len(sys.argv) > 1 else 29
k0, p0, m = config_input_device(2, seed=3, log_len=L)
n = k0.numel()
arr = pm.KeyedArray(k0.clone(), p0.clone())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for div in (0, 64, 32, 16, 8, 4, 3):
    scratch = 0 if div == 0 else n // div
    ts, sal = [], 0
    for r in range(6):
        arr.keys.copy_(k0)
        e0.record()
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, n, scratch_records=scratch)
        e1.record()
        st = pm.synchronize()
        ts.append(e0.elapsed_time(e1))
        sal = st[1]
    ok = bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item())
    ts = sorted(ts[1:])
    t = ts[len(ts) // 2]
    print(f"pool=N/{div if div else 'default'} ({scratch * 4 / 2**20:.0f} MB) {t:.3f} ms  salvage {sal / n:.3f} N  "
          f"frac {8 * n / t / 1e6 / 6451.8:.3f} ok={ok}", flush=True)
