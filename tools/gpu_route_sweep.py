"""In-place merge time per route and size: library routing vs the scheduled engine forced
vs the bounded-pool engine forced (config 2 shapes, 2^L per side).

usage: python tools/gpu_route_sweep.py [L ...]
"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device

Ls = [int(x) for x in sys.argv[1:]] or [18, 20, 21, 22, 23, 24, 25, 26]
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for L in Ls:
    k0, p0, m = config_input_device(2, seed=5, log_len=L)
    n = k0.numel()
    ref = torch.sort(k0).values
    row = []
    for route in ("auto", "flow", "bounded"):
        _ops.set_engine_only(route != "auto")
        _ops.set_flow_mode("bounded" if route == "bounded" else "auto")
        a = pm.KeyedArray(k0.clone(), p0.clone())
        ts = []
        for r in range(8):
            a.keys.copy_(k0)
            ev0.record()
            with pm.deferred_checks():
                _ops.merge(a, 0, m, n)
                ev1.record()
            ts.append(ev0.elapsed_time(ev1))
        assert torch.equal(a.keys, ref)
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        row.append(f"{route} {t * 1e3:8.1f} us ({8 * n / t / 1e6 / 6451.8:.2f})")
    _ops.set_engine_only(False)
    _ops.set_flow_mode("auto")
    print(f"2^{L}/side: " + " | ".join(row), flush=True)
