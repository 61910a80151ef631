"""One scheduled-engine merge at 2^L per side (after warm-up) for ncu captures.

usage: python tools/prof_flow.py [L] [mode] [reps]
"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device

L = int(sys.argv[1]) if len(sys.argv) > 1 else 29
mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
_ops.set_flow_mode(mode)
import os
k0, p0, m = config_input_device(int(os.environ.get("CFG", "2")), seed=3, log_len=L)
n = k0.numel()
arr = pm.KeyedArray(k0.clone(), p0.clone())
for r in range(reps):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n)
print("sorted:", bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item()))
