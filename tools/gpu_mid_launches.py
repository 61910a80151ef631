"""One in-place and one copy-mode merge at 2^L per side (config 2), for an ncu launch list."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k0, p0, m = config_input_device(2, seed=5, log_len=L)
n = k0.numel()
a = pm.KeyedArray(k0.clone(), p0.clone())
dk = torch.empty_like(k0)
for r in range(3):
    a.keys.copy_(k0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"inplace {r}")
    with pm.deferred_checks():
        _ops.merge(a, 0, m, n)
    pm.synchronize()
    torch.cuda.nvtx.range_pop()
    _ops.merge_copy(k0, p0, dk, torch.empty_like(p0), m)
    pm.synchronize()
print("ok", torch.equal(a.keys, dk))
