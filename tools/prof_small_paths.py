"""Drivers for ncu captures of the round-2 kernels outside the scheduled engine:
the grid merge (k_merge_grid, 2^20 int32 records per side) and the equal-block
swap of a pure rotation (k_swap_blocks, 2^29 + 2^29 int32)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm  # noqa: E402
from paper_2005_12648_b200 import _ops  # noqa: E402
from paper_2005_12648_b200.workloads import config_input_device  # noqa: E402

k0, p0, m = config_input_device(2, seed=3, log_len=20)
arr = pm.KeyedArray(k0.clone(), p0.clone())
for _ in range(3):
    arr.keys.copy_(k0)
    _ops.merge(arr, 0, m, k0.numel())
h = 1 << 29
k1 = torch.cat([torch.arange(h, device="cuda", dtype=torch.int32) + h, torch.arange(h, device="cuda", dtype=torch.int32)])
arr = pm.KeyedArray(k1.clone())
for _ in range(2):
    arr.keys.copy_(k1)
    _ops.merge(arr, 0, h, 2 * h)
torch.cuda.synchronize()
print("ok", bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item()))
