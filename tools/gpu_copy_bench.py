"""Tuning: pm_merge_copy throughput (the streaming 1-read/1-write merge) at 2^L per side."""
import sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
dk, dp = torch.empty_like(k0), torch.empty_like(p0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(8):
    e0.record()
    _ops.merge_copy(k0, p0, dk, dp, m)
    e1.record()
    pm.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
n = k0.numel()
ms = ts[len(ts) // 2]
byt = 2 * n * (k0.element_size() + p0.shape[1])
print(f"cfg{cfg} L={L} merge_copy med {ms:.3f} ms  {n / ms / 1e6:.1f} G rec/s  {byt / ms / 1e6:.0f} GB/s "
      f"({byt / ms / 1e6 / 6537 * 100:.1f}% of 6537)")
assert bool(torch.all(dk[1:] >= dk[:-1]).item())
