"""Tuning: buffered-mode pm_merge (scratch = min run) and pm_merge_copy at 2^L per side."""
import sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); L = int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=1, log_len=L)
n = k0.numel()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def med(f, reps=7):
    ts = []
    for r in range(reps):
        f(0)
        e0.record(); f(1); e1.record(); pm.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts) // 2]
dk, dp = torch.empty_like(k0), torch.empty_like(p0)
arr = pm.KeyedArray(k0.clone(), p0.clone())
def copy(timed):
    if timed: _ops.merge_copy(k0, p0, dk, dp, m)
def buf(timed):
    if not timed:
        arr.keys.copy_(k0); return
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n, scratch_records=min(m, n - m))
tc, tb = med(copy), med(buf)
assert bool(torch.all(dk[1:] >= dk[:-1]).item()) and bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item())
w = k0.element_size() + p0.shape[1]
print(f"L={L} copy {tc:.3f} ms ({2*n*w/tc/1e6/6537*100:.1f}% HBM)  buffered {tb:.3f} ms ({2*n*w/tb/1e6/6537*100:.1f}% algorithmic)")
