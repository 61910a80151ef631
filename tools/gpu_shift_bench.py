"""Tuning: pm_shift (block exchange A|B -> B|A) throughput at n records."""
import sys
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
L = int(sys.argv[1]); frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
n = 1 << L
k0 = torch.arange(n, dtype=torch.int32, device="cuda")
la = int(n * frac)
arr = pm.KeyedArray(k0.clone(), torch.empty((n, 0), dtype=torch.uint8, device="cuda"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(5):
    arr.keys.copy_(k0)
    torch.cuda.synchronize()
    e0.record()
    with pm.deferred_checks():
        _ops.shift(arr, 0, la, n - la)
    e1.record()
    pm.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
want = torch.cat([k0[la:], k0[:la]])
assert torch.equal(arr.keys, want)
print(f"shift n=2^{L} la={la}: med {ts[2]:.3f} ms = {2*n*4/ts[2]/1e6:.0f} GB/s algorithmic ({2*n*4/ts[2]/1e6/6537*100:.1f}%)")
