"""Small/medium in-place merges (config 2, 2^L per side) timed like bench.py's size sweep:
CUDA events around one direct C-ABI pm_merge call (no Python wrapper in between)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm  # noqa: F401
from paper_2005_12648_b200 import _capi
from paper_2005_12648_b200.workloads import config_input_device

L_ = _capi.lib()
ctx = _capi.context(0)
st = torch.cuda.current_stream()
for L in (10, 12, 14, 15, 16, 17, 18, 19, 20):
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    a = k0.clone()
    n = a.numel()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(8):
        a.copy_(k0)
        e0.record(st)
        rc = L_.pm_merge(ctx, ctypes.c_void_p(a.data_ptr()), 4, ctypes.c_void_p(0), 0, 0, m, n, 0,
                         ctypes.c_void_p(st.cuda_stream))
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    _capi.status(0, st.cuda_stream)
    print(L, round(sorted(ts[1:])[3] * 1e3, 1), "us", bool(torch.equal(a, k0.sort().values)), flush=True)
