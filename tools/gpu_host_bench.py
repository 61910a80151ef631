"""pm_merge_host (host buffers, H2D + merge + D2H pipelined) at 2^L per side: median seconds and G rec/s."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm  # noqa: F401
from paper_2005_12648_b200 import _capi
from paper_2005_12648_b200.workloads import config_input_device

L = int(sys.argv[1]) if len(sys.argv) > 1 else 29
k0, p0, m = config_input_device(2, seed=1, log_len=L)
n = k0.numel()
h0 = k0.cpu().pin_memory()
h = torch.empty_like(h0).pin_memory()
lib, ctx = _capi.lib(), _capi.context(0)
ts = []
for r in range(4):
    h.copy_(h0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.pm_merge_host(ctx, ctypes.c_void_p(h.data_ptr()), 4, ctypes.c_void_p(0), 0, 0, m, n, None)
    _capi.check(rc, "pm_merge_host")
    ts.append(time.perf_counter() - t0)
ok = bool(torch.all(h[1:] >= h[:-1]).item())
t = sorted(ts[1:])[1]
print(f"L={L} host merge {t * 1e3:.1f} ms = {n / t / 1e9:.2f} G rec/s ok={ok}")
