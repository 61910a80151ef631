"""Timeline of pm_merge_host (library built with -DPM_HOST_TRACE=1: `make variant
VNAME=trace VFLAGS=-DPM_HOST_TRACE=1`): per chunk upload / merge / D2H end and
the staged chunks' move into place; plus this host's memcpy rate with 1-8 threads.

usage: PM_LIB=libparmerge_b200_trace.so python tools/gpu_e2e_trace.py L
"""
import ctypes
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2005_12648_b200 import _capi  # noqa: E402
from paper_2005_12648_b200.workloads import config_input_device  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 29
src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory().numpy()
dst = torch.empty(1 << 30, dtype=torch.uint8).pin_memory().numpy()
for nt in (1, 2, 4, 8):
    per = len(src) // nt

    def work(t):
        np.copyto(dst[t * per:(t + 1) * per], src[t * per:(t + 1) * per])

    ts = []
    for _ in range(3):
        th = [threading.Thread(target=work, args=(t,)) for t in range(nt)]
        t0 = time.perf_counter()
        [x.start() for x in th]
        [x.join() for x in th]
        ts.append(time.perf_counter() - t0)
    print(f"host memcpy {nt} threads: {len(src) / min(ts) / 1e9:.1f} GB/s", flush=True)
del src, dst
k0, p0, m = config_input_device(2, seed=3, log_len=L)
n = k0.numel()
hk0 = k0.cpu().pin_memory()
hk = torch.empty_like(hk0).pin_memory()
lib = _capi.lib()
ctx = _capi.context(0)
for i in range(3):
    hk.copy_(hk0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _capi.check(lib.pm_merge_host(ctx, ctypes.c_void_p(hk.data_ptr()), 4, None, 0, 0, m, n, None), "pm_merge_host")
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms", file=sys.stderr, flush=True)
print("sorted:", bool(torch.all(hk[1:] >= hk[:-1]).item()))
