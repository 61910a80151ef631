"""Host-side cost of one pm_merge call (the C-ABI enqueue: workspace checks,
occupancy queries, launches of the plan, salvage copy, merge and the gated
fallback kernels) and how much of it the GPU sees as idle time at the start of
a step, per library variant.

usage: python tools/gpu_host_overhead.py cfg L v1 v2 ...
"""
import os
import subprocess
import sys

CODE = r'''
import ctypes, sys, time, statistics, torch
sys.path.insert(0, '.')
from paper_2005_12648_b200 import _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg, L = int(sys.argv[1]), int(sys.argv[2])
k0, p0, m = config_input_device(cfg, seed=3, log_len=L)
n = k0.numel(); ks = k0.element_size(); w = p0.shape[1]
keys = k0.clone(); pay = p0.clone()
lib = _capi.lib(); ctx = _capi.context(0)
st = torch.cuda.current_stream()
def call():
    rc = lib.pm_merge(ctx, ctypes.c_void_p(keys.data_ptr()), ks, ctypes.c_void_p(pay.data_ptr() if w else 0), w, 0, m, n, 0,
                      ctypes.c_void_p(st.cuda_stream))
    _capi.check(rc, "pm_merge")
busy = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); busy2 = torch.empty_like(busy)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for pre in (False, True):
    ts, hs = [], []
    for i in range(12):
        keys.copy_(k0); pay.copy_(p0); torch.cuda.synchronize()
        if pre:  # keep the GPU busy while the host enqueues the merge
            for _ in range(4): busy2.copy_(busy)
        e0.record(st)
        t0 = time.perf_counter(); call(); hs.append((time.perf_counter() - t0) * 1e6)
        e1.record(st); e1.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    res[pre] = (statistics.median(ts), statistics.median(hs[2:]))
print(f"step {res[False][0]*1e3:.1f} us (GPU idle at start)  {res[True][0]*1e3:.1f} us (GPU busy while enqueuing)  "
      f"host enqueue {res[False][1]:.1f} us / {res[True][1]:.1f} us")
'''
for v in sys.argv[3:]:
    env = dict(os.environ, PM_LIB="libparmerge_b200.so" if v in ("", "main") else f"libparmerge_b200_{v}.so")
    out = subprocess.run([sys.executable, "-c", CODE, sys.argv[1], sys.argv[2]], env=env, capture_output=True, text=True)
    print(f"{v:>8s}: {out.stdout.strip() or out.stderr.strip()[-400:]}", flush=True)
