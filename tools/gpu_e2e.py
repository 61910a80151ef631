"""pm_merge_host (pinned host buffers, H2D + merge + D2H) at 2^L per side, per library variant.

usage: python tools/gpu_e2e.py L v1 v2 ...
"""
import os
import subprocess
import sys

CODE = r'''
import ctypes, sys, time, torch
sys.path.insert(0, '.')
from paper_2005_12648_b200 import _capi
from paper_2005_12648_b200.workloads import config_input_device
L = int(sys.argv[1])
k0, p0, m = config_input_device(2, seed=3, log_len=L)
n = k0.numel()
hk0 = k0.cpu().pin_memory(); hk = torch.empty_like(hk0).pin_memory()
lib = _capi.lib(); ctx = _capi.context(0)
ts = []
for i in range(9):
    hk.copy_(hk0); torch.cuda.synchronize()
    t0 = time.perf_counter()
    _capi.check(lib.pm_merge_host(ctx, ctypes.c_void_p(hk.data_ptr()), 4, None, 0, 0, m, n, None), "pm_merge_host")
    ts.append(time.perf_counter() - t0)
ok = bool(torch.all(hk[1:] >= hk[:-1]).item())
s = sorted(ts[1:])
t = s[len(s) // 2]
print(f"ok={ok} median {t*1e3:.1f} ms (min {s[0]*1e3:.1f}, max {s[-1]*1e3:.1f}, mean {sum(s)/len(s)*1e3:.1f})  "
      f"{n / t / 1e9:.2f} G rec/s  PCIe {2 * 4 * n / t / 1e9:.1f} GB/s both ways")
'''
for v in sys.argv[2:]:
    env = dict(os.environ, PM_LIB="libparmerge_b200.so" if v in ("", "main") else f"libparmerge_b200_{v}.so")
    out = subprocess.run([sys.executable, "-c", CODE, sys.argv[1]], env=env, capture_output=True, text=True)
    print(f"{v:>8s}: {out.stdout.strip() or out.stderr.strip()[-300:]}", flush=True)
