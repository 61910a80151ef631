"""Compare library variants (PM_LIB=libparmerge_b200_<v>.so builds) on one in-place merge.

usage: python tools/gpu_variants.py L v1 v2 ...   ('' or 'main' = the default library)
Each variant runs in a fresh subprocess; prints plan/engine ms (CUDA events), salvage and correctness.
env: CFG (workload config, default 2), MODE (flow mode, default auto)
"""
import os
import subprocess
import sys

L = sys.argv[1]
CODE = r'''
import ctypes, sys, torch
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi, _ops
from paper_2005_12648_b200.workloads import config_input_device
L = int(sys.argv[1]); cfg = int(sys.argv[2]); mode = sys.argv[3]
_ops.set_flow_mode(mode)
k0, p0, m = config_input_device(cfg, seed=3, log_len=L)
n = k0.numel()
ref = torch.sort(k0, stable=True).values
arr = pm.KeyedArray(k0.clone(), p0.clone())
lib = _capi.lib(); ctx = _capi.context(0); lib.pm_set_timing(ctx, 1)
ts = []
for r in range(7):
    arr.keys.copy_(k0)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n)
    st = pm.synchronize()
    a, b = ctypes.c_float(), ctypes.c_float()
    lib.pm_kernel_ms(ctx, ctypes.byref(a), ctypes.byref(b))
    ts.append((a.value + b.value, a.value, b.value))
ts = sorted(ts[1:])
t, pl, en = ts[len(ts) // 2]
rb = k0.element_size() + p0.shape[1]
print(f"ok={torch.equal(arr.keys, ref)} plan {pl:.3f} engine {en:.3f} total {t:.3f} ms frac {2 * rb * n / t / 1e6 / 6451.8:.3f} "
      f"sal {st[1] / n:.3f}N mode {st[4]} est_angle {st[5] / n:.3f} est_tf {st[6] / n:.3f}")
'''
cfg = os.environ.get("CFG", "2")
mode = os.environ.get("MODE", "auto")
for v in sys.argv[2:]:
    env = dict(os.environ)
    env["PM_LIB"] = "libparmerge_b200.so" if v in ("", "main") else f"libparmerge_b200_{v}.so"
    out = subprocess.run([sys.executable, "-c", CODE, L, cfg, mode], env=env, capture_output=True, text=True)
    print(f"{v or 'main':>10s}: {out.stdout.strip() or out.stderr.strip()[-400:]}", flush=True)
