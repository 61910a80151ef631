"""Time pm_shift's one-pass slide (stash + k_slide + stash) at 2^30 records and check it
against torch's concatenation.  usage: python tools/gpu_slide.py [lib ...]  (PM_LIB variants,
'main' = the default library); each variant runs in a fresh subprocess."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
n = 1 << 30
g = torch.Generator(device="cuda"); g.manual_seed(1)
k0 = torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, w, la in (("keys small-left 1%", 0, n // 100), ("keys small-right 1%", 0, n - n // 100 - 3),
                    ("keys small-left D%16=0", 0, 4 << 20), ("kv4 small-left 1%", 4, (n // 2) // 100)):
    nn = n if w == 0 else n // 2
    keys = k0[:nn].clone()
    pay = torch.empty((nn, w), dtype=torch.uint8, device="cuda")
    if w:
        pay.view(torch.int32).view(-1).copy_(k0[nn:2 * nn])
    want = torch.cat([keys[la:], keys[:la]])
    arr = pm.KeyedArray(keys, pay)
    ts = []
    for r in range(6):
        arr.keys.copy_(k0[:nn])
        if w:
            arr.payload.view(torch.int32).view(-1).copy_(k0[nn:2 * nn])
        torch.cuda.synchronize()
        e0.record()
        _ops.shift(arr, 0, la, nn - la)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    pm.synchronize()
    ok = torch.equal(arr.keys, want)
    if w:
        wp = torch.cat([k0[nn:2 * nn][la:], k0[nn:2 * nn][:la]])
        ok = ok and torch.equal(arr.payload.view(torch.int32).view(-1), wp)
    t = sorted(ts[1:])[len(ts[1:]) // 2]
    rb = 4 + w
    print(f"{name:26s} ok={ok} {t:.3f} ms  {2 * nn * rb / t / 1e6:.0f} GB/s frac {2 * nn * rb / t / 1e6 / 6451.8:.3f}")
'''
for v in sys.argv[1:] or ["main"]:
    env = dict(os.environ)
    if v != "main":
        env["PM_LIB"] = f"libparmerge_b200_{v}.so"
    print(f"== {v}", flush=True)
    subprocess.run([sys.executable, "-c", CODE], env=env, check=False)
