"""Wide payload rows: in-place pm_merge and pm_merge_copy over ~2 GB of records per width.

usage: python tools/gpu_wide_bench.py [total_MB [w1,w2,...]]   (PM_LIB selects a tuning build)
Prints, per row width, the median time and the fraction of the 1R+1W roofline.
"""
import json
import os
import sys

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6537.0
total = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 2 << 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.Generator(device="cuda").manual_seed(7)
widths = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else (60, 124, 252, 508, 1020, 2044, 16380, 65536)
for w in widths:
    n = total // (4 + w)
    m = n // 2
    k0 = torch.randint(0, 2**31 - 1, (n,), device="cuda", generator=g, dtype=torch.int32)
    k0[:m] = k0[:m].sort().values
    k0[m:] = k0[m:].sort().values
    p0 = torch.randint(0, 256, (n, w), device="cuda", generator=g, dtype=torch.uint8)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    dk, dp = torch.empty_like(k0), torch.empty_like(p0)

    def med(f, reset, reps=5):
        ts = []
        for _ in range(reps + 1):
            reset()
            e0.record()
            f()
            e1.record()
            pm.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts = sorted(ts[1:])
        return ts[len(ts) // 2]

    def reset():
        arr.keys.copy_(k0)
        arr.payload.copy_(p0)

    def inplace():
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, n)

    ti = med(inplace, reset)
    order = torch.sort(k0, stable=True).indices
    ok = bool(torch.equal(arr.keys, k0[order])) and bool(torch.equal(arr.payload, p0[order]))
    tc = med(lambda: _ops.merge_copy(k0, p0, dk, dp, m), lambda: None)
    okc = bool(torch.equal(dk, k0[order])) and bool(torch.equal(dp, p0[order]))
    by = 2 * n * (4 + w)
    print(json.dumps({"w": w, "n": n, "inplace_ms": round(ti, 3), "inplace_frac": round(by / ti / 1e6 / peak, 3),
                      "copy_ms": round(tc, 3), "copy_frac": round(by / tc / 1e6 / peak, 3), "ok": ok and okc}),
          flush=True)
    del arr, dk, dp, k0, p0, order
    torch.cuda.empty_cache()
