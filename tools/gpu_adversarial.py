"""Engine stress on adversarial layouts at large sizes: the scheduled engine (order chosen per job)
and the bounded-pool engine, in place, device-timed (median of 3 after a warm-up).

Each case: merge, compare with a stable device sort, print time.  Cases: B entirely
before A (one big rotation), perfect interleave, tiny B inside A, tiny A, heavy
duplicates, all equal keys, already sorted.
"""
import sys
import time

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops

L = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = 1 << L
h = n // 2
g = torch.Generator(device="cuda").manual_seed(11)
ar = torch.arange(h, device="cuda", dtype=torch.int32)
cases = {
    "rotation (B < A)": (torch.cat([ar + h, ar]), h),
    "perfect interleave": (torch.cat([2 * ar, 2 * ar + 1]), h),
    "tiny B inside A": (torch.cat([torch.arange(n - 7, device="cuda", dtype=torch.int32) * 2,
                                   torch.tensor([5, 1001, 2_000_001, 5_000_001, 7_000_001, 9_000_001, 2**30],
                                                device="cuda", dtype=torch.int32)]), n - 7),
    "tiny A": (torch.cat([torch.tensor([3, 10**6, 10**8], device="cuda", dtype=torch.int32),
                          torch.arange(n - 3, device="cuda", dtype=torch.int32)]), 3),
    "duplicates (4 values)": (torch.cat([torch.randint(0, 4, (h,), generator=g, device="cuda", dtype=torch.int32).sort().values,
                                         torch.randint(0, 4, (h,), generator=g, device="cuda", dtype=torch.int32).sort().values]), h),
    "all equal": (torch.zeros(n, device="cuda", dtype=torch.int32), h),
    "already sorted": (torch.arange(n, device="cuda", dtype=torch.int32), h),
    "uneven 1/16": (torch.cat([torch.randint(0, 2**31 - 1, (n // 16,), generator=g, device="cuda", dtype=torch.int32).sort().values,
                               torch.randint(0, 2**31 - 1, (n - n // 16,), generator=g, device="cuda", dtype=torch.int32).sort().values]), n // 16),
}
ok_all = True
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, (k0, m) in cases.items():
    idx = torch.arange(k0.numel(), device="cuda", dtype=torch.int32)
    pay0 = idx.view(torch.uint8).view(-1, 4)
    ref = torch.sort(k0.to(torch.int64), stable=True)
    for mode in ("auto", "bounded"):
        arr = pm.KeyedArray(k0.clone(), pay0.clone())
        _ops.set_engine_only(True)
        _ops.set_flow_mode(mode)
        ts, err, st = [], "", None
        try:
            for r in range(4):
                arr.keys.copy_(k0)
                arr.payload.copy_(pay0)
                ev0.record()
                with pm.deferred_checks():
                    _ops.merge(arr, 0, m, k0.numel())
                    ev1.record()
                ts.append(ev0.elapsed_time(ev1))
            st = pm.synchronize()
        except Exception as ex:  # noqa: BLE001
            err = str(ex)[:120]
        _ops.set_engine_only(False)
        _ops.set_flow_mode("auto")
        ok = not err and torch.equal(arr.keys.to(torch.int64), ref.values) and torch.equal(
            arr.payload.contiguous().view(torch.int32).view(-1).to(torch.int64), ref.indices)
        ok_all &= bool(ok)
        order = {1: "two-front", 2: "angle"}.get(st[4], "bounded") if st else "?"
        t = sorted(ts[1:])[len(ts[1:]) // 2] if len(ts) > 1 else float("nan")
        print(f"{name:24s} n=2^{L} {mode:8s} {t:8.3f} ms  order={order:9s} salvage={st[1] / k0.numel() if st else 0:.3f}N "
              f"ok={ok} {err}", flush=True)
print("ALL OK" if ok_all else "FAILURES")
