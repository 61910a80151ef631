"""Pure rotations (every B key below every A key) at 2^L records: pm_merge (the
scheduled engine's gated block-exchange route when the salvage overflows) and
pm_shift (the block exchange itself), keys only and with a 4-byte payload;
device-timed, median of 5."""
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm  # noqa: E402
from paper_2005_12648_b200 import _ops  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << L
peak = 6451.8
for la in (n // 2, n // 3, 2 * n // 5, 3 * n // 10, 7 * n // 10):
    lb = n - la
    for w in (0, 4):
        k0 = torch.cat([torch.arange(lb, device="cuda", dtype=torch.int32) + lb, torch.arange(la, device="cuda", dtype=torch.int32)])
        k0 = torch.cat([k0[lb:lb + la] + n, k0[:0]]) if False else torch.cat([torch.arange(la, device="cuda", dtype=torch.int32) + lb,
                                                                          torch.arange(lb, device="cuda", dtype=torch.int32)])
        p0 = torch.arange(n, device="cuda", dtype=torch.int32).view(torch.uint8).view(n, 4)[:, :w].contiguous()
        arr = pm.KeyedArray(k0.clone(), p0.clone())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for what in ("merge", "shift"):
            ts = []
            for i in range(6):
                arr.keys.copy_(k0)
                arr.payload.copy_(p0)
                torch.cuda.synchronize()
                e0.record()
                if what == "merge":
                    with pm.deferred_checks():
                        _ops.merge(arr, 0, la, n)
                else:
                    _ops.shift(arr, 0, la, lb)
                e1.record()
                e1.synchronize()
                if i:
                    ts.append(e0.elapsed_time(e1))
            ok = bool(torch.equal(arr.keys, torch.sort(k0).values))
            t = statistics.median(ts)
            rec = 4 + w
            print(f"{what:5s} la={la} lb={lb} w={w}: {t:.3f} ms  {2 * n * rec / t / 1e6 / peak:.2f} of 1R+1W roofline  ok={ok}",
                  flush=True)
