"""Small jobs through every in-place kernel, for compute-sanitizer (tools/sanitize.sh).

Each case is checked against torch's stable sort; sizes are kept small because the
sanitizers slow kernels down by orders of magnitude."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops

g = torch.Generator(device="cuda").manual_seed(1)


def job(n, payload=0, dom=2**31 - 1):
    h = n // 2
    a = torch.randint(0, dom, (h,), generator=g, device="cuda", dtype=torch.int32).sort().values
    b = torch.randint(0, dom, (n - h,), generator=g, device="cuda", dtype=torch.int32).sort().values
    k = torch.cat([a, b])
    idx = torch.arange(n, device="cuda", dtype=torch.int32)
    return k, idx.view(torch.uint8).view(-1, 4) if payload else torch.empty((n, 0), dtype=torch.uint8, device="cuda"), h


def run(tag, n, engine_only, mode, payload=0, dom=2**31 - 1, scratch=0):
    k0, p0, h = job(n, payload, dom)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    _ops.set_engine_only(engine_only)
    _ops.set_flow_mode(mode)
    try:
        _ops.merge(arr, 0, h, n, scratch_records=scratch)
    finally:
        _ops.set_engine_only(False)
        _ops.set_flow_mode("auto")
    ref = torch.sort(k0.to(torch.int64), stable=True)
    ok = torch.equal(arr.keys.to(torch.int64), ref.values)
    if payload:
        ok = ok and torch.equal(arr.payload.contiguous().view(torch.int32).view(-1).to(torch.int64), ref.indices)
    print(f"{tag}: n={n} ok={ok}", flush=True)
    assert ok


sizes = [int(x) for x in sys.argv[1:]] or [1 << 16, 1 << 18]
for n in sizes:
    run("k_flow (angle/auto)", n, True, "auto", payload=4)
    run("k_flow (two-front)", n, True, "two_front")
    run("k_flow fallback -> k_engine", n, True, "fallback", payload=4, dom=50)
    run("k_engine (bounded pool)", n, True, "bounded", payload=4)
    run("k_buffered in place (min-side budget)", n, True, "bounded", payload=4, scratch=n // 2)
run("k_merge_small", 4000, False, "auto", payload=4)
run("k_merge_cluster", 1 << 16, False, "auto", payload=4)
run("staged copy mode", 1 << 20, False, "auto")
# block exchange: one-pass slide and the reversals
for la, lb in ((1000, 1 << 17), (1 << 16, 1 << 16 - 3)):
    k = torch.randint(0, 1000, (la + lb,), generator=g, device="cuda", dtype=torch.int32)
    arr = pm.KeyedArray(k.clone())
    pm.linear_shift(arr, la, lb)
    assert torch.equal(arr.keys, torch.cat([k[la:], k[:la]]))
    _ops.set_engine_only(True)
    arr = pm.KeyedArray(k.clone())
    pm.linear_shift(arr, la, lb)
    _ops.set_engine_only(False)
    assert torch.equal(arr.keys, torch.cat([k[la:], k[:la]]))
    print(f"shift {la},{lb} ok", flush=True)
# wide rows: in-place cycle walk
from paper_2005_12648_b200 import _capi  # noqa: E402
n = 3000
k0 = torch.randint(0, 100, (n,), generator=g, device="cuda", dtype=torch.int32)
k0[:1500] = k0[:1500].sort().values
k0[1500:] = k0[1500:].sort().values
rows = torch.randint(0, 256, (n, 300), generator=g, device="cuda", dtype=torch.uint8)
arr = pm.KeyedArray(k0.clone(), rows.clone())
_ops.merge(arr, 0, 1500, n)
ref = torch.sort(k0.to(torch.int64), stable=True)
assert torch.equal(arr.keys.to(torch.int64), ref.values) and torch.equal(arr.payload, rows[ref.indices])
print("wide rows ok", flush=True)
print("SANITIZE_CASES_DONE", flush=True)
