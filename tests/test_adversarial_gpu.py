"""Adversarial layouts at 2^23 records through every in-place engine route (the
scheduled engine with each order and its fallback, the bounded-pool engine, the
library's routing): one big rotation, perfect interleave, tiny runs, heavy
duplicates, all-equal and already-sorted inputs, a 1/16 split.  Payload = original
index, so stability is checked exactly (== stable argsort)."""
import pytest
import torch

pm = pytest.importorskip("paper_2005_12648_b200")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

L = 23


def _cases():
    n, h = 1 << L, 1 << (L - 1)
    g = torch.Generator(device="cuda").manual_seed(11)
    ar = torch.arange(h, device="cuda", dtype=torch.int32)
    rnd = lambda k, hi: torch.randint(0, hi, (k,), generator=g, device="cuda", dtype=torch.int32).sort().values  # noqa: E731
    t = lambda xs: torch.tensor(xs, device="cuda", dtype=torch.int32)  # noqa: E731
    return {
        "rotation": (torch.cat([ar + h, ar]), h),
        "interleave": (torch.cat([2 * ar, 2 * ar + 1]), h),
        "tiny_b": (torch.cat([torch.arange(n - 5, device="cuda", dtype=torch.int32) * 2, t([5, 1001, 2_000_001, 5_000_001, 2**30])]), n - 5),
        "tiny_a": (torch.cat([t([3, 10**6, 10**8]), torch.arange(n - 3, device="cuda", dtype=torch.int32)]), 3),
        "dups4": (torch.cat([rnd(h, 4), rnd(h, 4)]), h),
        "equal": (torch.zeros(n, device="cuda", dtype=torch.int32), h),
        "sorted": (torch.arange(n, device="cuda", dtype=torch.int32), h),
        "uneven": (torch.cat([rnd(n // 16, 2**31 - 1), rnd(n - n // 16, 2**31 - 1)]), n // 16),
    }


@pytest.mark.parametrize("route", ["auto", "flow", "two_front", "angle", "fallback", "bounded"])
@pytest.mark.parametrize("case", ["rotation", "interleave", "tiny_b", "tiny_a", "dups4", "equal", "sorted", "uneven"])
def test_adversarial_layouts(case, route):
    """route: the library's routing; the scheduled engine with its order chosen per job,
    or forced (two-front / angle), or its device-side fallback forced; the bounded-pool
    engine."""
    from paper_2005_12648_b200 import _ops

    k0, m = _cases()[case]
    idx = torch.arange(k0.numel(), device="cuda", dtype=torch.int32)
    arr = pm.KeyedArray(k0.clone(), idx.view(torch.uint8).view(-1, 4).clone())
    _ops.set_engine_only(route != "auto")
    _ops.set_flow_mode("auto" if route in ("auto", "flow") else route)
    try:
        _ops.merge(arr, 0, m, k0.numel())
    finally:
        _ops.set_engine_only(False)
        _ops.set_flow_mode("auto")
    ref = torch.sort(k0.to(torch.int64), stable=True)
    assert torch.equal(arr.keys.to(torch.int64), ref.values)
    assert torch.equal(arr.payload.contiguous().view(torch.int32).view(-1).to(torch.int64), ref.indices)
