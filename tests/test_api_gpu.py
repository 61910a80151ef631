"""C-ABI behaviour around the kernels: calls on several streams sharing one context,
the caller's current device left alone, span checks of the block exchange."""
import numpy as np
import pytest
import torch

pm = pytest.importorskip("paper_2005_12648_b200")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2005_12648_b200 import _ops  # noqa: E402


def _job(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = n // 2
    k = torch.cat([torch.randint(0, 2**31 - 1, (h,), generator=g, device="cuda", dtype=torch.int32).sort().values,
                   torch.randint(0, 2**31 - 1, (n - h,), generator=g, device="cuda", dtype=torch.int32).sort().values])
    return k, h


@pytest.mark.parametrize("mode", ["auto", "bounded"])
def test_streams_share_one_context(mode):
    """Merges issued back to back on two streams use the same per-device workspace;
    the library orders them (an event on the previous stream), so none corrupts another."""
    _ops.set_engine_only(True)
    _ops.set_flow_mode(mode)
    try:
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        jobs = [_job(1 << 21, s) for s in range(6)]
        arrs = [pm.KeyedArray(k.clone()) for k, _ in jobs]
        torch.cuda.synchronize()
        with pm.deferred_checks():
            for i, (a, (k, h)) in enumerate(zip(arrs, jobs)):
                with torch.cuda.stream(streams[i % 2]):
                    _ops.merge(a, 0, h, k.numel())
            torch.cuda.synchronize()
        for a, (k, h) in zip(arrs, jobs):
            assert torch.equal(a.keys, torch.sort(k).values)
    finally:
        _ops.set_engine_only(False)
        _ops.set_flow_mode("auto")


def test_current_device_untouched():
    before = torch.cuda.current_device()
    k, h = _job(1 << 18, 3)
    a = pm.KeyedArray(k.clone())
    _ops.merge(a, 0, h, k.numel())
    assert torch.cuda.current_device() == before


def test_shift_span_checked():
    a = pm.KeyedArray(torch.arange(10, dtype=torch.int32, device="cuda"))
    with pytest.raises(IndexError):
        pm.shift_region(a, 6, 3, 3, "linear")
    with pytest.raises(IndexError):
        pm.shift_region(a, -1, 2, 2, "linear")
    pm.shift_region(a, 4, 3, 3, "linear")
    assert a.keys.cpu().tolist() == [0, 1, 2, 3, 7, 8, 9, 4, 5, 6]


def test_merge_host_from_many_threads():
    """pm_merge_host called concurrently from host threads on one context (the
    reference's worker pool does this for its leaf merges): each call is exact."""
    import concurrent.futures as cf

    from oracle import oracle as orc
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(8)
    jobs = []
    for i in range(24):
        n = int(rng.integers(1000, 300000))
        h = int(rng.integers(1, n))
        k = np.concatenate([np.sort(rng.integers(0, 1000, h)), np.sort(rng.integers(0, 1000, n - h))]).astype(np.int32)
        p = rng.integers(0, 256, (n, 4), dtype=np.uint8)
        wk, wp = k.copy(), p.copy()
        orc.seq_merge_buffered(wk, wp, 0, h, n)
        jobs.append((k, p, h, wk, wp))
    with cf.ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda j: _ops.merge_host(j[0], j[1], 0, j[2], len(j[0])), jobs))
    for k, p, h, wk, wp in jobs:
        assert np.array_equal(k, wk) and np.array_equal(p, wp)


@pytest.mark.parametrize("n", [1 << 20, 1 << 24])
def test_staged_path_skips_ordered_runs(n):
    """A medium job whose runs are already in order (A[m-1] <= B[0]) leaves the array
    untouched and costs no merge pass (gated on the device); an out-of-order job of
    the same shape still merges."""
    from paper_2005_12648_b200 import _ops

    k = torch.arange(n, dtype=torch.int32, device="cuda")
    p = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint8).view(-1, 4)
    a = pm.KeyedArray(k.clone(), p.clone())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    _ops.merge(a, 0, n // 2, n)
    ev1.record()
    torch.cuda.synchronize()
    assert torch.equal(a.keys, k) and torch.equal(a.payload, p)
    kk = torch.cat([k[n // 2:], k[:n // 2]])
    b = pm.KeyedArray(kk.clone(), p.clone())
    _ops.merge(b, 0, n // 2, n)
    assert torch.equal(b.keys, k)
