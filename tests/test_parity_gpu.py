"""GPU parity: the CUDA path (through the C-ABI) against the reference's own outputs.

Bit-exact for every case: keys AND payload bytes (stable order of equal keys).
Golden fixtures come from the reference itself (tests/golden/make_golden.py);
random cases are checked against the pinned CPU oracle (oracle/), which
restates the reference's stable merge (_kernels.py:227-313).
"""
import hashlib

import numpy as np
import pytest
import torch

import golden_io
from gen import config_input, random_instance
from oracle import oracle as orc

pm = pytest.importorskip("paper_2005_12648_b200")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(autouse=True, params=["auto", "flow", "bounded"])
def route(request):
    """Every parity test runs three times: with the library's own routing (one-CTA
    small jobs, staged medium jobs, wide-record path, the scheduled engine for large
    jobs), with every in-place merge forced through the scheduled engine (pm_flow.cu,
    its order chosen per job, device-side fallback), and forced through the
    bounded-pool engine (k_engine)."""
    from paper_2005_12648_b200 import _ops

    _ops.set_engine_only(request.param != "auto")
    _ops.set_flow_mode("bounded" if request.param == "bounded" else "auto")
    yield request.param
    _ops.set_engine_only(False)
    _ops.set_flow_mode("auto")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def to_gpu(keys, payload):
    return pm.KeyedArray(torch.from_numpy(np.ascontiguousarray(keys)).cuda(),
                         torch.from_numpy(np.ascontiguousarray(payload)).cuda())


def assert_same(arr, keys, payload, what=""):
    k, p = arr.numpy()
    assert np.array_equal(k, keys), f"keys differ {what}: first bad index {np.flatnonzero(k != keys)[:5]}"
    assert np.array_equal(p, payload), f"payload differs {what}"


@pytest.mark.parametrize("name", ["merge_i32.npz", "merge_i64.npz"])
@pytest.mark.parametrize("method", ["buffered", "rotation", "srecpar", "soptmov"])
def test_golden_merges(name, method):
    for c in golden_io.merge_cases(name):
        s, m, e = (int(x) for x in c["job"])
        arr = to_gpu(c["keys"], c["payload"])
        job = pm.MergeJob(s, m, e)
        if method == "buffered":
            pm.seq_merge_buffered(arr, job)
        elif method == "rotation":
            pm.seq_merge_rotation(arr, job)
        elif method == "srecpar":
            pm.merge_srecpar(arr, job, 8)
        else:
            pm.merge_soptmov(arr, job, 4)
        assert_same(arr, c["out_keys"], c["out_payload"], f"{name} {method} job={s,m,e}")


def test_golden_reference_parallel_keys():
    # the reference's own t>1 strategies: identical keys (their payload order is unstable)
    for c in golden_io.merge_cases("merge_i32.npz"):
        s, m, e = (int(x) for x in c["job"])
        arr = to_gpu(c["keys"], c["payload"])
        pm.merge_srecpar(arr, pm.MergeJob(s, m, e), 8, size_limit=2)
        assert np.array_equal(arr.keys.cpu().numpy(), c["srecpar_keys"])
        assert np.array_equal(arr.keys.cpu().numpy(), c["soptmov_keys"])


def test_golden_find_median():
    cases = list(golden_io.median_cases())
    for a, b, piv in cases:
        assert tuple(pm.find_median(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())) == piv


def test_golden_shifts():
    for c in golden_io.shift_cases():
        la, lb = (int(x) for x in c["len"])
        for fn in (pm.linear_shift, pm.circular_shift):
            arr = to_gpu(c["keys"], c["payload"])
            fn(arr, la, lb)
            assert_same(arr, c["out_keys"], c["out_payload"], f"shift {la},{lb}")


def test_golden_plans_and_traces():
    for c in golden_io.plan_cases():
        s, m, e, t = (int(x) for x in c["job"])
        arr = to_gpu(c["keys"], c["payload"])
        job = pm.MergeJob(s, m, e)
        plan = pm.plan_intervals(arr, job, t)
        assert np.array_equal(np.array(plan.leaf_sources, np.int64).reshape(-1, 2), c["sources"])
        fin = np.array([(j.start, j.middle, j.end) for j in plan.final_positions], np.int64).reshape(-1, 3)
        assert np.array_equal(fin, c["finals"])
        trace = pm.division_trace(arr, job, t, size_limit=2)
        got = np.array([(r.level, r.split_index, r.pivots[0], r.pivots[1], r.shift_start, r.shift_len_a,
                         r.shift_len_b) for r in trace.records], np.int64).reshape(-1, 7)
        assert np.array_equal(got, c["trace_pivots"])
        assert sha(*trace.divided.numpy()) == str(c["divided_sha"])
        # reorder_multi realises the same layout
        work = arr.copy()
        if t > 1 and len(work) and int(c["keys"].max()) < 2**30:
            pm.reorder_multi(work, plan, pm.derive_marker(work, s, e))
            gathered_k = np.concatenate([c["keys"][a:a + n] for a, n in plan.leaf_sources])
            gathered_p = np.concatenate([c["payload"][a:a + n] for a, n in plan.leaf_sources])
            assert_same(work, gathered_k, gathered_p, "reorder_multi")


@pytest.mark.parametrize("width", [0, 4, 8, 12, 3])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_random_vs_oracle(width, dtype):
    rng = np.random.default_rng(1000 + width + (7 if dtype == np.int64 else 0))
    sizes = [0, 1, 2, 17, 255, 4096, 8191, 8192, 8193, 40000, 150000, 1 << 20]
    for size in sizes:
        for domain in (3, 1000, 2**31 - 1):
            split = float(rng.choice([0.0, 0.05, 0.25, 0.5, 0.75, 0.97, 1.0, rng.random()]))
            keys, payload, middle = random_instance(rng, size, split, domain, width)
            keys = keys.astype(dtype)
            if dtype == np.int64 and domain > 1000:
                keys = keys * np.int64(2**31) + rng.integers(0, 2**31, size)
                keys[:middle].sort()
                keys[middle:].sort()
            lo = int(rng.integers(0, 40))
            hi = int(rng.integers(0, 40))
            kk = np.concatenate([np.full(lo, -5, dtype), keys, np.full(hi, -7, dtype)])
            pp = np.concatenate([np.full((lo, width), 1, np.uint8), payload, np.full((hi, width), 2, np.uint8)])
            want_k, want_p = kk.copy(), pp.copy()
            orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
            arr = to_gpu(kk, pp)
            pm.merge_srecpar(arr, pm.MergeJob(lo, lo + middle, lo + size), 8)
            assert_same(arr, want_k, want_p, f"size={size} dom={domain} split={split} w={width}")


def test_shift_random_sizes():
    rng = np.random.default_rng(77)
    for la, lb in [(1, 1 << 20), (1 << 20, 1), (100000, 33333), (8192, 8192), (5, 7), (123457, 654321)]:
        for width in (0, 4, 9):
            keys = rng.integers(-1000, 1000, la + lb).astype(np.int32)
            payload = rng.integers(0, 256, (la + lb, width), dtype=np.uint8)
            want_k, want_p = orc.rotate_oracle(keys, payload, la)
            arr = to_gpu(keys, payload)
            pm.linear_shift(arr, la, lb)
            assert_same(arr, want_k, want_p, f"shift {la},{lb},w={width}")


def test_config1_matches_reference_checksum():
    g = golden_io.big()
    keys, payload, middle = config_input(1, seed=0)
    assert sha(keys) == g["cfg1_in"]
    arr = to_gpu(keys, payload)
    pm.merge_srecpar(arr, pm.MergeJob(0, middle, len(keys)), 8)
    assert sha(arr.keys.cpu().numpy()) == g["cfg1_out"]


def test_config4_reduced_matches_reference_checksum():
    g = golden_io.big()
    keys, payload, middle = config_input(4, seed=0, log_len=18)
    arr = to_gpu(keys, payload)
    pm.merge_srecpar(arr, pm.MergeJob(0, middle, len(keys)), 8)
    assert sha(*arr.numpy()) == g["cfg4s_out"]


def test_config3_reduced_matches_reference_checksum():
    g = golden_io.big()
    keys, payload, middle = config_input(3, seed=0, log_len=20, log_len_b=12)
    arr = to_gpu(keys, payload)
    pm.merge_srecpar(arr, pm.MergeJob(0, middle, len(keys)), 8)
    assert sha(arr.keys.cpu().numpy()) == g["cfg3s_out"]


def _device_stable_check(arr, keys_in_sorted_ref=None):
    k = arr.keys
    assert bool(torch.all(k[1:] >= k[:-1]).item())


@pytest.mark.parametrize("cfg,log_len", [(2, 24), (4, 24), (3, 26), (2, 29), (4, 26), (3, 28)])
def test_full_size_properties(cfg, log_len):
    """Size-independent properties at large sizes, up to BASELINE.json's full configs
    (config 2: 2^30 int32; config 4: 2^27 key+index records; config 3: 2^28 + 2^16
    int64): equal to a stable device sort, and for config 4 payload == stable argsort."""
    from paper_2005_12648_b200.workloads import config_input_device

    kw = {"log_len_b": 16} if cfg == 3 else {}
    keys, payload, middle = config_input_device(cfg, seed=3, log_len=log_len, **kw)
    ref_sorted = torch.sort(keys.to(torch.int64), stable=True)
    arr = pm.KeyedArray(keys.clone(), payload.clone())
    pm.merge_srecpar(arr, pm.MergeJob(0, middle, len(keys)), 8)
    assert torch.equal(arr.keys.to(torch.int64), ref_sorted.values)
    if cfg == 4:  # payload = original index: stable merge == stable argsort
        idx = arr.payload.contiguous().view(torch.int32).view(-1).to(torch.int64)
        assert torch.equal(idx, ref_sorted.indices)


def test_error_behaviour():
    arr = pm.KeyedArray(torch.tensor([2, 1], dtype=torch.int32).cuda())
    with pytest.raises(ValueError):
        pm.merge_srecpar(arr, pm.MergeJob(0, 1, 2), 3)
    with pytest.raises(IndexError):
        pm.seq_merge_rotation(arr, pm.MergeJob(0, 1, 5))
    with pytest.raises(ValueError):
        pm.linear_shift(arr, 1, 2)
    with pytest.raises(pm.MarkerOverflow):
        big = pm.KeyedArray(np.array([pm.KEY_MIN, 0, pm.KEY_MAX, pm.KEY_MIN + 1, 5], np.int32))
        pm.merge_soptmov(big, pm.MergeJob(0, 3, 5), 2, strict_marker=True)


def test_fast_path_untouched():
    arr = pm.KeyedArray(np.array([1, 2, 3, 3, 4, 9], np.int32), np.arange(24, dtype=np.uint8).reshape(6, 4))
    before = arr.copy()
    pm.merge_soptmov(arr, pm.MergeJob(0, 4, 6), 4)
    assert arr.equals(before)


@pytest.mark.parametrize("width", [0, 4, 5])
def test_buffered_mode_vs_oracle(width):
    """seq_merge_buffered's min-side buffer -> the streaming buffered kernel (both directions)."""
    rng = np.random.default_rng(4242 + width)
    for size in (3, 100, 8193, 50000, 300000, 1 << 20):
        for split in (0.1, 0.5, 0.9):
            for domain in (7, 2**31 - 1):
                keys, payload, middle = random_instance(rng, size, split, domain, width)
                lo = int(rng.integers(0, 9))
                kk = np.concatenate([np.full(lo, -4, np.int32), keys, np.full(5, -6, np.int32)])
                pp = np.concatenate([np.zeros((lo, width), np.uint8), payload, np.ones((5, width), np.uint8)])
                want_k, want_p = kk.copy(), pp.copy()
                orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
                arr = to_gpu(kk, pp)
                pm.seq_merge_buffered(arr, pm.MergeJob(lo, lo + middle, lo + size))
                assert_same(arr, want_k, want_p, f"buffered size={size} split={split} w={width}")


@pytest.mark.parametrize("width", [0, 4])
def test_scratch_sizes_vs_oracle(width):
    """pm_merge's scratch_records argument (pool size) never changes the result."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(9090 + width)
    for size in (50000, 1 << 20, 3 << 20):
        for split in (0.3, 0.5):
            keys, payload, middle = random_instance(rng, size, split, 2**31 - 1, width)
            want_k, want_p = keys.copy(), payload.copy()
            orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
            mn = min(middle, size - middle)
            for scratch in (0, 1000, size // 64, size // 8, size // 4, mn - 1, mn, size):
                arr = to_gpu(keys, payload)
                _ops.merge(arr, 0, middle, size, scratch_records=scratch)
                assert_same(arr, want_k, want_p, f"size={size} split={split} scratch={scratch}")


@pytest.mark.parametrize("width", [0, 4, 8, 3])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_merge_copy_vs_oracle(width, dtype):
    """pm_merge_copy: out-of-place stable merge == the reference's stable merge."""
    import torch

    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(5150 + width)
    for size in (1, 2, 100, 8191, 70000, 1 << 20):
        for split in (0.0, 0.3, 0.5, 1.0):
            for domain in (5, 2**31 - 1):
                keys, payload, middle = random_instance(rng, size, split, domain, width)
                keys = keys.astype(dtype)
                want_k, want_p = keys.copy(), payload.copy()
                orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
                sk = torch.from_numpy(keys).cuda()
                sp = torch.from_numpy(payload).cuda()
                dk = torch.full_like(sk, -1)
                dp = torch.zeros_like(sp)
                _ops.merge_copy(sk, sp, dk, dp, middle)
                pm.synchronize()
                assert np.array_equal(dk.cpu().numpy(), want_k), f"keys size={size} split={split}"
                assert np.array_equal(dp.cpu().numpy(), want_p), f"payload size={size} split={split}"
                assert np.array_equal(sk.cpu().numpy(), keys)  # the source is untouched


def test_merge_copy_errors():
    import torch

    from paper_2005_12648_b200 import _ops

    k = torch.arange(10, dtype=torch.int32, device="cuda")
    p = torch.zeros((10, 0), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        _ops.merge_copy(k, p, k, p, 5)  # overlap
    with pytest.raises(ValueError):
        _ops.merge_copy(k, p, torch.empty(9, dtype=torch.int32, device="cuda"), p[:9], 5)
    with pytest.raises(ValueError):
        _ops.merge_copy(k, p, torch.empty_like(k), p.clone(), 11)


def test_distributed_merge_single_rank_nccl():
    """merge_distributed over a 1-rank NCCL group: splits, exchange and the copy merge."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2005_12648_b200.dist import merge_distributed

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(77)
        keys, payload, middle = random_instance(rng, 300000, 0.4, 1000, 4)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, len(keys))
        k = torch.from_numpy(keys).cuda()
        p = torch.from_numpy(payload).cuda()
        # the split search itself (its rounds run only when a diagonal is interior)
        from paper_2005_12648_b200.dist import global_splits

        diags = [0, 1, 777, 150000, middle, len(keys) - 5, len(keys)]
        got = global_splits(k, diags, middle)
        want = [int(orc.merge_path(keys[:middle], keys[middle:], d)) for d in diags]
        assert got == want
        rk, rp = merge_distributed(k, p, middle)
        assert np.array_equal(rk.cpu().numpy(), want_k) and np.array_equal(rp.cpu().numpy(), want_p)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("width", [0, 4, 5])
def test_merge_host_vs_oracle(width):
    """pm_merge_host: chunk-pipelined H2D / device merge / in-place D2H == the stable merge."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(2024 + width)
    for size, split, domain, dtype in ((1000, 0.5, 100, np.int32), (10_000_000, 0.5, 2**31 - 1, np.int32),
                                       (9_000_001, 0.13, 50, np.int32), (6_000_000, 0.8, 2**31 - 1, np.int64)):
        keys, payload, middle = random_instance(rng, size, split, domain, width)
        keys = keys.astype(dtype)
        lo, hi = 7, 5
        kk = np.concatenate([np.full(lo, -3, dtype), keys, np.full(hi, -9, dtype)])
        pp = np.concatenate([np.full((lo, width), 1, np.uint8), payload, np.full((hi, width), 2, np.uint8)])
        want_k, want_p = kk.copy(), pp.copy()
        orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
        _ops.merge_host(kk, pp, lo, lo + middle, lo + size)
        assert np.array_equal(kk, want_k), f"keys size={size}"
        assert np.array_equal(pp, want_p), f"payload size={size}"


@pytest.mark.parametrize("dtype,width", [(np.int32, 4), (np.int64, 12), (np.int32, 0)])
@pytest.mark.parametrize("layout", ["rotation", "inside", "tiny_a", "tiny_b", "interleave", "halves_swap"])
def test_merge_host_write_back_order(layout, dtype, width):
    """pm_merge_host writes merged chunks back in the order their output ranges
    become free (uploads in merge order): layouts whose ranges free up far from
    chunk order, each over several pipeline chunks, == the stable merge."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(99)
    n = 9 << 20  # several 2M-record chunks
    if layout == "rotation":  # every B key below every A key
        la = 5 << 20
        a = np.sort(rng.integers(1000, 2000, la))
        b = np.sort(rng.integers(0, 1000, n - la))
    elif layout == "inside":  # B inside a narrow window of A
        la = n - (1 << 20)
        a = np.sort(rng.integers(0, 2**31 - 1, la))
        b = np.sort(rng.integers(2**30, 2**30 + 1000, n - la))
    elif layout == "tiny_a":
        la = 3
        a = np.array([5, 2**30, 2**31 - 2])
        b = np.sort(rng.integers(0, 2**31 - 1, n - la))
    elif layout == "tiny_b":
        la = n - 2
        a = np.sort(rng.integers(0, 2**31 - 1, la))
        b = np.array([0, 2**31 - 1])
    elif layout == "interleave":
        la = n // 2
        a = np.arange(la) * 2
        b = np.arange(n - la) * 2 + 1
    else:  # halves swap order, equal keys across the boundary
        la = n // 3
        a = np.sort(rng.integers(500, 1000, la))
        b = np.sort(rng.integers(0, 501, n - la))
    keys = np.concatenate([a, b]).astype(dtype)
    payload = np.random.default_rng(5).integers(0, 256, (n, width), dtype=np.uint8)
    want_k, want_p = keys.copy(), payload.copy()
    orc.seq_merge_buffered(want_k, want_p, 0, la, n)
    _ops.merge_host(keys, payload, 0, la, n)
    assert np.array_equal(keys, want_k), layout
    assert np.array_equal(payload, want_p), layout


@pytest.mark.parametrize("dtype,width", [(np.int32, 0), (np.int32, 4), (np.int64, 12), (np.int32, 5), (np.int64, 64)])
def test_grid_merge_sizes_vs_oracle(dtype, width):
    """The one-launch grid merge's range (32 KB .. ~14 MB of records in shared-memory
    tiles, k_merge_grid) and just beyond it (the staged path): sizes around the
    CTA-count and tile boundaries, odd offsets (every 16-byte phase of the pieces),
    heavy duplicates, skewed splits."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(4242 + width)
    rec = np.dtype(dtype).itemsize + width
    top = (148 * 100 * 1024) // rec
    for size in (300_001, 151_552, 1 << 20, top - 1, top, top + 1, 3 * top + 12_345):  # (beyond top: the staged path)
        for domain, split in ((3, 0.5), (2**31 - 1, 0.3), (1000, 0.97)):
            keys, payload, middle = random_instance(rng, size, split, domain, width)
            keys = keys.astype(dtype)
            lo, hi = int(rng.integers(0, 16)), int(rng.integers(0, 9))
            kk = np.concatenate([np.full(lo, -5, dtype), keys, np.full(hi, 2**31 - 1, dtype)])
            pp = np.concatenate([np.full((lo, width), 1, np.uint8), payload, np.full((hi, width), 2, np.uint8)])
            want_k, want_p = kk.copy(), pp.copy()
            orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
            arr = to_gpu(kk, pp)
            _ops.merge(arr, lo, lo + middle, lo + size)
            assert_same(arr, want_k, want_p, f"size={size} dom={domain} split={split} w={width} lo={lo}")


@pytest.mark.parametrize("size", [100, 5000, 300_000, 1 << 21])
def test_already_ordered_jobs_unchanged(size):
    """A[last] <= B[0] (ties included): nothing moves (srecpar.py:56-57) on every
    route -- keys and payload bytes unchanged."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(size)
    middle = size // 3
    a = np.sort(rng.integers(0, 1000, middle))
    b = np.sort(rng.integers(999, 2000, size - middle))
    b[0] = a[-1]  # a tie across the boundary still needs no move
    keys = np.concatenate([a, b]).astype(np.int32)
    payload = rng.integers(0, 256, (size, 4), dtype=np.uint8)
    arr = to_gpu(keys, payload)
    _ops.merge(arr, 0, middle, size)
    assert_same(arr, keys, payload, f"size={size}")


@pytest.mark.parametrize("dtype,width", [(np.int32, 4), (np.int64, 12), (np.int32, 0)])
def test_large_jobs_vs_oracle(dtype, width):
    """2^22..2^24-record jobs (multi-level salvage, several waves of the grid) vs the oracle,
    through every device path: in place (bounded pool), buffered, copy, host."""
    import torch

    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(31337 + width)
    for size, split, domain in ((1 << 22, 0.5, 2**31 - 1), (3 << 22, 0.3, 1000), (1 << 24, 0.6, 2**31 - 1)):
        keys, payload, middle = random_instance(rng, size, split, domain, width)
        keys = keys.astype(dtype)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
        for mode in ("inplace", "buffered"):
            arr = to_gpu(keys, payload)
            _ops.merge(arr, 0, middle, size, scratch_records=(min(middle, size - middle) if mode == "buffered" else 0))
            assert_same(arr, want_k, want_p, f"{mode} size={size}")
        sk, sp = torch.from_numpy(keys).cuda(), torch.from_numpy(payload).cuda()
        dk, dp = torch.empty_like(sk), torch.empty_like(sp)
        _ops.merge_copy(sk, sp, dk, dp, middle)
        pm.synchronize()
        assert np.array_equal(dk.cpu().numpy(), want_k) and np.array_equal(dp.cpu().numpy(), want_p)
        hk, hp = keys.copy(), payload.copy()
        _ops.merge_host(hk, hp, 0, middle, size)
        assert np.array_equal(hk, want_k) and np.array_equal(hp, want_p)


@pytest.mark.parametrize("width", [16, 32, 64, 100])
def test_wide_payload_rows(width):
    """Wide payload rows shrink the tiles (pick_tiles); every device path stays exact."""
    import torch

    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(777 + width)
    for size, split, domain in ((5000, 0.5, 50), (300_000, 0.35, 2**31 - 1)):
        keys, payload, middle = random_instance(rng, size, split, domain, width)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
        for scratch in (0, min(middle, size - middle)):
            arr = to_gpu(keys, payload)
            _ops.merge(arr, 0, middle, size, scratch_records=scratch)
            assert_same(arr, want_k, want_p, f"w={width} size={size} scratch={scratch}")
        sk, sp = torch.from_numpy(keys).cuda(), torch.from_numpy(payload).cuda()
        dk, dp = torch.empty_like(sk), torch.empty_like(sp)
        _ops.merge_copy(sk, sp, dk, dp, middle)
        pm.synchronize()
        assert np.array_equal(dk.cpu().numpy(), want_k) and np.array_equal(dp.cpu().numpy(), want_p)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_shift_offsets_and_alignment(dtype):
    """pm_shift on sub-ranges at every 16-byte phase, odd and even lengths, both key sizes
    (vectorised block jobs + element-wise edge jobs)."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(4040)
    n = 300_003
    base = rng.integers(-10**6, 10**6, n).astype(dtype)
    pay = np.zeros((n, 0), np.uint8)
    for lo in (0, 1, 2, 3, 5, 17):
        for la, lb in ((70_001, 90_000), (1, 150_000), (150_001, 3), (40_000, 40_000), (2, 2), (0, 10)):
            keys = base.copy()
            want = keys.copy()
            seg = np.concatenate([want[lo + la:lo + la + lb], want[lo:lo + la]])
            want[lo:lo + la + lb] = seg
            arr = to_gpu(keys, pay)
            _ops.shift(arr, lo, la, lb)
            pm.synchronize()
            got, _ = arr.numpy()
            assert np.array_equal(got, want), f"lo={lo} la={la} lb={lb} {dtype.__name__}"


@pytest.mark.parametrize("width", [0, 1, 4, 8, 12])
def test_shift_equal_blocks(width):
    """Equal blocks take the one-pass block swap (pm_shift and the gated rotation
    route): every byte phase of keys and payload rows (16-byte, 4-byte and byte words)."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(808 + width)
    n = 200_011
    for dtype in (np.int32, np.int64):
        base = rng.integers(-10**6, 10**6, n).astype(dtype)
        pbase = rng.integers(0, 256, (n, width), dtype=np.uint8)
        for lo in (0, 1, 3, 4):
            for L in (1, 2, 3, 4, 5, 31, 64, 99_999):
                keys, pay = base.copy(), pbase.copy()
                want_k, want_p = keys.copy(), pay.copy()
                want_k[lo:lo + 2 * L] = np.concatenate([keys[lo + L:lo + 2 * L], keys[lo:lo + L]])
                want_p[lo:lo + 2 * L] = np.concatenate([pay[lo + L:lo + 2 * L], pay[lo:lo + L]])
                arr = to_gpu(keys, pay)
                _ops.shift(arr, lo, L, L)
                pm.synchronize()
                assert_same(arr, want_k, want_p, f"lo={lo} L={L} w={width} {dtype.__name__}")


def _wide_cases(rng, width):
    """Wide-row instances: random, heavy duplicates, exact interleave (many short
    cycles), B entirely before A (one rotation), all-equal keys (identity).
    Sizes shrink with the row width (at most ~150 MB of rows per case)."""
    big = width > 4096
    out = []
    for size, split, domain in ((3000, 0.5, 40), (2000 if big else 20_000, 0.3, 2**31 - 1)):
        out.append(random_instance(rng, size, split, domain, width))
    n = 1024 if big else 4096
    pay = lambda k: rng.integers(0, 256, (k, width), dtype=np.uint8)  # noqa: E731
    ev = np.arange(0, 2 * n, 2, dtype=np.int32)
    out.append((np.concatenate([ev, ev + 1]), pay(2 * n), n))           # perfect shuffle
    out.append((np.concatenate([ev + 10 * n, ev]), pay(2 * n), n))      # rotation
    out.append((np.zeros(2 * n, np.int32), pay(2 * n), n // 3))          # identity
    return out


@pytest.mark.parametrize("width", [252, 301, 508, 1020, 16380, 65536])
def test_wide_records_vs_oracle(width):
    """Rows up to the reference's 65 540-byte elements (bench.py:22): the wide-record
    path (key+index merge, then gather / in-place cycle permutation) is exact."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(9000 + width)
    cases = _wide_cases(rng, width)
    for keys, payload, middle in cases:
        size = len(keys)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
        arr = to_gpu(keys, payload)
        _ops.merge(arr, 0, middle, size)
        assert_same(arr, want_k, want_p, f"in place w={width} size={size} m={middle}")
        sk, sp = torch.from_numpy(keys).cuda(), torch.from_numpy(payload).cuda()
        dk, dp = torch.empty_like(sk), torch.empty_like(sp)
        _ops.merge_copy(sk, sp, dk, dp, middle)
        pm.synchronize()
        assert np.array_equal(dk.cpu().numpy(), want_k) and np.array_equal(dp.cpu().numpy(), want_p)
        if size <= 20_000 and width <= 1020:
            hk, hp = keys.copy(), payload.copy()
            _ops.merge_host(hk, hp, 0, middle, size)
            assert np.array_equal(hk, want_k) and np.array_equal(hp, want_p)


@pytest.mark.parametrize("width", [508, 16380])
def test_wide_records_offset_jobs_public_api(width):
    """Sub-range jobs (start > 0) through merge_srecpar / merge_soptmov with wide rows;
    the rows outside the job are untouched."""
    rng = np.random.default_rng(31 + width)
    n = 6000 if width < 4096 else 1500
    keys, payload, _ = random_instance(rng, n, 0.5, 1000, width)
    s, e = 137, n - 91
    m = (s + e) // 2 + 7
    keys[s:m].sort()
    keys[m:e].sort()
    want_k, want_p = keys.copy(), payload.copy()
    orc.seq_merge_buffered(want_k, want_p, s, m, e)
    for fn in (pm.merge_srecpar, pm.merge_soptmov):
        arr = to_gpu(keys, payload)
        fn(arr, pm.MergeJob(s, m, e), 8)
        assert_same(arr, want_k, want_p, f"{fn.__name__} w={width}")


@pytest.mark.parametrize("cut_every", [1, 16, 1 << 30])
@pytest.mark.parametrize("width", [4, 60, 4096 + 16, 333])
def test_wide_row_permutation_cycles(cut_every, width):
    """The in-place cycle walk on arbitrary permutations: random (long cycles; with no
    cuts they exceed the bounded walk and take the pointer-doubling fallback), many
    2-cycles, identity, one n-cycle."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(width * 7 + cut_every % 97)
    n = 20_000 if width < 1000 else 3000
    perms = [rng.permutation(n), np.arange(n), np.roll(np.arange(n), 1),
             np.arange(n).reshape(-1, 2)[:, ::-1].reshape(-1)]
    for perm in perms:
        perm = perm.astype(np.int32)
        rows = rng.integers(0, 256, (n, width), dtype=np.uint8)
        dp = torch.from_numpy(rows).cuda()
        _ops.permute_rows(dp, torch.from_numpy(perm).cuda(), cut_every)
        pm.synchronize()
        assert np.array_equal(dp.cpu().numpy(), rows[perm]), f"cut_every={cut_every} width={width}"


@pytest.mark.parametrize("width", [32, 60, 301, 508, 16380])
def test_shift_wide_rows(width):
    """Block exchange with wide payload rows (warp-wide row swaps), both shift kinds and
    sub-range regions, against the oracle's rotation."""
    rng = np.random.default_rng(500 + width)
    sizes = [(1, 777), (777, 1), (1000, 333), (5, 7)] if width < 4096 else [(100, 33), (1, 64), (7, 5)]
    for la, lb in sizes:
        keys = rng.integers(-1000, 1000, la + lb + 10).astype(np.int32)
        payload = rng.integers(0, 256, (la + lb + 10, width), dtype=np.uint8)
        wk, wp = keys.copy(), payload.copy()
        wk[3:3 + la + lb], wp[3:3 + la + lb] = orc.rotate_oracle(keys[3:3 + la + lb], payload[3:3 + la + lb], la)
        for kind in ("linear", "circular"):
            arr = to_gpu(keys, payload)
            pm.shift_region(arr, 3, la, lb, kind)
            assert_same(arr, wk, wp, f"shift_region {kind} {la},{lb},w={width}")


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("width", [0, 4, 300])
def test_merge_peers_block_distributed(dtype, width):
    """pm_merge_peers over a peer-pointer table, every rank of a simulated world on one
    GPU (separate allocations stand in for the peers' blocks; no kernel waits on another
    rank).  Rank outputs concatenated == the oracle's stable merge of the global A|B."""
    import torch

    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(4242 + width + (1 if dtype == np.int64 else 0))
    for world, block, afrac, domain in ((1, 5000, 0.5, 1000), (2, 4096, 0.5, 2**31 - 1), (3, 3001, 0.37, 50),
                                         (5, 2000, 0.71, 2**31 - 1), (4, 8192, 0.5, 7), (3, 1000, 0.0, 10),
                                         (3, 1000, 1.0, 10)):
        n = world * block
        la = int(n * afrac)
        keys = np.concatenate([np.sort(rng.integers(0, domain, la)), np.sort(rng.integers(0, domain, n - la))])
        keys = keys.astype(dtype)
        pay = rng.integers(0, 256, (n, width), dtype=np.uint8)
        want_k, want_p = keys.copy(), pay.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, la, n)
        bk = [torch.from_numpy(keys[k * block:(k + 1) * block].copy()).cuda() for k in range(world)]
        bp = [torch.from_numpy(pay[k * block:(k + 1) * block].copy()).cuda() for k in range(world)]
        for r in range(world):
            ok = torch.empty_like(bk[0])
            op = torch.empty_like(bp[0]) if width else None
            _ops.merge_peers(bk, bp if width else None, la, r, ok, op)
            pm.synchronize()
            sl = slice(r * block, (r + 1) * block)
            assert np.array_equal(ok.cpu().numpy(), want_k[sl]), f"world={world} rank={r} keys"
            if width:
                assert np.array_equal(op.cpu().numpy(), want_p[sl]), f"world={world} rank={r} payload"


def test_distributed_merge_p2p_single_rank_nccl():
    """merge_distributed_p2p over a 1-rank NCCL group (the peer table holds this block)."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2005_12648_b200.dist import merge_distributed_p2p

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29637"
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(78)
        for width in (0, 4):
            keys, payload, middle = random_instance(rng, 300000, 0.4, 1000, width)
            want_k, want_p = keys.copy(), payload.copy()
            orc.seq_merge_buffered(want_k, want_p, 0, middle, len(keys))
            k = torch.from_numpy(keys).cuda()
            p = torch.from_numpy(payload).cuda()
            rk, rp = merge_distributed_p2p(k, p if width else None, middle)
            assert np.array_equal(rk.cpu().numpy(), want_k)
            if width:
                assert np.array_equal(rp.cpu().numpy(), want_p)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("width", [256, 1020])
def test_wide_records_int64_keys(width):
    """int64 keys with wide rows (the key+row-index merge runs with 12-byte records)."""
    from paper_2005_12648_b200 import _ops

    rng = np.random.default_rng(1234 + width)
    for size, split in ((7000, 0.5), (20_001, 0.81)):
        m = int(size * split)
        keys = np.concatenate([np.sort(rng.integers(-2**62, 2**62, m)), np.sort(rng.integers(-2**62, 2**62, size - m))])
        keys[: m // 3] = np.sort(rng.integers(-5, 5, m // 3))  # duplicates in A's prefix
        keys[:m].sort()
        payload = rng.integers(0, 256, (size, width), dtype=np.uint8)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, m, size)
        arr = to_gpu(keys, payload)
        _ops.merge(arr, 0, m, size)
        assert_same(arr, want_k, want_p, f"int64 wide w={width} size={size}")
