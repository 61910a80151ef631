"""The scheduled in-place engine (pm_flow.cu) on its own: every order mode against the
pinned oracle (oracle/, the reference's stable core _kernels.py:227-313), the
device-side fallback, workspace reuse across geometries, and BASELINE config 5
(L_A = L_B = 2^32 int32, 32 GiB) on one GPU."""
import numpy as np
import pytest
import torch

from gen import random_instance
from oracle import oracle as orc

pm = pytest.importorskip("paper_2005_12648_b200")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2005_12648_b200 import _ops  # noqa: E402

MODE_OF = {"two_front": 1, "angle": 2}  # pm_status stats[4] after a scheduled merge


@pytest.fixture
def flow_mode():
    def set_mode(mode):
        _ops.set_engine_only(True)
        _ops.set_flow_mode(mode)
    yield set_mode
    _ops.set_engine_only(False)
    _ops.set_flow_mode("auto")


def to_gpu(keys, payload):
    return pm.KeyedArray(torch.from_numpy(np.ascontiguousarray(keys)).cuda(),
                         torch.from_numpy(np.ascontiguousarray(payload)).cuda())


@pytest.mark.parametrize("mode", ["auto", "two_front", "angle", "fallback"])
@pytest.mark.parametrize("width,dtype", [(0, np.int32), (4, np.int32), (12, np.int32), (0, np.int64), (5, np.int64)])
def test_modes_vs_oracle(flow_mode, mode, width, dtype):
    flow_mode(mode)
    rng = np.random.default_rng(31337 + width + (3 if dtype == np.int64 else 0))
    for size in (9000, 70000, 300001, 1 << 21):
        for domain in (5, 2**31 - 1):
            split = float(rng.choice([0.02, 0.3, 0.5, 0.77, 0.99]))
            keys, payload, middle = random_instance(rng, size, split, domain, width)
            keys = keys.astype(dtype)
            lo, hi = int(rng.integers(0, 5000)), int(rng.integers(0, 300))
            kk = np.concatenate([np.full(lo, -3, dtype), keys, np.full(hi, -9, dtype)])
            pp = np.concatenate([np.full((lo, width), 7, np.uint8), payload, np.full((hi, width), 8, np.uint8)])
            want_k, want_p = kk.copy(), pp.copy()
            orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
            arr = to_gpu(kk, pp)
            st = _ops.merge(arr, lo, lo + middle, lo + size)
            k, p = arr.numpy()
            assert np.array_equal(k, want_k), f"{mode} size={size} dom={domain} split={split} w={width}"
            assert np.array_equal(p, want_p), f"{mode} payload size={size} dom={domain} split={split}"
            if mode in MODE_OF and st[4]:
                assert st[4] == MODE_OF[mode]


@pytest.mark.parametrize("mode", ["auto", "two_front", "angle", "fallback", "bounded"])
@pytest.mark.parametrize("koff,poff,width", [(1, 0, 4), (2, 3, 3), (3, 1, 8), (1, 1, 0)])
def test_misaligned_bases(flow_mode, mode, koff, poff, width):
    """Keys / payload views off the 16-byte grid (slot boundaries are then unaligned):
    every engine stages the pieces exactly (no superset copies) and stays bit-exact."""
    flow_mode(mode)
    rng = np.random.default_rng(5 + koff + 7 * poff)
    for size in (200001, 1 << 21):
        keys, payload, middle = random_instance(rng, size, 0.4, 2**31 - 1, width)
        dk = torch.from_numpy(np.concatenate([np.zeros(koff, np.int32), keys])).cuda()
        pflat = np.concatenate([np.zeros(poff, np.uint8), payload.reshape(-1)])
        dp = torch.from_numpy(pflat).cuda()[poff:].view(size, width) if width else torch.empty((size, 0), dtype=torch.uint8).cuda()
        arr = pm.KeyedArray(dk[koff:], dp)
        assert arr.keys.data_ptr() % 16 != 0
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
        _ops.merge(arr, 0, middle, size)
        k, p = arr.numpy()
        assert np.array_equal(k, want_k) and np.array_equal(p, want_p), (mode, koff, poff, width, size)


def test_pool_overflow_falls_back(flow_mode):
    """A near-rotation needs half the job salvaged (> the pool's N/4 under the
    itinerary order): the plan raises the overflow word and the gated bounded-pool
    engine merges instead."""
    flow_mode("angle")
    h = 1 << 22
    ar = torch.arange(h, device="cuda", dtype=torch.int32)
    k0 = torch.cat([ar + h, ar])
    k0[-1] = 3 * h  # B's last key above A's first: not a pure rotation
    arr = pm.KeyedArray(k0.clone())
    st = _ops.merge(arr, 0, h, 2 * h)
    assert torch.equal(arr.keys, torch.sort(k0).values)
    assert st[4] == 0 and st[13] == 0  # no scheduled order reported: the bounded-pool engine ran


@pytest.mark.parametrize("mode", ["auto", "angle"])
@pytest.mark.parametrize("la,lb,width,dtype", [(1 << 22, 1 << 22, 0, torch.int32), (3 << 21, 5 << 20, 4, torch.int32),
                                                (1 << 21, 1 << 21, 12, torch.int64), (1 << 20, 1 << 22, 0, torch.int64)])
def test_pure_rotation_block_exchange(flow_mode, mode, la, lb, width, dtype):
    """Every B key below every A key (ties are not a rotation) with salvage over the
    pool: the gated three-reversal block exchange runs instead of the bounded-pool
    engine (stats[13]); keys and payload rows exactly B then A."""
    flow_mode(mode)
    g = torch.Generator(device="cuda").manual_seed(la + lb + width)
    a = torch.randint(1000, 2000, (la,), device="cuda", dtype=torch.int64, generator=g).sort().values.to(dtype)
    b = torch.randint(0, 1000, (lb,), device="cuda", dtype=torch.int64, generator=g).sort().values.to(dtype)
    k0 = torch.cat([a, b])
    n = la + lb
    p0 = torch.randint(0, 256, (n, width), device="cuda", dtype=torch.uint8, generator=g)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    st = _ops.merge(arr, 0, la, n)
    assert torch.equal(arr.keys, torch.cat([b, a]))
    assert torch.equal(arr.payload, torch.cat([p0[la:], p0[:la]]))
    if la == lb:  # equal runs: the block swap, decided in the sample phase
        assert st[13] == 1
    if st[13] == 0:  # the plan's salvage fitted the pool: the scheduled engine merged it
        assert st[4] in (1, 2)
    else:
        assert st[4] == 0


def test_lean_plan_small_jobs(flow_mode):
    """Below PM_FLOW_TF_Q regions the plan is the lean two-front one with an N/2 pool:
    the same near-rotation fits it (no fallback), and a uniform job reports the
    two-front order; both bit-exact."""
    flow_mode("auto")
    h = 1 << 22
    ar = torch.arange(h, device="cuda", dtype=torch.int32)
    k0 = torch.cat([ar + h, ar])
    k0[-1] = 3 * h  # (not a pure rotation: those take the block swap)
    arr = pm.KeyedArray(k0.clone())
    _ops.set_engine_only(True)
    try:
        st = _ops.merge(arr, 0, h, 2 * h)
        assert torch.equal(arr.keys, torch.sort(k0).values)
        assert st[4] == 1  # two-front order (FC_MODE 0, reported + 1)
        g = torch.Generator(device="cuda").manual_seed(9)
        k1 = torch.randint(0, 1 << 20, (2 * h,), device="cuda", dtype=torch.int32, generator=g)
        k1[:h] = k1[:h].sort().values
        k1[h:] = k1[h:].sort().values
        p1 = torch.arange(2 * h, device="cuda", dtype=torch.int32).view(torch.uint8).view(2 * h, 4)
        arr = pm.KeyedArray(k1.clone(), p1.clone())
        st = _ops.merge(arr, 0, h, 2 * h)
        order = torch.sort(k1, stable=True).indices
        assert torch.equal(arr.keys, k1[order]) and torch.equal(arr.payload, p1[order])
        assert st[4] == 1
    finally:
        _ops.set_engine_only(False)


@pytest.mark.parametrize("kind", ["window", "translated", "uniform"])
def test_early_two_front_decision(flow_mode, kind):
    """Above PM_FLOW_TF_Q regions the plan counts the two-front salvage first and
    skips the itinerary phases when it is already below n/32 (config-3-like skew,
    a translated run); a uniform job still evaluates and takes the angle order.
    Key + index payload, checked against a stable sort."""
    flow_mode("auto")
    g = torch.Generator(device="cuda").manual_seed(77)
    la = 1 << 27
    if kind == "window":  # B (2^16) inside a narrow window of A, as config 3
        a = torch.randint(-(1 << 62), 1 << 62, (la,), device="cuda", dtype=torch.int64, generator=g).sort().values
        lo, hi = a[la // 2 - (1 << 12)].item(), a[la // 2 + (1 << 12)].item()
        b = torch.randint(lo, hi, (1 << 16,), device="cuda", dtype=torch.int64, generator=g).sort().values
    elif kind == "translated":  # B = A's keys shifted up by a little: a near-translation
        a = torch.randint(0, 1 << 40, (la,), device="cuda", dtype=torch.int64, generator=g).sort().values
        b = a[: la // 2] + (1 << 20)
    else:
        a = torch.randint(0, 1 << 40, (la,), device="cuda", dtype=torch.int64, generator=g).sort().values
        b = torch.randint(0, 1 << 40, (la,), device="cuda", dtype=torch.int64, generator=g).sort().values
    k0 = torch.cat([a, b])
    n = k0.numel()
    p0 = torch.arange(n, device="cuda", dtype=torch.int32).view(torch.uint8).view(n, 4)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    st = _ops.merge(arr, 0, la, n)
    order = torch.sort(k0, stable=True).indices
    assert torch.equal(arr.keys, k0[order]) and torch.equal(arr.payload, p0[order])
    if kind == "uniform":
        assert st[4] == 2 and st[5] < n  # angle order, both orders evaluated
    elif kind == "window":
        assert st[4] == 1 and st[5] == 2**64 - 1  # two fronts, angle phases skipped
    if st[5] == 2**64 - 1:
        assert st[4] == 1 and st[6] * 32 <= n


@pytest.mark.parametrize("dist", ["exp", "steps", "clustered"])
def test_split_search_skewed_keys(flow_mode, dist):
    """The split phase interpolates between sample values before its binary search;
    key distributions far from linear (exponential, step-like, clustered) must give
    the same bit-exact merge (the bracket invariant never depends on the guess)."""
    flow_mode("auto")
    rng = np.random.default_rng({"exp": 1, "steps": 2, "clustered": 3}[dist])
    n = 1 << 22
    if dist == "exp":
        raw = np.exp(rng.uniform(0, 21, n)).astype(np.int64)
    elif dist == "steps":
        raw = (rng.integers(0, 6, n) * (1 << 28) + rng.integers(0, 3, n)).astype(np.int64)
    else:
        c = rng.integers(0, 2**31 - 2**20, 7)
        raw = c[rng.integers(0, 7, n)] + rng.integers(0, 2**10, n)
    keys = raw.astype(np.int32)
    m = int(n * 0.45)
    keys[:m].sort()
    keys[m:].sort()
    payload = np.arange(n, dtype=np.int32).view(np.uint8).reshape(n, 4)
    want_k, want_p = keys.copy(), payload.copy()
    orc.seq_merge_buffered(want_k, want_p, 0, m, n)
    arr = to_gpu(keys, payload)
    _ops.merge(arr, 0, m, n)
    k, p = arr.numpy()
    assert np.array_equal(k, want_k) and np.array_equal(p, want_p), dist


def test_geometries_back_to_back(flow_mode):
    """Workspace and pool reuse across shrinking / growing jobs and key widths."""
    flow_mode("auto")
    rng = np.random.default_rng(77)
    for size, dtype, width in [(1 << 22, np.int32, 0), (3 << 18, np.int64, 0), (1 << 23, np.int32, 4),
                               (12345, np.int32, 0), (1 << 22, np.int64, 8)]:
        keys, payload, middle = random_instance(rng, size, 0.5, 2**31 - 1, width)
        keys = keys.astype(dtype)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, size)
        arr = to_gpu(keys, payload)
        _ops.merge(arr, 0, middle, size)
        k, p = arr.numpy()
        assert np.array_equal(k, want_k) and np.array_equal(p, want_p), (size, dtype, width)


def _mix(x, a, b):
    """int64 hash of int64 keys (wrapping arithmetic): multiset fingerprints."""
    y = x * a + b
    y = y ^ (y >> 29)
    return y * 0x5851F42D4C957F2D


def test_config5_single_gpu_full_size():
    """BASELINE config 5 on ONE B200: L_A = L_B = 2^32 uniform int32 (2^33 records,
    32 GiB) merged in place by the scheduled engine (int64 record indices end to end).
    Checks: sorted output; two multiset fingerprints of input == output; the exact
    rank of 256 pivot values (records < v, from searchsorted on regenerated runs);
    64 output windows equal to an independent merge of the regenerated runs."""
    from paper_2005_12648_b200.workloads import sorted_uniform_device

    L = 1 << 32
    free = torch.cuda.mem_get_info()[0]
    if free < (80 << 30):  # pragma: no cover
        pytest.skip("needs ~80 GB of free device memory")
    keys = torch.empty(2 * L, dtype=torch.int32, device="cuda")
    sorted_uniform_device(L, 50, out=keys[:L])
    sorted_uniform_device(L, 51, out=keys[L:])
    fp_in = [0, 0]
    C = 1 << 28
    for c in range(0, 2 * L, C):
        x = keys[c:c + C].to(torch.int64)
        fp_in[0] += int(_mix(x, 0x9E3779B97F4A7C15, 7).sum().item())
        fp_in[1] += int(_mix(x, 0xD1B54A32D192ED03, 11).sum().item())
    arr = pm.KeyedArray(keys)
    st = _ops.merge(arr, 0, L, 2 * L)
    assert st[2] > 0 and st[4] in (1, 2)  # the scheduled engine ran
    fp_out = [0, 0]
    for c in range(0, 2 * L, C):
        blk = keys[c:min(c + C + 1, 2 * L)]
        assert bool(torch.all(blk[1:] >= blk[:-1]).item()), f"unsorted near {c}"
        x = keys[c:c + C].to(torch.int64)
        fp_out[0] += int(_mix(x, 0x9E3779B97F4A7C15, 7).sum().item())
        fp_out[1] += int(_mix(x, 0xD1B54A32D192ED03, 11).sum().item())
    M64 = (1 << 64) - 1
    assert [v & M64 for v in fp_out] == [v & M64 for v in fp_in]
    # regenerate the runs; exact ranks of pivot values and exact output windows
    runs = torch.empty(2 * L, dtype=torch.int32, device="cuda")
    A, B = sorted_uniform_device(L, 50, out=runs[:L]), sorted_uniform_device(L, 51, out=runs[L:])
    g = torch.Generator(device="cuda").manual_seed(9)
    piv = torch.randint(0, 2**31, (256,), generator=g, device="cuda", dtype=torch.int32)
    want = torch.searchsorted(A, piv).to(torch.int64) + torch.searchsorted(B, piv).to(torch.int64)
    got = torch.searchsorted(keys, piv).to(torch.int64)
    assert torch.equal(got, want)
    W = 4096
    starts = torch.randint(0, 2 * L - W, (64,), generator=g, device="cuda", dtype=torch.int64).tolist()
    for p in starts:
        # stable merge path: i records of A among the first p outputs
        lo, hi = max(0, p - L), min(p, L)
        while lo < hi:
            mid = (lo + hi) // 2
            if int(A[mid].item()) <= int(B[p - 1 - mid].item()):
                lo = mid + 1
            else:
                hi = mid
        a0, b0 = lo, p - lo
        cand = torch.cat([A[a0:a0 + W], B[b0:b0 + W]]).sort(stable=True).values[:W]
        assert torch.equal(keys[p:p + W], cand), f"window at {p}"


@pytest.mark.parametrize("width", [0, 4, 7])
def test_reorder_prescribed_layouts(width):
    """pm_reorder (reorder_multi's one-pass device realisation): random leaf layouts
    A_0 B_0 A_1 B_1 ... over sizes up to 2^22 against a host gather of the slices."""
    rng = np.random.default_rng(404 + width)
    for n, t in [(1 << 12, 2), (100003, 8), (1 << 20, 64), (3 << 20, 1024), (1 << 22, 16)]:
        la = int(rng.integers(1, n))
        cuts_a = np.sort(rng.integers(0, la + 1, t - 1))
        cuts_b = np.sort(rng.integers(0, n - la + 1, t - 1))
        ea = np.diff(np.concatenate([[0], cuts_a, [la]]))
        eb = np.diff(np.concatenate([[0], cuts_b, [n - la]]))
        sizes = [int(x) for pair in zip(ea, eb) for x in pair]
        keys = rng.integers(-2**31, 2**31 - 1, n).astype(np.int32)
        payload = rng.integers(0, 256, (n, width), dtype=np.uint8)
        lo = int(rng.integers(0, 50))
        kk = np.concatenate([np.full(lo, 9, np.int32), keys, np.full(3, 8, np.int32)])
        pp = np.concatenate([np.zeros((lo, width), np.uint8), payload, np.ones((3, width), np.uint8)])
        srcs, a0, b0 = [], 0, la
        for i in range(t):
            srcs.append((a0, int(ea[i])))
            srcs.append((b0, int(eb[i])))
            a0 += int(ea[i])
            b0 += int(eb[i])
        want_k = kk.copy()
        want_p = pp.copy()
        want_k[lo:lo + n] = np.concatenate([keys[s:s + c] for s, c in srcs])
        want_p[lo:lo + n] = np.concatenate([payload[s:s + c] for s, c in srcs])
        arr = to_gpu(kk, pp)
        _ops.reorder(arr, lo, lo + n, sizes)
        k, p = arr.numpy()
        assert np.array_equal(k, want_k) and np.array_equal(p, want_p), (n, t, width)


@pytest.mark.parametrize("cfg", [4, 3, 2])
def test_full_size_matches_reference_checksum(cfg):
    """BASELINE configs 2/3/4 at FULL size (2^30 int32; 2^28 + 2^16 int64 skew; 2^27
    key + index records) against sha256 checksums of the REFERENCE's own stable core
    on the same seeded inputs (tests/golden/make_golden_full.py)."""
    import hashlib

    import golden_io
    from gen import config_input

    g = golden_io.load("big_full.npz")
    keys, payload, middle = config_input(cfg, seed=0, log_len=29 if cfg == 2 else None)

    def sha(*arrays):
        h = hashlib.sha256()
        for a in arrays:
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    assert sha(keys, payload) == str(g[f"cfg{cfg}_in"]), "host generator drifted from the golden input"
    arr = to_gpu(keys, payload)
    del keys, payload
    pm.merge_srecpar(arr, pm.MergeJob(0, middle, len(arr)), 8)
    k, p = arr.numpy()
    assert sha(k, p) == str(g[f"cfg{cfg}_out"])
