"""Acceptance criteria of the reference (tests/test_acceptance.py) run against the device path.

* correctness sweep: 1000 seeded instances (sizes 0..16384, forced edges, heavy
  duplicates, random-walk runs) through every strategy at t in {1,2,4,8,16};
  keys AND payload (the stable order) must equal the pinned oracle's merge --
  stricter than the reference's key-only check;
* layout equivalence: the plan's leaf sources gathered in order equal the array
  the recursive division leaves, and the leaf jobs agree (plan_intervals vs
  division_trace);
* pivot contract and median quality: every Alg. 1 / optimal pivot on the
  division tree keeps the cross inequalities, and at t = 2 the heuristic is
  never better than the optimum.
"""
import numpy as np
import pytest
import torch

from gen import generate_input
from oracle import oracle as orc

pm = pytest.importorskip("paper_2005_12648_b200")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _instance(rng, i):
    forced = (0, 1, 2, 3, 16383, 16384)
    size = forced[i] if i < len(forced) else min(16384, int(2 ** rng.uniform(0.0, 14.0)))
    split = (0.25, 0.5, 0.75, float(rng.random()))[i % 4]
    width = (0, 4, 12)[i % 3]
    if i % 5 == 0:
        keys, _, middle = generate_input(size, split, seed=int(rng.integers(1 << 30)))
    else:
        domain = int(rng.choice([4, 100, 10**6]))
        middle = int(size * split + 0.5)
        keys = np.concatenate([np.sort(rng.integers(0, domain, middle)),
                               np.sort(rng.integers(0, domain, size - middle))]).astype(np.int32)
    payload = rng.integers(0, 256, (size, width), dtype=np.uint8)
    return keys, payload, middle


def test_correctness_sweep_all_strategies():
    rng = np.random.default_rng(8102024)
    for i in range(1000):
        keys, payload, middle = _instance(rng, i)
        n = len(keys)
        want_k, want_p = keys.copy(), payload.copy()
        orc.seq_merge_buffered(want_k, want_p, 0, middle, n)
        dk, dp = torch.from_numpy(keys).cuda(), torch.from_numpy(payload).cuda()
        job = pm.MergeJob(0, middle, n)
        runs = [("seq-rotation", lambda a: pm.seq_merge_rotation(a, job)),
                ("seq-buffered", lambda a: pm.seq_merge_buffered(a, job))]
        for t in (1, 2, 4, 8, 16):
            runs += [(f"soptmov t={t}", lambda a, t=t: pm.merge_soptmov(a, job, t)),
                     (f"srecpar-ls t={t}", lambda a, t=t: pm.merge_srecpar(a, job, t, shift_kind=pm.LINEAR)),
                     (f"srecpar-cs t={t}", lambda a, t=t: pm.merge_srecpar(a, job, t, shift_kind=pm.CIRCULAR))]
        for name, run in runs:
            arr = pm.KeyedArray(dk.clone(), dp.clone())
            run(arr)
            k, p = arr.numpy()
            assert np.array_equal(k, want_k), f"{name} keys, instance {i} (n={n}, middle={middle})"
            assert np.array_equal(p, want_p), f"{name} payload, instance {i} (n={n}, middle={middle})"


def test_layout_equivalence_plan_vs_division():
    rng = np.random.default_rng(15)
    for i in range(120):
        size = int(rng.integers(32, 4096))
        split = float(rng.choice([0.25, 0.5, 0.75, rng.random()]))
        if i % 2 == 0:
            keys, payload, middle = generate_input(size, split, seed=int(rng.integers(1 << 30)), elem_bytes=8)
        else:
            middle = int(size * split + 0.5)
            keys = np.concatenate([np.sort(rng.integers(0, 10**6, middle)),
                                   np.sort(rng.integers(0, 10**6, size - middle))]).astype(np.int32)
            payload = np.empty((size, 0), np.uint8)
        arr = pm.KeyedArray(keys, payload)
        job = pm.MergeJob(0, middle, size)
        for t in (2, 4, 8, 16):
            plan = pm.plan_intervals(arr, job, t)
            gathered = np.concatenate([keys[s:s + n] for s, n in plan.leaf_sources])
            trace = pm.division_trace(arr, job, t, size_limit=2)
            assert np.array_equal(trace.divided.keys.cpu().numpy(), gathered), (size, t)
            if len(trace.records) == t - 1:
                assert list(trace.leaf_jobs) == list(plan.final_positions), (size, t)


def _tree_max(keys, middle, t, median_fn):
    pairs = [(keys[:middle], keys[middle:])]
    for _ in range(t.bit_length() - 1):
        nxt = []
        for a, b in pairs:
            p_a, p_b = median_fn(a, b)
            assert pm.pivot_invariants_hold(a, b, (p_a, p_b)), (len(a), len(b), p_a, p_b)
            nxt += [(a[:p_a], b[:p_b]), (a[p_a:], b[p_b:])]
        pairs = nxt
    return max(len(a) + len(b) for a, b in pairs)


def test_pivot_contract_and_median_quality():
    for t in (2, 4, 8, 16):
        for exp in range(8, 15):
            for split in (0.25, 0.5, 0.75):
                keys, _, middle = generate_input(2**exp, split, seed=1000 + exp)
                dk = torch.from_numpy(keys).cuda()
                heur = _tree_max(dk, middle, t, pm.find_median)
                best = _tree_max(dk, middle, t, pm.find_median_optimal)
                if t == 2:  # one division cannot beat the single-level optimum
                    assert heur >= best, (exp, split)
