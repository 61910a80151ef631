"""The engine protocol (tests/model_engine.py mirrors pm_engine.cu) under random
interleavings: always terminates, never runs out of salvage space with the
bounded pool, and produces the reference's stable merge / rotation exactly."""
import random

import numpy as np
import pytest

from gen import random_instance
from model_engine import EngineModel
from oracle import oracle as orc


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("inflight", [1, 3, 12])
@pytest.mark.parametrize("mu", [1, 4])
def test_model_merge_matches_oracle(seed, inflight, mu):
    rng = np.random.default_rng(seed)
    size = int(rng.integers(200, 3000))
    split = float(rng.choice([0.1, 0.5, 0.9, rng.random()]))
    domain = int(rng.choice([5, 100, 10**6]))
    keys, payload, middle = random_instance(rng, size, split, domain, 2)
    lo = int(rng.integers(0, 20))
    kk = np.concatenate([np.full(lo, -3, np.int32), keys, np.full(7, -9, np.int32)])
    pp = np.concatenate([np.zeros((lo, 2), np.uint8), payload, np.ones((7, 2), np.uint8)])
    want_k, want_p = kk.copy(), pp.copy()
    orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
    T = 64 // mu
    scratch = inflight * (mu + 4) + 16  # the device's O(grid * tile) pool rule
    m = EngineModel(kk.copy(), pp.copy(), lo, lo + middle, lo + size, T, mu, scratch)
    m.run(inflight, random.Random(seed * 31 + inflight))
    assert np.array_equal(m.keys, want_k) and np.array_equal(m.pay, want_p)


@pytest.mark.parametrize("seed", range(4))
def test_model_rotation_matches_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    la, lb = (int(x) for x in rng.integers(1, 1500, 2))
    keys = rng.integers(-50, 50, la + lb).astype(np.int32)
    pay = rng.integers(0, 256, (la + lb, 3), dtype=np.uint8)
    wk, wp = orc.rotate_oracle(keys, pay, la)
    m = EngineModel(keys.copy(), pay.copy(), 0, la, la + lb, 16, 4, 40, mode="rotate")
    m.run(5, random.Random(seed))
    assert np.array_equal(m.keys, wk) and np.array_equal(m.pay, wp)


def test_model_skew_uses_identity_regions():
    rng = np.random.default_rng(9)
    a = np.sort(rng.integers(0, 10**6, 4000)).astype(np.int32)
    b = np.sort(rng.integers(500000, 500100, 100)).astype(np.int32)
    keys = np.concatenate([a, b])
    pay = np.zeros((len(keys), 0), np.uint8)
    wk = np.sort(keys, kind="stable")
    m = EngineModel(keys.copy(), pay.copy(), 0, 4000, 4100, 16, 4, 40)
    m.run(6, random.Random(1))
    assert np.array_equal(m.keys, wk)
