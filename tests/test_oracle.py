"""Pin the CPU oracle (oracle/) against the reference's own outputs (CPU only).

The golden vectors were produced by the reference package itself
(tests/golden/make_golden.py); the known-answer examples restate the frozen
examples in the reference's tests (test_median.py:68-87, test_shift.py:24-51,
test_soptmov.py:37-41).
"""
import hashlib

import numpy as np
import pytest

import golden_io
from gen import config_input
from oracle import oracle as orc


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_known_answers_find_median():
    a32 = lambda x: np.array(x, np.int32)  # noqa: E731
    assert orc.find_median(a32([1, 2]), a32([3, 4])) == (2, 0)
    assert orc.find_median(a32([5, 6]), a32([1, 2])) == (0, 2)
    assert orc.find_median(a32([]), a32([1, 2, 3])) == (0, 0)
    assert orc.find_median(a32([1, 2]), a32([])) == (2, 0)
    assert orc.find_median(a32([1, 3, 5, 7]), a32([2, 4, 6, 8])) == (2, 2)


def test_known_answers_shift():
    k = np.array([10, 11, 1, 2, 3], np.int32)
    orc.linear_shift(k, None, 0, 2, 3)
    assert k.tolist() == [1, 2, 3, 10, 11]
    k = np.array([1, 2, 9], np.int32)
    orc.circular_shift(k, None, 0, 2, 1)
    assert k.tolist() == [9, 1, 2]


def test_known_answer_plan():
    k = np.array([1, 3, 5, 7, 2, 4, 6, 8], np.int32)
    src, fin = orc.plan_intervals(k, 0, 4, 8, 2)
    assert src == [(0, 2), (4, 2), (2, 2), (6, 2)]
    assert fin == [(0, 2, 4), (4, 6, 8)]


def test_find_median_matches_reference():
    n = 0
    for a, b, piv in golden_io.median_cases():
        assert orc.find_median(a, b) == piv
        n += 1
    assert n == 3000


@pytest.mark.parametrize("name", ["merge_i32.npz", "merge_i64.npz"])
def test_buffered_merge_matches_reference(name):
    for c in golden_io.merge_cases(name):
        s, m, e = (int(x) for x in c["job"])
        k, p = c["keys"].copy(), c["payload"].copy()
        orc.seq_merge_buffered(k, p, s, m, e)
        assert np.array_equal(k, c["out_keys"]) and np.array_equal(p, c["out_payload"])
        # independent restatement: stable argsort
        k2, p2 = orc.stable_merge_numpy(c["keys"], c["payload"], s, m, e)
        assert np.array_equal(k2, c["out_keys"]) and np.array_equal(p2, c["out_payload"])
        # rotation merge is stable too and must agree element-exactly
        if name == "merge_i32.npz":
            for circ in (False, True):
                k3, p3 = c["keys"].copy(), c["payload"].copy()
                orc.rotation_merge(k3, p3, s, m, e, circ)
                assert np.array_equal(k3, c["out_keys"]) and np.array_equal(p3, c["out_payload"])


def test_srecpar_port_sorts_like_reference():
    for c in golden_io.merge_cases("merge_i32.npz"):
        s, m, e = (int(x) for x in c["job"])
        k, p = c["keys"].copy(), c["payload"].copy()
        orc.srecpar_buffered(k, p, s, m, e, 8, size_limit=2)
        assert np.array_equal(k, c["srecpar_keys"])


def test_shifts_match_reference():
    for c in golden_io.shift_cases():
        la, lb = (int(x) for x in c["len"])
        for fn in (orc.linear_shift, orc.circular_shift):
            k, p = c["keys"].copy(), c["payload"].copy()
            fn(k, p, 0, la, lb)
            assert np.array_equal(k, c["out_keys"]) and np.array_equal(p, c["out_payload"])
        k, p = orc.rotate_oracle(c["keys"], c["payload"], la)
        assert np.array_equal(k, c["out_keys"]) and np.array_equal(p, c["out_payload"])


def test_plan_matches_reference():
    for c in golden_io.plan_cases():
        s, m, e, t = (int(x) for x in c["job"])
        src, fin = orc.plan_intervals(c["keys"], s, m, e, t)
        assert np.array_equal(np.array(src, np.int64).reshape(-1, 2), c["sources"])
        assert np.array_equal(np.array(fin, np.int64).reshape(-1, 3), c["finals"])


def test_merge_path_is_stable_split():
    rng = np.random.default_rng(7)
    for _ in range(200):
        la, lb = (int(x) for x in rng.integers(0, 60, 2))
        a = np.sort(rng.integers(0, 8, la)).astype(np.int32)
        b = np.sort(rng.integers(0, 8, lb)).astype(np.int32)
        keys = np.concatenate([a, b])
        tag = np.arange(la + lb)
        order = np.argsort(keys, kind="stable")
        for d in range(la + lb + 1):
            assert orc.merge_path(a, b, d) == int((tag[order[:d]] < la).sum())


def test_big_checksums_match_reference():
    g = golden_io.big()
    keys, payload, middle = config_input(1, seed=0)
    assert sha(keys) == g["cfg1_in"]
    orc.seq_merge_buffered(keys, payload, 0, middle, len(keys))
    assert sha(keys) == g["cfg1_out"]
    keys, payload, middle = config_input(4, seed=0, log_len=18)
    assert sha(keys, payload) == g["cfg4s_in"]
    orc.seq_merge_buffered(keys, payload, 0, middle, len(keys))
    assert sha(keys, payload) == g["cfg4s_out"]
    keys, payload, middle = config_input(3, seed=0, log_len=20, log_len_b=12)
    assert sha(keys) == g["cfg3s_in"]
    orc.seq_merge_buffered(keys, payload, 0, middle, len(keys))
    assert sha(keys) == g["cfg3s_out"]
