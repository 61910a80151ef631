"""Host-side API logic that needs no GPU (validation, counts, cycle law)."""
import math

import pytest

import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import shift as pmshift


def test_job_validation():
    with pytest.raises(ValueError):
        pm.MergeJob(2, 1, 2)
    j = pm.MergeJob(1, 4, 9)
    assert (j.size, j.len_a, j.len_b) == (8, 3, 5)


def test_config_validation():
    with pytest.raises(ValueError):
        pm.RecParConfig(-1)
    with pytest.raises(ValueError):
        pm.RecParConfig(2, size_limit=1)
    with pytest.raises(ValueError):
        pm.RecParConfig(2, shift_kind="diagonal")
    for t in (0, 3, 6, 12):
        with pytest.raises(ValueError):
            pm.check_threads(t)
    assert pm.check_threads(16) == 16


def test_cycle_structure_law():
    # gcd(la, lb) cycles of (la+lb)/gcd each, a disjoint cover (shift.py:113-131)
    for la in range(1, 49):
        for lb in range(1, 49):
            cycles = pm.circular_cycles(la, lb)
            g = math.gcd(la, lb)
            assert len(cycles) == g
            assert [c[0] for c in cycles] == list(range(g))
            assert all(len(c) == (la + lb) // g for c in cycles)
            assert sorted(i for c in cycles for i in c) == list(range(la + lb))
    assert pm.circular_cycles(0, 5) == []
    with pytest.raises(ValueError):
        pm.circular_cycles(-1, 2)


def test_marker_codec_examples():
    c = pm.MarkerCodec(0, 9, 10)
    assert c.mark(5) == 15 and c.is_marked(15) and not c.is_marked(9) and c.unmark(15) == 5


def test_shift_kind_validation():
    with pytest.raises(ValueError):
        pmshift.check_shift_kind("diagonal")
    assert pmshift.check_shift_kind(pm.CIRCULAR) == "circular"
