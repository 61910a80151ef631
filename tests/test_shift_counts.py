"""Instrumented-shift counts pinned to the reference (tests/golden/shift_counts.npz,
made by tests/golden/make_golden_counts.py from the reference's own
linear_shift_instrumented / circular_shift_instrumented / circular_cycles,
shift.py:58-131; its tests test_shift.py:30-36,78-95 check the same bounds)."""
import hashlib

import numpy as np
import pytest

import golden_io

pm = pytest.importorskip("paper_2005_12648_b200")
from paper_2005_12648_b200 import shift as sh  # noqa: E402


def _golden():
    z = golden_io.load("shift_counts.npz")
    return z["counts"], z["digests"], z


def test_counts_match_reference():
    rows, _, _ = _golden()
    for la, lb, ls, lw, lc, cs, cw, cc in rows.tolist():
        lin = sh.linear_shift_counts(la, lb)
        circ = sh.circular_shift_counts(la, lb)
        assert (lin.swaps, lin.writes, lin.cycles) == (ls, lw, lc), (la, lb)
        assert (circ.swaps, circ.writes, circ.cycles) == (cs, cw, cc), (la, lb)
        # the reference's documented bounds (test_shift.py:78-95)
        assert lin.swaps <= la + lb and circ.writes == (la + lb if la and lb else 0)


def test_cycle_orbits_match_reference():
    _, _, z = _golden()
    flat, lens = z["cyc_flat"].tolist(), z["cyc_len"].tolist()
    pos = k = 0
    for la, lb, norb in z["cyc_pairs"].tolist():
        orbits = sh.circular_cycles(la, lb)
        assert len(orbits) == norb, (la, lb)
        for o in orbits:
            assert o == flat[pos:pos + lens[k]], (la, lb)
            pos += lens[k]
            k += 1


@pytest.mark.gpu
def test_instrumented_shifts_on_device():
    import torch

    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    rows, digests, _ = _golden()
    for (la, lb, ls, lw, lc, cs, cw, cc), dig in zip(rows.tolist(), digests.tolist()):
        if (la + lb > 96 and la + lb < 1000) or (la % 5 and la + lb < 96):
            continue  # a spread of the grid plus every large pair
        n = la + lb
        keys = np.arange(n, dtype=np.int32)
        payload = (np.arange(n * 3, dtype=np.int64) % 251).astype(np.uint8).reshape(n, 3)
        for fn, want in ((pm.linear_shift_instrumented, (ls, lw, lc)), (pm.circular_shift_instrumented, (cs, cw, cc))):
            arr = pm.KeyedArray(torch.from_numpy(keys.copy()).cuda(), torch.from_numpy(payload.copy()).cuda())
            st = fn(arr, la, lb)
            assert (st.swaps, st.writes, st.cycles) == want, (fn.__name__, la, lb)
            k, p = arr.numpy()
            h = hashlib.sha256()
            h.update(np.ascontiguousarray(k).tobytes())
            h.update(np.ascontiguousarray(p).tobytes())
            assert h.hexdigest() == dig, (fn.__name__, la, lb)
