"""Pivot search (mirror of ``parmerge.median``).

``find_median`` runs the reference's Alg. 1 double binary search on the GPU
(``pm_find_median``, median.py:23-60) and returns the identical pivot pair.
The GPU merge pipeline itself splits with the *stable* merge path
(``find_splits``); Alg. 1 lets equal keys cross the split, which is why the
reference's parallel merges are unstable.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _ops


class PivotPair(NamedTuple):
    """Split offsets (p_a into run A, p_b into run B), median.py:11-20."""

    p_a: int
    p_b: int


def find_median(a, b, *, key=None) -> PivotPair:
    """Double binary search for a balanced valid pivot pair (median.py:23-60), on the device.

    ``a``/``b`` are sorted int32/int64 runs: CUDA tensors (zero-copy) or host
    sequences (copied to the device).  ``key=`` extractors are host-only and are
    not supported on the GPU path.
    """
    if key is not None:
        raise NotImplementedError("find_median(key=...) is not supported on the GPU path")
    return PivotPair(*_ops.find_median(a, b))


def find_splits(a, b, diagonals) -> torch.Tensor:
    """Stable merge-path A-counts at ``diagonals`` (A wins ties), on the device."""
    return _ops.find_splits(a, b, torch.as_tensor(diagonals))


def find_median_optimal(a, b, *, key=None) -> PivotPair:
    """Best-balance valid pivot pair (median.py:63-73), computed with device searches.

    Same definition and tie rule as the reference (smallest p_a, then p_b).
    """
    if key is not None:
        raise NotImplementedError("find_median_optimal(key=...) is not supported on the GPU path")
    ta, tb = _ops._run_tensor(a), _ops._run_tensor(b)
    if ta.dtype != tb.dtype:
        ta, tb = ta.to(torch.int64), tb.to(torch.int64)
    la, lb = ta.numel(), tb.numel()
    total = la + lb
    if la == 0:
        return PivotPair(0, min(max(total // 2, 0), lb))
    dev = ta.device
    lo = torch.zeros(la + 1, dtype=torch.int64, device=dev)
    lo[1:] = torch.searchsorted(tb, ta, right=False)
    hi = torch.full((la + 1,), lb, dtype=torch.int64, device=dev)
    hi[:la] = torch.searchsorted(tb, ta, right=True)
    pa = torch.arange(la + 1, dtype=torch.int64, device=dev)
    floor_c = torch.minimum(torch.maximum(torch.div(total - 2 * pa, 2, rounding_mode="floor"), lo), hi)
    ceil_c = torch.minimum(torch.maximum(torch.div(total - 2 * pa + 1, 2, rounding_mode="floor"), lo), hi)
    bal_floor = (2 * (pa + floor_c) - total).abs()
    bal_ceil = (2 * (pa + ceil_c) - total).abs()
    pb = torch.where(bal_ceil < bal_floor, ceil_c, floor_c)
    bal = torch.minimum(bal_floor, bal_ceil)
    i = int(torch.argmin(bal).item())
    return PivotPair(i, int(pb[i].item()))


def pivot_invariants_hold(a, b, pivots, *, key=None) -> bool:
    """Check the two cross inequalities a pivot pair must satisfy (median.py:126-136)."""
    k = key if key is not None else (lambda x: x)
    p_a, p_b = pivots
    a = a.tolist() if isinstance(a, (torch.Tensor, np.ndarray)) else a
    b = b.tolist() if isinstance(b, (torch.Tensor, np.ndarray)) else b
    la, lb = len(a), len(b)
    in_range = 0 <= p_a <= la and 0 <= p_b <= lb
    # left part of each run <= right part of the other (where both sides exist)
    a_left_ok = not (in_range and 0 < p_a and p_b < lb) or k(a[p_a - 1]) <= k(b[p_b])
    b_left_ok = not (in_range and 0 < p_b and p_a < la) or k(b[p_b - 1]) <= k(a[p_a])
    return in_range and a_left_ok and b_left_ok
