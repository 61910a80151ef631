"""Golden operation counts of the reference's instrumented shifts (run in the build container).

    python tests/golden/make_golden_counts.py

Calls the REFERENCE's ``linear_shift_instrumented`` / ``circular_shift_instrumented``
(shift.py:58-110) and ``circular_cycles`` (shift.py:113-131) -- pure Python, no
numba -- imported from /root/reference/pkg/src (read-only), for every
(len_a, len_b) in [0, 48]^2 plus a few larger pairs, and records the returned
ShiftStats, the shifted keys' checksum and (for small pairs) the cycle orbits.
Output: tests/golden/shift_counts.npz (committed; the GPU box never reads
/root/reference).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import parmerge as ref  # noqa: E402  (the reference, read-only)
from parmerge import shift as ref_shift  # noqa: E402


def main():
    pairs = [(a, b) for a in range(49) for b in range(49)]
    pairs += [(100, 37), (37, 100), (1000, 1), (1, 1000), (512, 512), (999, 333), (1024, 768), (4097, 61)]
    rows = []
    digests = []
    for la, lb in pairs:
        n = la + lb
        keys = np.arange(n, dtype=np.int32)
        payload = (np.arange(n * 3, dtype=np.int64) % 251).astype(np.uint8).reshape(n, 3)
        a1 = ref.KeyedArray(keys.copy(), payload.copy())
        s1 = ref_shift.linear_shift_instrumented(a1, la, lb)
        a2 = ref.KeyedArray(keys.copy(), payload.copy())
        s2 = ref_shift.circular_shift_instrumented(a2, la, lb)
        assert np.array_equal(a1.keys, a2.keys)
        rows.append((la, lb, s1.swaps, s1.writes, s1.cycles, s2.swaps, s2.writes, s2.cycles))
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(a1.keys).tobytes())
        h.update(np.ascontiguousarray(a1.payload).tobytes())
        digests.append(h.hexdigest())
    cyc_pairs, cyc_flat, cyc_len = [], [], []
    for la in range(13):
        for lb in range(13):
            orbits = ref_shift.circular_cycles(la, lb)
            cyc_pairs.append((la, lb, len(orbits)))
            for o in orbits:
                cyc_len.append(len(o))
                cyc_flat.extend(int(x) for x in o)
    np.savez_compressed(os.path.join(HERE, "shift_counts.npz"),
                        counts=np.array(rows, np.int64), digests=np.array(digests),
                        cyc_pairs=np.array(cyc_pairs, np.int64), cyc_len=np.array(cyc_len, np.int64),
                        cyc_flat=np.array(cyc_flat, np.int64))
    print(f"{len(rows)} count rows, {len(cyc_pairs)} orbit pairs")


if __name__ == "__main__":
    main()
