"""Golden vectors for the benchmark harness from the REFERENCE (run in the build container).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_bench.py

Records the reference's median-quality study (bench.py median_quality_study,
Fig. 5 of the paper) on a small grid and sha256 digests of its input
generator (bench.py generate_input) so that paper_2005_12648_b200.bench is
pinned to both.  Output: tests/golden/bench.npz (committed).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

from parmerge import bench as rb  # noqa: E402  (the reference, read-only)

SIZES = tuple(2**k for k in range(4, 13))
SPLITS = (0.25, 0.5, 0.75)


def main():
    cfg = rb.BenchConfig(sizes=SIZES, splits=SPLITS, seed=1)
    rows = rb.median_quality_study(cfg)
    q = np.array([[r.t, r.size, r.rel_diff] for r in rows], dtype=np.float64)
    gens = []
    for size, split, seed, eb in ((0, 0.5, 1, 4), (1, 0.5, 1, 4), (1000, 0.25, 3, 4), (4097, 0.75, 9, 64),
                                  (333, 0.5, 1, 512)):
        arr, middle = rb.generate_input(size, split, seed, eb)
        h = hashlib.sha256(np.ascontiguousarray(arr.keys).tobytes())
        h.update(np.ascontiguousarray(arr.payload).tobytes())
        gens.append((size, split, seed, eb, middle, h.hexdigest()))
    np.savez(os.path.join(HERE, "bench.npz"), quality=q,
             quality_sizes=np.array(SIZES), quality_splits=np.array(SPLITS),
             gen_params=np.array([g[:5] for g in gens], dtype=np.float64),
             gen_sha=np.array([g[5] for g in gens]))
    print("wrote bench.npz:", len(rows), "quality rows,", len(gens), "generator digests")


if __name__ == "__main__":
    main()
