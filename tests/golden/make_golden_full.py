"""Reference checksums at BASELINE.json's FULL config sizes (run in the build container).

    NUMBA_CACHE_DIR=/tmp/numba_cache_golden python tests/golden/make_golden_full.py

The reference's own stable core (seq_merge_buffered, seqmerge.py:55-75; for int64
keys _kernels.buffered_merge directly, records.py truncates to int32) run on the
seeded host inputs of workloads.config_input at full size:
  config 2: int32, L_A = L_B = 2^29 (2^30 records), seed 0
  config 3: int64, L_A = 2^28, L_B = 2^16 in a narrow window, seed 0
  config 4: int32 keys in [0, 1024) + int32 index payload, L_A = L_B = 2^26, seed 0
Records sha256 of the inputs and outputs (tests/golden/big_full.npz, committed);
tests/test_parity_gpu.py regenerates the inputs on the GPU box with the same numpy
generator and compares the device merge's output checksum.
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
from parmerge import _kernels  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from gen import config_input  # noqa: E402  (tests/gen.py)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    _kernels.warmup()
    out = {}
    for cfg in (4, 3, 2):
        keys, payload, middle = config_input(cfg, seed=0, log_len=29 if cfg == 2 else None)
        out[f"cfg{cfg}_in"] = sha(keys, payload)
        if cfg == 3:  # int64: the numba kernel directly
            k = keys.copy()
            pl = np.empty((len(k), 0), np.uint8)
            n = min(middle, len(k) - middle)
            _kernels.buffered_merge(k, pl, 0, middle, len(k), np.empty(n, np.int64), np.empty((n, 0), np.uint8))
            out[f"cfg{cfg}_out"] = sha(k, pl)
        else:
            arr = ref.KeyedArray(keys.copy(), payload.copy())
            ref.seq_merge_buffered(arr, ref.MergeJob(0, middle, len(keys)))
            out[f"cfg{cfg}_out"] = sha(arr.keys, arr.payload)
        print(cfg, out[f"cfg{cfg}_in"][:16], out[f"cfg{cfg}_out"][:16], flush=True)
        del keys, payload
    np.savez(os.path.join(HERE, "big_full.npz"), **{k: np.array(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
