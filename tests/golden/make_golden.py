"""Generate golden vectors from the REFERENCE implementation (run in the build container).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only; numba
needs a writable cache dir) and records, for seeded inputs, what the reference
itself returns.  The fixtures (``*.npz``) are committed; the GPU box never
reads /root/reference.  The fixtures pin both the CPU oracle (oracle/) and the
CUDA path (tests/test_parity_gpu.py).

What is recorded, with the reference entry point that produced it:
  merge_*.npz     seq_merge_buffered          (seqmerge.py:55-75)   -- stable, payload exact
                  seq_merge_rotation          (seqmerge.py:37-52)   -- must equal buffered
                  merge_srecpar/merge_soptmov (keys; they are unstable at t>1)
  merge_i64.npz   _kernels.buffered_merge called directly with int64 arrays
                  (KeyedArray truncates keys to int32, records.py:9,27)
  median.npz      find_median                 (median.py:23-60)
  shift.npz       linear_shift / circular_shift (shift.py:38-47), with payload
  plan.npz        plan_intervals              (soptmov.py:93-123) + division_trace layout
  big.npz         sha256 of seq_merge_buffered output on config-1 / config-4-shaped inputs
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
from gen import config_input, random_instance  # noqa: E402  (tests/gen.py)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def merge_cases():
    rng = np.random.default_rng(20261019)
    out = {}
    i = 0
    sizes = [0, 1, 2, 3, 5, 16, 31, 64, 100, 257, 511, 1000, 2049]
    for size in sizes:
        for split in (0.0, 0.25, 0.5, 0.75, 1.0, float(rng.random())):
            for domain in (4, 1000, 2**31 - 1):
                w = int(rng.choice([0, 4, 8, 12])) if size < 1000 else int(rng.choice([0, 4]))
                keys, payload, middle = random_instance(rng, size, split, domain, w)
                arr = ref.KeyedArray(keys.copy(), payload.copy())
                job = ref.MergeJob(0, middle, size)
                ref.seq_merge_buffered(arr, job)
                rot = ref.KeyedArray(keys.copy(), payload.copy())
                ref.seq_merge_rotation(rot, job)
                assert rot.equals(arr)
                srp = ref.KeyedArray(keys.copy(), payload.copy())
                ref.merge_srecpar(srp, job, 8, size_limit=2)
                sop = ref.KeyedArray(keys.copy(), payload.copy())
                ref.merge_soptmov(sop, job, 4)
                p = f"c{i}_"
                out[p + "keys"] = keys
                out[p + "payload"] = payload
                out[p + "job"] = np.array([0, middle, size], np.int64)
                out[p + "out_keys"] = arr.keys
                out[p + "out_payload"] = arr.payload
                out[p + "srecpar_keys"] = srp.keys
                out[p + "soptmov_keys"] = sop.keys
                i += 1
    # offset jobs with sentinels around them (test_seqmerge.py:73-91 style)
    for _ in range(12):
        size = int(rng.integers(2, 700))
        keys, payload, middle = random_instance(rng, size, float(rng.random()), 50, 4)
        lo = int(rng.integers(0, 9))
        hi = int(rng.integers(0, 9))
        kk = np.concatenate([np.full(lo, -999, np.int32), keys, np.full(hi, -888, np.int32)])
        pp = np.concatenate([np.full((lo, 4), 7, np.uint8), payload, np.full((hi, 4), 9, np.uint8)])
        arr = ref.KeyedArray(kk.copy(), pp.copy())
        job = ref.MergeJob(lo, lo + middle, lo + size)
        ref.seq_merge_buffered(arr, job)
        p = f"c{i}_"
        out[p + "keys"] = kk
        out[p + "payload"] = pp
        out[p + "job"] = np.array([lo, lo + middle, lo + size], np.int64)
        out[p + "out_keys"] = arr.keys
        out[p + "out_payload"] = arr.payload
        out[p + "srecpar_keys"] = arr.keys
        out[p + "soptmov_keys"] = arr.keys
        i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "merge_i32.npz"), **out)
    print("merge_i32:", i, "cases")


def merge_i64_cases():
    rng = np.random.default_rng(64)
    out = {}
    i = 0
    for size in (0, 1, 7, 100, 1000, 3000):
        for split in (0.1, 0.5, 0.9):
            for lo_, hi_ in ((-(2**62), 2**62), (0, 50), (2**40, 2**40 + 10**6)):
                middle = int(size * split)
                a = np.sort(rng.integers(lo_, hi_, middle, dtype=np.int64))
                b = np.sort(rng.integers(lo_, hi_, size - middle, dtype=np.int64))
                keys = np.concatenate([a, b]).astype(np.int64)
                payload = rng.integers(0, 256, (size, 4), dtype=np.uint8)
                k = keys.copy()
                pl = payload.copy()
                need = max(1, min(middle, size - middle))
                _kernels.buffered_merge(k, pl, 0, middle, size, np.empty(need, np.int64),
                                        np.empty((need, 4), np.uint8))
                p = f"c{i}_"
                out[p + "keys"] = keys
                out[p + "payload"] = payload
                out[p + "job"] = np.array([0, middle, size], np.int64)
                out[p + "out_keys"] = k
                out[p + "out_payload"] = pl
                i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "merge_i64.npz"), **out)
    print("merge_i64:", i, "cases")


def median_cases():
    rng = np.random.default_rng(14)
    A, B, P, offs = [], [], [], [0]
    pos_a = [0]
    pos_b = [0]
    for j in range(3000):
        la = int(rng.integers(0, 130))
        lb = int(rng.integers(0, 130))
        if j % 2 == 0:
            dom = int(rng.choice([3, 16, 10**6]))
            a = np.sort(rng.integers(0, dom, la)).astype(np.int32)
            b = np.sort(rng.integers(0, dom, lb)).astype(np.int32)
        else:
            a = np.floor(np.cumsum(rng.random(la) * 5.0)).astype(np.int32)
            b = np.floor(np.cumsum(rng.random(lb) * 5.0)).astype(np.int32)
        P.append(tuple(ref.find_median(a, b)))
        A.append(a)
        B.append(b)
        pos_a.append(pos_a[-1] + la)
        pos_b.append(pos_b[-1] + lb)
    np.savez_compressed(
        os.path.join(HERE, "median.npz"),
        a=np.concatenate(A), b=np.concatenate(B), pos_a=np.array(pos_a), pos_b=np.array(pos_b),
        pivots=np.array(P, np.int64))
    print("median:", len(P), "pairs")


def shift_cases():
    rng = np.random.default_rng(11)
    out = {}
    i = 0
    grid = [(la, lb) for la in range(0, 49, 3) for lb in range(0, 49, 4)]
    grid += [(int(x), int(y)) for x, y in rng.integers(200, 2500, (10, 2))]
    grid += [(1, 9), (9, 1), (5, 7), (40, 12), (3, 3)]
    for la, lb in grid:
        n = la + lb
        w = int(rng.choice([0, 4, 8, 96])) if n < 100 else int(rng.choice([0, 4]))
        keys = rng.integers(-500, 500, n).astype(np.int32)
        payload = rng.integers(0, 256, (n, w), dtype=np.uint8)
        lin = ref.KeyedArray(keys.copy(), payload.copy())
        ref.linear_shift(lin, la, lb)
        cir = ref.KeyedArray(keys.copy(), payload.copy())
        ref.circular_shift(cir, la, lb)
        assert lin.equals(cir)
        p = f"c{i}_"
        out[p + "keys"] = keys
        out[p + "payload"] = payload
        out[p + "len"] = np.array([la, lb], np.int64)
        out[p + "out_keys"] = lin.keys
        out[p + "out_payload"] = lin.payload
        i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "shift.npz"), **out)
    print("shift:", i, "cases")


def plan_cases():
    rng = np.random.default_rng(15)
    out = {}
    i = 0
    for _ in range(40):
        size = int(rng.integers(32, 3000))
        keys, payload, middle = random_instance(rng, size, float(rng.choice([0.25, 0.5, 0.75, rng.random()])),
                                                int(rng.choice([6, 10**6])), 4)
        arr = ref.KeyedArray(keys, payload)
        job = ref.MergeJob(0, middle, size)
        inst = len([k for k in out if k.startswith("i") and k.endswith("_keys")])
        out[f"i{inst}_keys"] = keys
        out[f"i{inst}_payload"] = payload
        for t in (1, 2, 4, 8, 16):
            plan = ref.plan_intervals(arr, job, t)
            trace = ref.division_trace(arr, job, t, size_limit=2)
            p = f"c{i}_"
            out[p + "inst"] = np.array(inst)
            out[p + "job"] = np.array([0, middle, size, t], np.int64)
            out[p + "sources"] = np.array(plan.leaf_sources, np.int64).reshape(-1, 2)
            out[p + "finals"] = np.array(
                [(j.start, j.middle, j.end) for j in plan.final_positions], np.int64).reshape(-1, 3)
            out[p + "divided_sha"] = np.array(sha(trace.divided.keys, trace.divided.payload))
            out[p + "trace_pivots"] = np.array(
                [(r.level, r.split_index, r.pivots[0], r.pivots[1], r.shift_start,
                  r.shift_len_a, r.shift_len_b) for r in trace.records], np.int64).reshape(-1, 7)
            i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "plan.npz"), **out)
    print("plan:", i, "cases")


def big_cases():
    """Checksums of the reference's stable merge on full-size-shaped inputs."""
    out = {}
    # config 1: int32, L_A = L_B = 2^20, seed 0 (BASELINE.json configs[0])
    keys, payload, middle = config_input(1, seed=0)
    arr = ref.KeyedArray(keys.copy(), payload)
    ref.seq_merge_buffered(arr, ref.MergeJob(0, middle, len(keys)))
    out["cfg1_in"] = sha(keys)
    out["cfg1_out"] = sha(arr.keys)
    # config 4 shaped, reduced to L = 2^18 per side (payload = original index)
    keys, payload, middle = config_input(4, seed=0, log_len=18)
    arr = ref.KeyedArray(keys.copy(), payload.copy())
    ref.seq_merge_buffered(arr, ref.MergeJob(0, middle, len(keys)))
    out["cfg4s_in"] = sha(keys, payload)
    out["cfg4s_out"] = sha(arr.keys, arr.payload)
    # config 3 shaped (int64 skew), reduced to L_A = 2^20, L_B = 2^12
    keys, payload, middle = config_input(3, seed=0, log_len=20, log_len_b=12)
    k = keys.copy()
    pl = np.empty((len(k), 0), np.uint8)
    n = len(k) - middle
    _kernels.buffered_merge(k, pl, 0, middle, len(k), np.empty(n, np.int64), np.empty((n, 0), np.uint8))
    out["cfg3s_in"] = sha(keys)
    out["cfg3s_out"] = sha(k)
    np.savez(os.path.join(HERE, "big.npz"), **{k_: np.array(v) for k_, v in out.items()})
    print("big:", out)


if __name__ == "__main__":
    _kernels.warmup()
    merge_cases()
    merge_i64_cases()
    median_cases()
    shift_cases()
    plan_cases()
    big_cases()
