"""Randomised stress of every device merge path against the oracle (run for a time budget).

Usage: python tools/stress.py SECONDS [seed]
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from gen import random_instance
from oracle import oracle as orc

budget = float(sys.argv[1]); seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
t_end = time.time() + budget
n_jobs = 0
while time.time() < t_end:
    size = int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 400000), rng.integers(400000, 6_000_000)]))
    split = float(rng.random())
    domain = int(rng.choice([2, 50, 10**4, 2**31 - 1]))
    width = int(rng.choice([0, 0, 4, 8, 3, 12]))
    dtype = np.int64 if rng.random() < 0.3 else np.int32
    keys, payload, middle = random_instance(rng, size, split, domain, width)
    keys = keys.astype(dtype)
    lo, hi = int(rng.integers(0, 40)), int(rng.integers(0, 40))
    kk = np.concatenate([np.full(lo, -5, dtype), keys, np.full(hi, -7, dtype)])
    pp = np.concatenate([np.full((lo, width), 1, np.uint8), payload, np.full((hi, width), 2, np.uint8)])
    want_k, want_p = kk.copy(), pp.copy()
    orc.seq_merge_buffered(want_k, want_p, lo, lo + middle, lo + size)
    mode = int(rng.integers(0, 3))
    if mode == 0:  # in place, random pool
        scratch = int(rng.choice([0, size // 64, size // 4, min(middle, size - middle)]))
        arr = pm.KeyedArray(torch.from_numpy(kk).cuda(), torch.from_numpy(pp).cuda())
        _ops.merge(arr, lo, lo + middle, lo + size, scratch_records=scratch)
        gk, gp = arr.numpy()
    elif mode == 1:  # copy
        sk, sp = torch.from_numpy(kk[lo:lo + size].copy()).cuda(), torch.from_numpy(pp[lo:lo + size].copy()).cuda()
        dk, dp = torch.empty_like(sk), torch.empty_like(sp)
        _ops.merge_copy(sk, sp, dk, dp, middle)
        pm.synchronize()
        gk, gp = kk.copy(), pp.copy()
        gk[lo:lo + size], gp[lo:lo + size] = dk.cpu().numpy(), dp.cpu().numpy()
    else:  # host
        gk, gp = kk.copy(), pp.copy()
        _ops.merge_host(gk, gp, lo, lo + middle, lo + size)
    if not (np.array_equal(gk, want_k) and np.array_equal(gp, want_p)):
        print(f"MISMATCH mode={mode} size={size} split={split:.3f} domain={domain} w={width} dtype={dtype.__name__}")
        sys.exit(1)
    n_jobs += 1
print(f"stress ok: {n_jobs} jobs")
