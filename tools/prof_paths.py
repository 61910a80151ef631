"""Small driver for ncu captures of the non-engine kernels: copy-mode merge, min-side
buffered merge, slide and reversal shifts, wide-row gather and cycle walk, small
and cluster merges (one call each at a representative size)."""
import sys

import torch

sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device

k0, p0, m = config_input_device(2, seed=5, log_len=28)
n = k0.numel()
dk, dp = torch.empty_like(k0), torch.empty_like(p0)
with pm.deferred_checks():
    _ops.merge_copy(k0, p0, dk, dp, m)                                   # k_buffered (copy)
    a = pm.KeyedArray(k0.clone(), p0.clone())
    _ops.merge(a, 0, m, n, scratch_records=min(m, n - m))                 # k_copy_run + k_buffered
    a.keys.copy_(k0)
    _ops.shift(a, 0, n // 100, n - n // 100)                              # k_slide
    a.keys.copy_(k0)
    _ops.shift(a, 0, n // 2, n - n // 2)                                  # k_reverse_vec
    w = 508
    nw = (1 << 30) // (4 + w)
    kw = torch.randint(0, 2**31 - 1, (nw,), device="cuda", dtype=torch.int32)
    kw[: nw // 2] = kw[: nw // 2].sort().values
    kw[nw // 2:] = kw[nw // 2:].sort().values
    pw = torch.randint(0, 256, (nw, w), device="cuda", dtype=torch.uint8)
    _ops.merge_copy(kw, pw, torch.empty_like(kw), torch.empty_like(pw), nw // 2)   # k_gather_rows
    aw = pm.KeyedArray(kw.clone(), pw.clone())
    _ops.set_engine_only(True)                                            # in-place cycle walk (no staging)
    _ops.merge(aw, 0, nw // 2, nw)
    _ops.set_engine_only(False)
    ks, ps_, ms = config_input_device(2, seed=6, log_len=13)
    s = pm.KeyedArray(ks.clone(), ps_.clone())
    _ops.merge(s, 0, ms, ks.numel())                                      # k_merge_small
    kc, pc, mc = config_input_device(2, seed=7, log_len=16)
    c = pm.KeyedArray(kc.clone(), pc.clone())
    _ops.merge(c, 0, mc, kc.numel())                                      # k_merge_cluster
print("ok")
