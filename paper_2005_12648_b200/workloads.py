"""Seeded synthetic inputs for the BASELINE.json configs (no public dataset exists).

The reference's own harness draws random walks (``bench.py:110-146``); the
BASELINE configs instead use uniform sorted runs, so both are provided:

* ``config_input(cfg, seed, ...)``  -- numpy PCG64 ``default_rng(seed)``, A then B
  from one stream (SURVEY.md 8d recipe), host arrays.  Used for parity fixtures
  and CPU baselines at sizes numpy can sort quickly.
* ``config_input_device(cfg, seed, ...)`` -- the same distributions drawn with a
  seeded ``torch.Generator`` on the GPU and sorted there, for the full-size bench
  (2^29-2^30 records would take minutes to sort on the host).
* ``random_instance`` mirrors the reference test helper ``tests/support.py:17-29``.
* ``generate_input`` mirrors the reference's random-walk generator
  ``bench.py:110-146`` (value[0]=0, steps U[0,5) truncated to int32).
"""

from __future__ import annotations

import numpy as np

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1


def random_instance(rng, size, split, domain, payload_width=0):
    """Two adjacent sorted int32 runs plus random payload rows (support.py:21-29)."""
    middle = int(size * split)
    a = np.sort(rng.integers(0, domain, middle)).astype(np.int32)
    b = np.sort(rng.integers(0, domain, size - middle)).astype(np.int32)
    keys = np.concatenate([a, b]).astype(np.int32)
    payload = (rng.integers(0, 256, (size, payload_width), dtype=np.uint8)
               if payload_width else np.empty((size, 0), np.uint8))
    return keys, payload, middle


def generate_input(size: int, split: float, seed: int, elem_bytes: int = 4):
    """Random-walk runs as in the reference harness (bench.py:110-146)."""
    if size < 0:
        raise ValueError("size must be >= 0")
    rng = np.random.default_rng(seed)
    middle = min(int(size * split + 0.5), size)
    keys = np.empty(size, dtype=np.int32)
    for s, e in ((0, middle), (middle, size)):
        n = e - s
        if n:
            walk = np.empty(n, dtype=np.float64)
            walk[0] = 0.0
            if n > 1:
                np.cumsum(rng.random(n - 1) * 5.0, out=walk[1:])
            keys[s:e] = walk.astype(np.int32)
    pad = elem_bytes - 4
    if pad < 0:
        raise ValueError("elem_bytes must be >= 4")
    payload = rng.integers(0, 256, size=(size, pad), dtype=np.uint8) if pad else np.empty((size, 0), np.uint8)
    return keys, payload, middle


def config_input(cfg: int, seed: int = 0, log_len: int | None = None, log_len_b: int | None = None):
    """Host (numpy) input for BASELINE.json config ``cfg``; returns (keys, payload, middle).

    cfg 1/2: int32 uniform [0, 2^31), L_A = L_B = 2^log_len (default 20).
    cfg 3:   int64; A uniform over the full int64 range, L_A = 2^log_len (default 28);
             B uniform inside the window [A[c-L_B/2], A[c+L_B/2]], c = L_A/2,
             L_B = 2^log_len_b (default 16).
    cfg 4:   int32 keys in [0, 1024), L = 2^log_len (default 26) per side,
             payload = int32 original index (little-endian bytes, shape (N, 4)).
    """
    rng = np.random.default_rng(seed)
    if cfg in (1, 2):
        L = 1 << (20 if log_len is None else log_len)
        a = np.sort(rng.integers(0, 2**31, L, dtype=np.int32))
        b = np.sort(rng.integers(0, 2**31, L, dtype=np.int32))
        return np.concatenate([a, b]), np.empty((2 * L, 0), np.uint8), L
    if cfg == 3:
        la = 1 << (28 if log_len is None else log_len)
        lb = 1 << (16 if log_len_b is None else log_len_b)
        a = np.sort(rng.integers(INT64_MIN, INT64_MAX, la, dtype=np.int64, endpoint=True))
        c = la // 2
        lo = a[max(0, c - lb // 2)]
        hi = a[min(la - 1, c + lb // 2)]
        b = np.sort(rng.integers(lo, hi, lb, dtype=np.int64, endpoint=True))
        return np.concatenate([a, b]), np.empty((la + lb, 0), np.uint8), la
    if cfg == 4:
        L = 1 << (26 if log_len is None else log_len)
        a = np.sort(rng.integers(0, 1024, L, dtype=np.int32))
        b = np.sort(rng.integers(0, 1024, L, dtype=np.int32))
        idx = np.arange(2 * L, dtype=np.int32)
        return np.concatenate([a, b]), idx.view(np.uint8).reshape(2 * L, 4), L
    raise ValueError(f"unknown config {cfg}")


def config_input_device(cfg: int, seed: int = 0, log_len: int | None = None,
                        log_len_b: int | None = None, device="cuda"):
    """Device (torch) input with the same distributions as ``config_input``.

    Returns (keys, payload, middle) as CUDA tensors; payload is uint8 (N, w).
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if cfg in (1, 2):
        L = 1 << (20 if log_len is None else log_len)
        a = torch.randint(0, 2**31, (L,), generator=g, device=device, dtype=torch.int64)
        b = torch.randint(0, 2**31, (L,), generator=g, device=device, dtype=torch.int64)
        keys = torch.cat([a.sort().values, b.sort().values]).to(torch.int32)
        return keys, torch.empty((2 * L, 0), dtype=torch.uint8, device=device), L
    if cfg == 3:
        la = 1 << (28 if log_len is None else log_len)
        lb = 1 << (16 if log_len_b is None else log_len_b)
        # full-range int64: combine two 32-bit draws
        hi = torch.randint(-(2**31), 2**31, (la,), generator=g, device=device, dtype=torch.int64)
        lo = torch.randint(0, 2**32, (la,), generator=g, device=device, dtype=torch.int64)
        a = ((hi << 32) | lo).sort().values
        c = la // 2
        wlo = int(a[max(0, c - lb // 2)].item())
        whi = int(a[min(la - 1, c + lb // 2)].item())
        span = whi - wlo
        # uniform in [wlo, whi] via 62-bit draws modulo span+1 (span < 2^62 here)
        r = torch.randint(0, 2**62, (lb,), generator=g, device=device, dtype=torch.int64)
        b = (wlo + torch.remainder(r, span + 1)).sort().values
        return (torch.cat([a, b]), torch.empty((la + lb, 0), dtype=torch.uint8, device=device), la)
    if cfg == 4:
        L = 1 << (26 if log_len is None else log_len)
        a = torch.randint(0, 1024, (L,), generator=g, device=device, dtype=torch.int32).sort().values
        b = torch.randint(0, 1024, (L,), generator=g, device=device, dtype=torch.int32).sort().values
        idx = torch.arange(2 * L, dtype=torch.int32, device=device)
        return torch.cat([a, b]), idx.view(torch.uint8).reshape(2 * L, 4), L
    raise ValueError(f"unknown config {cfg}")


def sorted_uniform_device(n: int, seed: int, out=None, hi: int = 2**31, chunk: int = 1 << 27, buckets: int = 1024,
                          device="cuda"):
    """``sort(uniform int32 in [0, hi))`` of ``n`` draws on the device, for runs too
    large to sort in one piece (BASELINE config 5: 2^32 per run = 16 GiB).

    Exactly the sorted multiset of the seeded draws: pass 1 counts the draws per
    value bucket, pass 2 regenerates them chunk by chunk (same seed) and scatters
    each sorted chunk's bucket segments behind the bucket's cursor, pass 3 sorts
    each bucket in place.  Peak extra memory: a few chunks.
    """
    import torch

    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=device)
    shift = max(0, (hi - 1).bit_length() - (buckets - 1).bit_length())
    nb = ((hi - 1) >> shift) + 1
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    counts = torch.zeros(nb, dtype=torch.int64, device=device)
    for c0 in range(0, n, chunk):
        v = torch.randint(0, hi, (min(chunk, n - c0),), generator=g, device=device, dtype=torch.int64)
        counts += torch.bincount(v >> shift, minlength=nb)
        del v
    offs = torch.cumsum(counts, 0) - counts
    cursor = offs.tolist()
    edges = (torch.arange(nb, device=device, dtype=torch.int64) << shift).to(torch.int32)  # bucket starts
    g.manual_seed(seed)
    for c0 in range(0, n, chunk):
        v = torch.randint(0, hi, (min(chunk, n - c0),), generator=g, device=device, dtype=torch.int64)
        v = v.to(torch.int32).sort().values
        bnd = torch.searchsorted(v, edges).tolist() + [v.numel()]
        for b in range(nb):
            k = bnd[b + 1] - bnd[b]
            if k:
                out[cursor[b]:cursor[b] + k] = v[bnd[b]:bnd[b + 1]]
                cursor[b] += k
        del v
    for b, (o, c) in enumerate(zip(offs.tolist(), counts.tolist())):
        if c > 1:
            out[o:o + c] = out[o:o + c].sort().values
    return out
