"""Multi-rank host logic of the distributed merge (dist.py) on CPU with gloo, world_size 2 and 3.

The device engine is replaced by a numpy stable merge for the local step
(test-only); global split search and the two all-to-all exchanges are the
product code paths.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _np_local_merge(keys, payload, len_a):
    k = keys.numpy()
    order = np.argsort(k, kind="stable")  # A precedes B inside the buffer: stable == A wins ties
    keys.copy_(torch.from_numpy(k[order].copy()))
    if payload.shape[1]:
        payload.copy_(torch.from_numpy(payload.numpy()[order].copy()))


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_12648_b200.dist import merge_distributed

    keys, payload, la, bounds = case
    lo, hi = bounds[rank], bounds[rank + 1]
    k = torch.from_numpy(keys[lo:hi].copy())
    p = torch.from_numpy(payload[lo:hi].copy())
    rk, rp = merge_distributed(k, p, la, local_merge=_np_local_merge)
    out_q.put((rank, rk.numpy().copy(), rp.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _run(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict()
    for _ in range(world):
        r, k, p = q.get(timeout=120)
        res[r] = (k, p)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return np.concatenate([res[r][0] for r in range(world)]), np.concatenate([res[r][1] for r in range(world)])


@pytest.mark.parametrize("world,seed", [(2, 0), (2, 1), (3, 2)])
def test_distributed_merge_matches_stable_merge(world, seed):
    rng = np.random.default_rng(seed)
    la, lb = int(rng.integers(100, 3000)), int(rng.integers(100, 3000))
    dom = [4, 50, 10**6][seed % 3]
    a = np.sort(rng.integers(0, dom, la)).astype(np.int32)
    b = np.sort(rng.integers(0, dom, lb)).astype(np.int32)
    keys = np.concatenate([a, b])
    payload = np.arange(la + lb, dtype=np.int32).view(np.uint8).reshape(-1, 4).copy()
    n = la + lb
    cuts = sorted(int(x) for x in rng.integers(1, n, world - 1))
    bounds = [0] + cuts + [n]
    k, p = _run((keys, payload, la, bounds), world)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k, keys[order])
    assert np.array_equal(p, payload[order])
