"""Multi-process, one GPU: the peer-pointer-table paths of dist.py with real CUDA IPC.

World 2 and 3 processes on cuda:0 (gloo for the control plane: handle exchange and
barriers).  Each rank maps the others' blocks through CUDA IPC (torch storage
sharing) and (1) searches the global stable splits over the table (pm_peer_splits),
(2) merges its output block reading the peers' blocks directly (pm_merge_peers).
No kernel waits on another rank (the only cross-rank ordering is the host barrier
after each rank has read), so running the ranks on one GPU is faithful.  Checked
against the pinned CPU oracle on the gathered blocks."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _instance(world, n, seed):
    rng = np.random.default_rng(seed)
    N = world * n
    la = int(rng.integers(N // 4, 3 * N // 4))
    a = np.sort(rng.integers(0, 5000, la)).astype(np.int32)
    b = np.sort(rng.integers(0, 5000, N - la)).astype(np.int32)
    return np.concatenate([a, b]), la


def _worker(rank, world, port, n, seed, outdir):
    import torch.distributed as dist

    import paper_2005_12648_b200  # noqa: F401
    from paper_2005_12648_b200 import dist as pdist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    x, la = _instance(world, n, seed)
    idx = np.arange(world * n, dtype=np.int32).view(np.uint8).reshape(-1, 4)
    keys = torch.from_numpy(x[rank * n:(rank + 1) * n].copy()).cuda()
    pay = torch.from_numpy(idx[rank * n:(rank + 1) * n].copy()).cuda()
    peers = pdist.peer_blocks(keys, pay, None)
    offsets = [r * n for r in range(world + 1)]
    splits = pdist.global_splits_p2p(peers[0], offsets, la)
    np.save(os.path.join(outdir, f"splits{rank}.npy"), np.array(splits, np.int64))
    dist.barrier()
    k, p = pdist.merge_distributed_p2p(keys, pay, la)
    np.save(os.path.join(outdir, f"k{rank}.npy"), k.cpu().numpy())
    np.save(os.path.join(outdir, f"p{rank}.npy"), p.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_paths_multiprocess_ipc(world, tmp_path):
    import torch.multiprocessing as mp

    from oracle import oracle as orc

    n, seed = 300001, 7 + world
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_worker, args=(world, port, n, seed, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x, la = _instance(world, n, seed)
    idx = np.arange(world * n, dtype=np.int32).view(np.uint8).reshape(-1, 4)
    want_k, want_p = x.copy(), idx.copy()
    orc.seq_merge_buffered(want_k, want_p, 0, la, len(x))
    a_ref = [orc.merge_path(x[:la], x[la:], r * n) for r in range(world + 1)]
    for r in range(world):
        assert np.load(tmp_path / f"splits{r}.npy").tolist() == a_ref
    got_k = np.concatenate([np.load(tmp_path / f"k{r}.npy") for r in range(world)])
    got_p = np.concatenate([np.load(tmp_path / f"p{r}.npy") for r in range(world)])
    assert np.array_equal(got_k, want_k) and np.array_equal(got_p, want_p)
