"""Multi-GPU merge of a block-distributed A|B (BASELINE config 5).

Rank r holds the contiguous block X[off_r, off_r + n_r) of the concatenation
X = A|B (|A| = ``global_len_a``).  After ``merge_distributed`` rank r holds
the same block of the stable merge of A and B -- the distributed form of the
reference's parallel merge (srecpar.py:33-84: split, exchange, merge pairs),
with the GPUs as the partitions:

1. **Global split points** (the median search of the reference, made stable):
   for every rank boundary diagonal d = off_r, the number of A records among
   the first d outputs.  On CUDA with equal blocks the ranks map each other's
   blocks (CUDA IPC, cached) and one kernel launch runs every search over the
   peer-pointer table (pm_peer_splits, dependent NVLink loads).  Otherwise (gloo,
   CPU tensors, unequal blocks, PM_DIST_SPLITS=torch) all G+1 searches run
   together as a 33-ary search; each round all-reduces the 32 probe keys per
   diagonal that the owning ranks contribute (about log_33 N rounds).
2. **Partition exchange**: rank r needs A[a_r, a_{r+1}) and B[b_r, b_{r+1});
   every rank's A part and B part are already ordered by destination, so two
   ``all_to_all_single`` calls (NCCL send/recv over NVLink) deliver rank r's
   A slice followed by its B slice, contiguously.
3. **Local merge**: the received pair is merged out of place straight into the
   rank's block (``pm_merge_copy``: one read and one write per record).

The exchange uses a receive buffer of n_r records per rank (DESIGN.md notes
the chunked, O(chunk) variant as next work).  ``local_merge`` is injectable so
the host logic can be tested with the gloo backend on CPU tensors.
"""

from __future__ import annotations

from collections import OrderedDict
from typing import Callable

import torch
import torch.distributed as dist

_PROBES = 32


def _owned_values(keys_local: torch.Tensor, off: int, positions: torch.Tensor) -> torch.Tensor:
    """Values at global X positions owned by this rank, 0 elsewhere (for a SUM all-reduce)."""
    n = keys_local.numel()
    mine = (positions >= off) & (positions < off + n)
    idx = (positions - off).clamp(0, max(n - 1, 0))
    vals = keys_local[idx].to(torch.int64) if n else torch.zeros_like(positions)
    return torch.where(mine, vals, torch.zeros_like(vals))


def _split_search(keys_local: torch.Tensor, off: int, diags: torch.Tensor, la: int, lb: int, rounds: int,
                  group) -> tuple[torch.Tensor, torch.Tensor]:
    """The probe rounds of global_splits on device tensors; returns (lo, hi)."""
    dev = keys_local.device
    lo = torch.clamp(diags - lb, min=0)
    hi = torch.clamp(diags, max=la)
    k = torch.arange(1, _PROBES + 1, dtype=torch.int64, device=dev)
    for _ in range(rounds):
        span = hi - lo
        small = span <= _PROBES
        # probes: evenly spaced when the interval is wide, every index when it is small
        p_wide = lo[:, None] + (k[None, :] * span[:, None]) // (_PROBES + 1)
        p_small = lo[:, None] + (k[None, :] - 1)
        p = torch.where(small[:, None], p_small, p_wide)
        valid = p < hi[:, None]
        pa = torch.where(valid, p, lo[:, None])                      # A index
        pb = torch.clamp(diags[:, None] - 1 - pa, min=0)              # B index
        gpos = torch.stack([pa, la + pb], dim=-1)                    # global X positions
        vals = _owned_values(keys_local, off, gpos.reshape(-1)).reshape(gpos.shape)
        dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
        f = (vals[..., 0] <= vals[..., 1]) & valid                   # A[p] is among the first d
        # first probe with f false (or none)
        nf = (~f) & valid
        has = nf.any(dim=1)
        first = torch.where(has, nf.float().argmax(dim=1), torch.full_like(lo, _PROBES))
        last_true = torch.where(first > 0, p.gather(1, (first - 1).clamp(min=0)[:, None])[:, 0], lo - 1)
        new_hi = torch.where(has, p.gather(1, first.clamp(max=_PROBES - 1)[:, None])[:, 0], hi)
        # when no probe failed, everything up to the last valid probe is among the first d
        last_valid = torch.where(valid, p, lo[:, None] - 1).max(dim=1).values
        new_lo = torch.where(has, torch.where(first > 0, last_true + 1, lo), last_valid + 1)
        lo, hi = torch.where(span > 0, new_lo, lo), torch.where(span > 0, new_hi, hi)
    return lo, hi


# CUDA graphs of the probe rounds, per (keys buffer, geometry): ~30 small ops and a
# collective per round are replayed without host dispatch (NCCL supports capture).
# Bounded (least recently used first out); only with PM_DIST_GRAPHS=1 (opt-in).
_graphs: OrderedDict = OrderedDict()
_GRAPH_CAP = 8
_PEER_CAP = 64


def clear_caches() -> None:
    """Release the captured split-search graphs and the mapped peer blocks."""
    _graphs.clear()
    _PEER_TABLES.clear()
    _PEER_CACHE.clear()


def _peer_splits_enabled() -> bool:
    import os

    return os.environ.get("PM_DIST_SPLITS", "peer") != "torch"


def _graph_capture_enabled() -> bool:
    """CUDA-graph capture of the NCCL split-search rounds: opt-in (PM_DIST_GRAPHS=1).
    Capturing NCCL collectives has only run at one rank here; a capture that fails on
    one rank and not another would pair eager and graph collectives, so multi-rank
    jobs stay eager unless asked (the peer-table search needs no collectives at all)."""
    import os

    return os.environ.get("PM_DIST_GRAPHS", "0") == "1"


def global_splits(keys_local: torch.Tensor, offsets: list[int], global_len_a: int, group=None) -> list[int]:
    """A-count of the stable merge at every rank boundary diagonal (A wins ties)."""
    rank = dist.get_rank(group)
    off = offsets[rank]
    N = offsets[-1]
    la, lb = global_len_a, N - global_len_a
    dev = keys_local.device
    # each round cuts a span s to <= s // 33 + 1 and resolves spans <= 32 exactly, so
    # the round count is known up front: no host synchronisation inside the loop
    s = max(min(d, la) - max(d - lb, 0) for d in offsets)  # widest initial span (host side)
    rounds = 0 if s == 0 else 1
    while s > _PROBES:
        s = s // (_PROBES + 1) + 1
        rounds += 1
    if rounds == 0:
        return [min(max(d - lb, 0), la) for d in offsets]
    key = (keys_local.data_ptr(), keys_local.numel(), keys_local.dtype, off, tuple(offsets), la, rounds,
           id(group)) if (keys_local.is_cuda and dist.get_backend(group) == "nccl"
                          and _graph_capture_enabled()) else None
    ent = _graphs.get(key) if key else None
    if key is not None and ent is not None:
        _graphs.move_to_end(key)
    if ent is None:
        diags = torch.tensor(offsets, dtype=torch.int64, device=dev)
        lo, hi = _split_search(keys_local, off, diags, la, lb, rounds, group)
        if key is not None:
            try:  # capture for the next call with the same buffers and geometry
                g = torch.cuda.CUDAGraph()
                sd = diags.clone()
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(g):
                    slo, shi = _split_search(keys_local, off, sd, la, lb, rounds, group)
                _graphs[key] = (g, slo, shi)
            except Exception:  # (capture unsupported here: stay eager; the partial graph is dropped)
                torch.cuda.synchronize(dev)
                _graphs[key] = False
            while len(_graphs) > _GRAPH_CAP:
                _graphs.popitem(last=False)
    elif ent is False:
        diags = torch.tensor(offsets, dtype=torch.int64, device=dev)
        lo, hi = _split_search(keys_local, off, diags, la, lb, rounds, group)
    else:
        g, lo, hi = ent
        g.replay()
    res = torch.cat([lo, hi - lo]).tolist()
    assert not any(res[len(offsets):]), "global_splits: search did not converge"
    return [int(x) for x in res[:len(offsets)]]


def _default_local_merge(src_k: torch.Tensor, src_p: torch.Tensor, len_a: int, dst_k: torch.Tensor,
                         dst_p: torch.Tensor) -> None:
    """The received A|B pair merged straight into the rank's block (pm_merge_copy)."""
    from . import _ops

    _ops.merge_copy(src_k, src_p, dst_k, dst_p, len_a)


def merge_distributed(keys_local: torch.Tensor, payload_local: torch.Tensor | None, global_len_a: int,
                      group=None, local_merge: Callable | None = None, phases: dict | None = None):
    """Stable merge of the block-distributed A|B; returns this rank's output block.

    ``keys_local`` / ``payload_local`` are this rank's block (device tensors for
    NCCL).  Returns (keys, payload) of the same length, holding the merged
    records for this rank's block; the input tensors are overwritten too.
    ``phases`` (optional dict, CUDA tensors only) receives CUDA events around the
    split search, the exchange and the local merge, and the bytes this rank
    received from other ranks.
    """
    timed = phases is not None and keys_local.is_cuda
    if timed:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        evs[0].record()
    nvtx = keys_local.is_cuda
    if nvtx:  # NVTX phase ranges: split search / exchange / local merge
        torch.cuda.nvtx.range_push("dist: global splits")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = keys_local.device
    n = keys_local.numel()
    if payload_local is None:
        payload_local = torch.empty((n, 0), dtype=torch.uint8, device=dev)
    sizes = torch.tensor([n], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    offsets = [0]
    for t in all_sizes:
        offsets.append(offsets[-1] + int(t.item()))
    la = global_len_a
    peers = None
    if keys_local.is_cuda and world > 1 and _peer_splits_enabled() and len(set(offsets[i + 1] - offsets[i]
                                                                                for i in range(world))) == 1:
        try:  # the split search reads the peers' blocks directly (same box: CUDA IPC + NVLink)
            peers = peer_blocks(keys_local, None, group)
            if peers and not _all_peers_reachable(peers[0], keys_local.device):
                peers = None
        except RuntimeError:
            peers = None
    a = global_splits_p2p(peers[0], offsets, la) if peers else global_splits(keys_local, offsets, la, group)
    b = [offsets[i] - a[i] for i in range(world + 1)]
    off = offsets[rank]
    # this block's A part [off, min(off+n, la)) and B part [max(off, la), off+n) in X coordinates
    a_lo, a_hi = off, min(off + n, la)
    b_lo, b_hi = max(off, la), off + n
    send_a = [max(0, min(a_hi, a[r + 1]) - max(a_lo, a[r])) for r in range(world)]
    send_b = [max(0, min(b_hi, la + b[r + 1]) - max(b_lo, la + b[r])) for r in range(world)]
    # what every rank sends to me
    sa = torch.tensor(send_a, dtype=torch.int64, device=dev)
    sb = torch.tensor(send_b, dtype=torch.int64, device=dev)
    ra = torch.empty_like(sa)
    rb = torch.empty_like(sb)
    dist.all_to_all_single(ra, sa, group=group)
    dist.all_to_all_single(rb, sb, group=group)
    recv_a, recv_b = ra.tolist(), rb.tolist()
    na, nb = sum(recv_a), sum(recv_b)
    assert na == a[rank + 1] - a[rank] and nb == b[rank + 1] - b[rank] and na + nb == n
    split_at = max(0, min(n, la - off))
    out_k = torch.empty_like(keys_local)
    out_p = torch.empty_like(payload_local)
    if nvtx:
        torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push("dist: exchange (NCCL all-to-all)")
    if timed:
        evs[1].record()
        rec = keys_local.element_size() + payload_local.shape[1]
        phases["bytes_in_remote"] = sum(recv_a[r] + recv_b[r] for r in range(world) if r != rank) * rec
    dist.all_to_all_single(out_k[:na], keys_local[:split_at].contiguous(), recv_a, send_a, group=group)
    dist.all_to_all_single(out_k[na:], keys_local[split_at:].contiguous(), recv_b, send_b, group=group)
    if payload_local.shape[1]:
        dist.all_to_all_single(out_p[:na], payload_local[:split_at].contiguous(), recv_a, send_a, group=group)
        dist.all_to_all_single(out_p[na:], payload_local[split_at:].contiguous(), recv_b, send_b, group=group)
    if timed:
        evs[2].record()
    if nvtx:
        torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push("dist: local merge")
    if local_merge is None:
        _default_local_merge(out_k, out_p, na, keys_local, payload_local)
        if timed:
            evs[3].record()
            phases["events"] = evs
    else:  # (host-logic tests: any in-place merge of the received pair)
        local_merge(out_k, out_p, na)
        keys_local.copy_(out_k)
        payload_local.copy_(out_p)
    if nvtx:
        torch.cuda.nvtx.range_pop()
    return keys_local, payload_local


# ---------------------------------------------------------------------------------------------
# Exchange fused with the merge: every rank maps the others' blocks (CUDA IPC, NVLink peer
# access) and pm_merge_peers streams its A and B pieces straight out of peer memory into a
# staging block -- no all-to-all pass, no send/receive copies.
_PEER_CACHE: OrderedDict = OrderedDict()
_PEER_TABLES: dict = {}  # group -> (this rank's buffer key, the mapped table)


def _peer_view(meta, numel: int, dtype, shape_tail, elem_off: int) -> torch.Tensor:
    """A tensor over a peer's block (torch's CUDA IPC storage sharing), cached per handle."""
    key = (bytes(meta[1]), int(meta[3]))
    st = _PEER_CACHE.get(key)
    if st is None:
        st = torch.UntypedStorage._new_shared_cuda(*meta)
        _PEER_CACHE[key] = st
        while len(_PEER_CACHE) > _PEER_CAP:  # unmap the least recently used peer block
            _PEER_CACHE.popitem(last=False)
    else:
        _PEER_CACHE.move_to_end(key)
    t = torch.empty(0, dtype=dtype, device=st.device)
    t.set_(st, elem_off, (numel, *shape_tail))
    return t


def peer_blocks(keys_local: torch.Tensor, payload_local: torch.Tensor | None, group=None):
    """Every rank's block mapped into this process (CUDA IPC storage sharing, cached):
    ([keys blocks], [payload blocks]) in rank order; None unless all blocks are CUDA
    tensors of equal length."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = keys_local.numel()
    w = payload_local.shape[1] if payload_local is not None else 0
    # the table is exchanged once per set of buffers: later calls only agree (one tiny
    # all-reduce) that no rank's buffers changed
    my_key = (keys_local.data_ptr(), n, payload_local.data_ptr() if w else 0, w)
    cached = _PEER_TABLES.get(id(group))
    changed = torch.tensor([0 if cached is not None and cached[0] == my_key else 1], device=keys_local.device)
    dist.all_reduce(changed, op=dist.ReduceOp.MAX, group=group)
    if not int(changed.item()):
        return cached[1]
    sizes = [None] * world
    mine = (n, keys_local.untyped_storage()._share_cuda_(), keys_local.storage_offset(),
            payload_local.untyped_storage()._share_cuda_() if w else None, payload_local.storage_offset() if w else 0)
    dist.all_gather_object(sizes, mine, group=group)
    if any(s[0] != n for s in sizes):
        _PEER_TABLES.pop(id(group), None)
        return None
    pk, pp = [], []
    for r, (_, mk, ok, mp, op) in enumerate(sizes):
        if r == rank:
            pk.append(keys_local)
            pp.append(payload_local)
        else:
            pk.append(_peer_view(mk, n, keys_local.dtype, (), ok))
            pp.append(_peer_view(mp, n, torch.uint8, (w,), op) if w else payload_local)
    _PEER_TABLES[id(group)] = (my_key, (pk, pp))
    return pk, pp


def _all_peers_reachable(peer_keys: list, device) -> bool:
    """Every mapped block lives on this device or on one it can read directly (P2P)."""
    here = device.index
    return all(t.device.index == here or torch.cuda.can_device_access_peer(here, t.device.index) for t in peer_keys)


def global_splits_p2p(peer_keys: list, offsets: list[int], global_len_a: int) -> list[int]:
    """global_splits through the peer-pointer table: one kernel launch of one-thread
    stable merge-path searches reading the peers' blocks (pm_peer_splits), instead of
    the probe rounds with an all-reduce each."""
    from . import _ops

    return _ops.peer_splits(peer_keys, global_len_a, offsets)


def merge_distributed_p2p(keys_local: torch.Tensor, payload_local: torch.Tensor | None, global_len_a: int,
                          group=None):
    """merge_distributed with the exchange fused into the merge (pm_merge_peers).

    Every rank holds an equal-length block.  Blocks are shared once through CUDA IPC
    (``all_gather_object`` of the storage handles); each rank's merge reads its pieces
    from the peers' blocks over NVLink into a staging block, all ranks meet at a
    barrier (no block changes while a peer may still read it), and the staging block
    is copied into the rank's own block.
    """
    from . import _ops

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = keys_local.numel()
    if payload_local is None:
        payload_local = torch.empty((n, 0), dtype=torch.uint8, device=keys_local.device)
    w = payload_local.shape[1]
    if world == 1:  # nothing to map: the table is this block
        out_k = torch.empty_like(keys_local)
        out_p = torch.empty_like(payload_local)
        _ops.merge_peers([keys_local], [payload_local] if w else None, global_len_a, 0, out_k, out_p if w else None)
        keys_local.copy_(out_k)
        if w:
            payload_local.copy_(out_p)
        return keys_local, payload_local
    # the peer table is exchanged once per set of buffers (peer_blocks caches it;
    # later calls agree through one tiny all-reduce that no rank's buffers changed)
    table = peer_blocks(keys_local, payload_local if w else None, group=group)
    if table is None:
        raise ValueError("merge_distributed_p2p needs equal blocks on every rank")
    pk, pp = table
    out_k = torch.empty_like(keys_local)
    out_p = torch.empty_like(payload_local)
    _ops.merge_peers(pk, pp if w else None, global_len_a, rank, out_k, out_p if w else None)
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)  # every peer has finished reading this block
    keys_local.copy_(out_k)
    if w:
        payload_local.copy_(out_p)
    return keys_local, payload_local
