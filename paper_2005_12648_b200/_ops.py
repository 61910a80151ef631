"""Device operations: thin typed wrappers over the C-ABI (one call = one C-ABI entry).

All functions take GPU-resident tensors and enqueue work on the current torch
CUDA stream.  By default every mutating call then synchronises and checks the
device status word (``pm_status``) so errors surface at the call site, like the
reference's synchronous numba calls; ``deferred_checks()`` turns that off for
pipelines that check once at the end (the benchmark).
"""

from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _capi
from .records import KeyedArray, require_cuda

_check_each_call = True


@contextlib.contextmanager
def deferred_checks():
    """Skip the per-call synchronise+status check inside the block; check on exit."""
    global _check_each_call
    old = _check_each_call
    _check_each_call = False
    try:
        yield
    finally:
        _check_each_call = old
        synchronize()


def synchronize(device: int | None = None) -> tuple[int, int, int, int]:
    """Wait for the current stream and raise if any engine call failed; returns last-job stats."""
    dev = torch.cuda.current_device() if device is None else device
    return _capi.status(dev, torch.cuda.current_stream(dev).cuda_stream)


def _stream(dev: int) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr() if t.numel() else 0)


def merge(arr: KeyedArray, start: int, middle: int, end: int, scratch_records: int = 0):
    """Stable in-place merge of [start, middle) and [middle, end) on the device (pm_merge)."""
    require_cuda(arr)
    if start == middle or middle == end:
        return None
    dev = arr.keys.device.index
    rc = _capi.lib().pm_merge(_capi.context(dev), _ptr(arr.keys), arr.key_bytes, _ptr(arr.payload),
                              arr.payload.shape[1], start, middle, end, scratch_records, _stream(dev))
    _capi.check(rc, "pm_merge")
    if _check_each_call:
        return _capi.status(dev, torch.cuda.current_stream(dev).cuda_stream)
    return None


def merge_copy(src_keys: torch.Tensor, src_payload: torch.Tensor, dst_keys: torch.Tensor, dst_payload: torch.Tensor,
               len_a: int):
    """Out-of-place stable merge (pm_merge_copy): src = A|B with |A| = len_a -> dst.

    Device tensors: keys int32/int64 [n], payload uint8 [n, w] (w may be 0).
    """
    for t in (src_keys, src_payload, dst_keys, dst_payload):
        if not t.is_cuda:
            raise _capi.MergeEngineError("merge_copy needs CUDA tensors (no CPU fallback)")
    n = src_keys.numel()
    if dst_keys.numel() != n or src_keys.dtype != dst_keys.dtype or src_payload.shape != dst_payload.shape:
        raise ValueError("source and destination must have the same shape and dtype")
    if not 0 <= len_a <= n:
        raise ValueError("need 0 <= len_a <= len(src)")
    if n == 0:
        return None
    dev = src_keys.device.index
    w = src_payload.shape[1] if src_payload.dim() == 2 else 0
    rc = _capi.lib().pm_merge_copy(_capi.context(dev), _ptr(src_keys), _ptr(src_payload), _ptr(dst_keys),
                                   _ptr(dst_payload), src_keys.element_size(), w, len_a, n - len_a, _stream(dev))
    _capi.check(rc, "pm_merge_copy")
    if _check_each_call:
        return _capi.status(dev, torch.cuda.current_stream(dev).cuda_stream)
    return None


def merge_host(keys, payload, start: int, middle: int, end: int, device: int = 0):
    """In-place stable merge of host (numpy) arrays through pm_merge_host.

    keys: int32/int64 [n] C-contiguous; payload: uint8 [n, w] C-contiguous.  The
    transfer, the device merge and the write-back are pipelined per output chunk
    (pinned host memory overlaps both PCIe directions; pageable memory works too).
    """
    import numpy as np

    if keys.dtype not in (np.int32, np.int64) or not keys.flags.c_contiguous:
        raise ValueError("keys must be a C-contiguous int32/int64 array")
    if payload.ndim != 2 or payload.dtype != np.uint8 or not payload.flags.c_contiguous or len(payload) != len(keys):
        raise ValueError("payload must be a C-contiguous uint8 array of shape (len(keys), w)")
    w = payload.shape[1]
    rc = _capi.lib().pm_merge_host(_capi.context(device), ctypes.c_void_p(keys.ctypes.data), keys.itemsize,
                                   ctypes.c_void_p(payload.ctypes.data if w else 0), w, start, middle, end,
                                   ctypes.c_void_p(0))
    _capi.check(rc, "pm_merge_host")


def shift(arr: KeyedArray, lo: int, len_a: int, len_b: int):
    """In-place block exchange A|B -> B|A on the device (pm_shift).

    The span must lie inside the array: pm_shift is not given the array length, and a
    span past its end would write into neighbouring device allocations."""
    require_cuda(arr)
    if lo < 0 or len_a < 0 or len_b < 0 or lo + len_a + len_b > len(arr):
        raise IndexError(f"shift span [{lo}, {lo + len_a + len_b}) outside the array (length {len(arr)})")
    if len_a == 0 or len_b == 0:
        return None
    dev = arr.keys.device.index
    rc = _capi.lib().pm_shift(_capi.context(dev), _ptr(arr.keys), arr.key_bytes, _ptr(arr.payload),
                              arr.payload.shape[1], lo, len_a, len_b, _stream(dev))
    _capi.check(rc, "pm_shift")
    if _check_each_call:
        return _capi.status(dev, torch.cuda.current_stream(dev).cuda_stream)
    return None


def reorder(arr: KeyedArray, start: int, end: int, leaf_sizes: list[int]):
    """In-place permutation of [start, end) into the leaf layout A_0 B_0 A_1 B_1 ...
    (pm_reorder; ``leaf_sizes`` = [|A_0|, |B_0|, |A_1|, |B_1|, ...])."""
    require_cuda(arr)
    if len(leaf_sizes) % 2 or not leaf_sizes:
        raise ValueError("leaf_sizes must hold |A_i|, |B_i| pairs")
    dev = arr.keys.device.index
    tab = (ctypes.c_int64 * len(leaf_sizes))(*[int(x) for x in leaf_sizes])
    rc = _capi.lib().pm_reorder(_capi.context(dev), _ptr(arr.keys), arr.key_bytes, _ptr(arr.payload),
                                arr.payload.shape[1], start, end, tab, len(leaf_sizes) // 2, _stream(dev))
    _capi.check(rc, "pm_reorder")
    if _check_each_call:
        return _capi.status(dev, torch.cuda.current_stream(dev).cuda_stream)
    return None


def _run_tensor(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor) and x.is_cuda:
        t = x
        if t.dtype not in (torch.int32, torch.int64):
            raise TypeError(f"keys must be int32 or int64, got {t.dtype}")
        return t.contiguous()
    import numpy as np

    a = np.asarray(x)
    if a.dtype.kind not in "iu" and a.size:
        raise TypeError("GPU find_median needs integer keys (use key= only with the CPU reference)")
    a = np.ascontiguousarray(a, dtype=np.int64 if a.dtype.itemsize == 8 else np.int32) if a.size else a.astype(np.int32)
    return torch.from_numpy(a).cuda()


def find_median(a, b) -> tuple[int, int]:
    """Alg. 1 pivot pair computed on the device (pm_find_median); returns host ints."""
    ta, tb = _run_tensor(a), _run_tensor(b)
    if ta.dtype != tb.dtype:
        wide = torch.int64
        ta, tb = ta.to(wide), tb.to(wide)
    dev = ta.device.index
    out = torch.empty(2, dtype=torch.int64, device=ta.device)
    rc = _capi.lib().pm_find_median(_capi.context(dev), _ptr(ta), _ptr(tb), ta.element_size(), ta.numel(),
                                    tb.numel(), _ptr(out), _stream(dev))
    _capi.check(rc, "pm_find_median")
    pa, pb = out.tolist()
    return int(pa), int(pb)


def find_splits(a: torch.Tensor, b: torch.Tensor, diags: torch.Tensor) -> torch.Tensor:
    """Stable merge-path A-counts at the given diagonals (pm_find_splits), on the device."""
    ta, tb = _run_tensor(a), _run_tensor(b)
    if ta.dtype != tb.dtype:
        ta, tb = ta.to(torch.int64), tb.to(torch.int64)
    d = diags.to(device=ta.device, dtype=torch.int64).contiguous()
    out = torch.empty_like(d)
    dev = ta.device.index
    rc = _capi.lib().pm_find_splits(_capi.context(dev), _ptr(ta), _ptr(tb), ta.element_size(), ta.numel(),
                                    tb.numel(), _ptr(d), d.numel(), _ptr(out), _stream(dev))
    _capi.check(rc, "pm_find_splits")
    return out


def plan_nodes(arr: KeyedArray, start: int, middle: int, end: int, threads: int) -> list[tuple[int, int, int, int]]:
    """Level-order RunPairs of plan_intervals computed on the device (pm_plan_intervals)."""
    require_cuda(arr)
    dev = arr.keys.device.index
    n_nodes = 2 * threads - 1
    out = torch.empty(4 * n_nodes, dtype=torch.int64, device=arr.keys.device)
    rc = _capi.lib().pm_plan_intervals(_capi.context(dev), _ptr(arr.keys), arr.key_bytes, start, middle, end,
                                       threads, _ptr(out), _stream(dev))
    _capi.check(rc, "pm_plan_intervals")
    v = out.view(-1, 4).tolist()
    return [tuple(int(x) for x in r) for r in v]


def permute_rows(payload: torch.Tensor, idx: torch.Tensor, cut_every: int):
    """Debug: the wide-record path's in-place row permutation, payload[p] <- old payload[idx[p]]
    (pm_debug_permute_rows).  payload: CUDA uint8 [n, w]; idx: CUDA int32 [n], a permutation."""
    if not (payload.is_cuda and idx.is_cuda) or idx.dtype != torch.int32 or not payload.is_contiguous():
        raise ValueError("permute_rows needs contiguous CUDA tensors (uint8 rows, int32 indices)")
    dev = payload.device.index
    rc = _capi.lib().pm_debug_permute_rows(_capi.context(dev), _ptr(payload), payload.shape[1], _ptr(idx),
                                           payload.shape[0], cut_every, _stream(dev))
    _capi.check(rc, "pm_debug_permute_rows")


def set_engine_only(on: bool, device: int | None = None):
    """Debug: route in-place merges through the bounded-scratch engine even for small
    jobs (pm_debug_engine_only); tests use it to cover the engine at small sizes."""
    dev = torch.cuda.current_device() if device is None else device
    _capi.check(_capi.lib().pm_debug_engine_only(_capi.context(dev), int(bool(on))), "pm_debug_engine_only")


FLOW_MODES = {"bounded": 0, "auto": 1, "two_front": 2, "angle": 3, "fallback": 4}


def set_flow_mode(mode: str, device: int | None = None):
    """Debug/benchmark: which in-place engine pm_merge uses (pm_debug_flow).

    "auto" (default): the scheduled engine, order chosen per job, with the device-side
    fallback to the bounded-pool engine; "bounded": the bounded-pool engine only;
    "two_front" / "angle": the scheduled engine with that order forced; "fallback":
    plan, then force the fallback."""
    dev = torch.cuda.current_device() if device is None else device
    _capi.check(_capi.lib().pm_debug_flow(_capi.context(dev), FLOW_MODES[mode]), "pm_debug_flow")


def merge_peers(peer_keys: list, peer_payload: list | None, len_a: int, rank: int, out_keys: torch.Tensor,
                out_payload: torch.Tensor | None = None, ptrs: tuple[list[int], list[int]] | None = None):
    """pm_merge_peers: rank ``rank``'s block of the stable merge of the block-distributed
    A|B (blocks ``peer_keys[k]`` of equal length, A = the first ``len_a`` global records).

    ``ptrs`` optionally gives the (keys, payload) device addresses of the blocks directly
    (mapped peer memory from pm_ipc_open); otherwise the tensors' own addresses are used.
    """
    world = len(peer_keys)
    block = out_keys.numel()
    w = out_payload.shape[1] if out_payload is not None else 0
    kp = ptrs[0] if ptrs else [t.data_ptr() for t in peer_keys]
    pp = ptrs[1] if ptrs else ([t.data_ptr() for t in peer_payload] if w else [0] * world)
    tk = (ctypes.c_void_p * world)(*kp)
    tp = (ctypes.c_void_p * world)(*pp)
    dev = out_keys.device.index
    rc = _capi.lib().pm_merge_peers(_capi.context(dev), tk, tp if w else None, world, rank, block, len_a,
                                    out_keys.element_size(), w, _ptr(out_keys), _ptr(out_payload) if w else None,
                                    _stream(dev))
    _capi.check(rc, "pm_merge_peers")


def peer_splits(peer_keys: list, len_a: int, diags: list[int]) -> list[int]:
    """pm_peer_splits: the stable split (A records among the first d outputs) of every
    diagonal d of the block-distributed A|B, read through the peer-pointer table
    (blocks ``peer_keys[k]`` of equal length; one launch, dependent peer loads)."""
    world = len(peer_keys)
    block = peer_keys[0].numel()
    tk = (ctypes.c_void_p * world)(*[t.data_ptr() for t in peer_keys])
    dq = (ctypes.c_int64 * len(diags))(*[int(d) for d in diags])
    out = (ctypes.c_int64 * len(diags))()
    dev = peer_keys[0].device.index
    rc = _capi.lib().pm_peer_splits(_capi.context(dev), tk, world, block, len_a, peer_keys[0].element_size(),
                                    dq, len(diags), out, _stream(dev))
    _capi.check(rc, "pm_peer_splits")
    return [int(x) for x in out]


def ipc_handle(t: torch.Tensor) -> bytes:
    """64-byte CUDA IPC handle of the allocation holding ``t`` (pm_ipc_handle) and t's offset in it."""
    base = t.untyped_storage().data_ptr()
    h = ctypes.create_string_buffer(64)
    _capi.check(_capi.lib().pm_ipc_handle(ctypes.c_void_p(base), h), "pm_ipc_handle")
    return h.raw


def ipc_open(handle: bytes) -> int:
    """Map a peer's allocation (pm_ipc_open); returns the device address in this process."""
    p = ctypes.c_void_p()
    _capi.check(_capi.lib().pm_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)), "pm_ipc_open")
    return int(p.value)


def ipc_close(addr: int):
    _capi.check(_capi.lib().pm_ipc_close(ctypes.c_void_p(addr)), "pm_ipc_close")
