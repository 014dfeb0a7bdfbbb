"""Late swapping for large elements on the GPU path.

Mirrors the reference's bigelem module
(/root/reference/pkg/src/tsqsort/bigelem.py): sort position handles first,
then move every element once.  The handle sort is the device's (key, uint32
index) records sort -- the handles are the payload -- and the move is one
coalesced gather pass on the device (``tsq_apply_permutation``,
csrc/tsq_gather.cuh) instead of ``_apply``'s cycle walk
(bigelem.py:48-76).  ``apply_permutation`` still reports the reference's
move count -- each nontrivial cycle of length c costs c + 1 moves
(bigelem.py:79-86) -- computed from the cycle structure of the permutation,
so callers see the same numbers.

Large elements on the device are rows: ``Records(keys, rows)`` with ``rows``
a tensor whose first dimension is n (any dtype, any row width).  Host
sequences of Python objects (tuples with ``cmp=key_cmp``, numbers) sort their
keys on the device and are rearranged on the host, as the list write-back of
every host container is.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .stats import SortStats

__all__ = ["Permutation", "sort_indirect", "apply_permutation", "sort_large_elements"]


@dataclass(frozen=True)
class Permutation:
    """map[i] = origin position of the element that must end up at i
    (bigelem.py:18-28)."""

    map: tuple

    def __len__(self):
        return len(self.map)

    def is_identity(self) -> bool:
        return all(v == i for i, v in enumerate(self.map))


def _torch():
    import torch
    return torch


def _keys_of(ar, cmp):
    """Device-sortable keys of a container of elements (1-D tensor / array)."""
    torch = _torch()
    from .core import Records, _list_to_numpy, key_cmp
    if isinstance(ar, Records):
        return ar.keys
    if cmp is not None and cmp is not key_cmp:
        raise TypeError("custom comparators cannot run on the GPU path; pass cmp=None "
                        "(native order) or cmp=key_cmp for (key, ...) elements")
    if isinstance(ar, (np.ndarray, torch.Tensor)):
        if ar.ndim != 1:
            raise ValueError("late swapping of rows needs Records(keys, rows)")
        return ar
    values = list(ar)
    if cmp is key_cmp:
        return _list_to_numpy([v[0] for v in values])
    return _list_to_numpy(values)


def _handle_sort(keys, sorter):
    """Sort (key, index) records on the device: returns (perm, stats) with
    perm a CUDA uint32 tensor of origins (the sorted handle sequence)."""
    torch = _torch()
    from .core import Records, Sorter
    if sorter is None:
        sorter = Sorter()
    kt = keys if isinstance(keys, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(keys))
    dev = sorter._device()
    kd = kt.to(f"cuda:{dev}", copy=True).contiguous()
    n = kd.numel()
    perm = torch.arange(n, dtype=torch.int64, device=kd.device).to(torch.uint32)
    stats = sorter.sort_with_stats(Records(kd, perm))
    return kd, perm, stats


def cycle_moves(perm) -> tuple:
    """(moves, cycles) the reference's cycle walk spends on ``perm``
    (bigelem.py:48-76): c + 1 moves per nontrivial cycle of length c.
    Cycles are counted by pointer jumping (each element learns the smallest
    position on its cycle in log2 n gather rounds), on the device for device
    permutations."""
    torch = _torch()
    p = perm if isinstance(perm, torch.Tensor) else torch.as_tensor(np.asarray(perm, dtype=np.int64))
    p = p.to(torch.int64)
    n = p.numel()
    if n == 0:
        return 0, 0
    idx = torch.arange(n, dtype=torch.int64, device=p.device)
    moved = p != idx
    nmoved = int(moved.sum().item())
    if nmoved == 0:
        return 0, 0
    label, nxt = idx.clone(), p.clone()
    for _ in range(max(1, int(n - 1).bit_length())):
        label = torch.minimum(label, label[nxt])
        nxt = nxt[nxt]
    cycles = int(((label == idx) & moved).sum().item())
    return nmoved + cycles, cycles


def sort_indirect(ar, cmp=None, sorter=None) -> Permutation:
    """Sort position handles over ``ar`` on the device and return the
    permutation; ``ar`` is not moved (bigelem.py:37-45)."""
    from .core import Records
    n = len(ar.keys) if isinstance(ar, Records) else len(ar)
    if n == 0:
        return Permutation(())
    if n == 1:
        return Permutation((0,))
    _, perm, _ = _handle_sort(_keys_of(ar, cmp), sorter)
    return Permutation(tuple(perm.to(_torch().int64).cpu().tolist()))


def _rows_gather(rows, perm_dev):
    """rows[:] = rows[perm] on the device through one gather pass."""
    torch = _torch()
    dev = perm_dev.device
    host = not rows.is_cuda if isinstance(rows, torch.Tensor) else True
    rt = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(rows)
    src = rt.to(dev).contiguous() if host or not rt.is_contiguous() else rt
    n = src.shape[0]
    row_bytes = src[0].numel() * src.element_size() if n else 0
    dst = torch.empty_like(src)
    st = N.lib().tsq_apply_permutation(
        ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), n, row_bytes,
        ctypes.c_void_p(perm_dev.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != N.TSQ_OK:
        raise N.TsqError(st, "tsq_apply_permutation")
    rt.copy_(dst)  # back into the caller's rows (device or host)
    if host:
        torch.cuda.current_stream(dev).synchronize()


def apply_permutation(ar, perm) -> int:
    """Rearrange ``ar`` so that ar[i] becomes old ar[perm.map[i]]; returns
    the reference's element-move count (bigelem.py:79-86).  Device rows move
    in one gather pass; host sequences are rearranged in place."""
    torch = _torch()
    from .core import Records
    m = perm.map if isinstance(perm, Permutation) else perm
    target = ar.payload if isinstance(ar, Records) else ar
    n = len(target)
    if len(m) != n:
        raise ValueError("permutation length does not match the array")
    if n == 0:
        return 0
    moves, _ = cycle_moves(m)
    if moves == 0:
        return 0
    if isinstance(target, (torch.Tensor, np.ndarray)):
        pd = torch.as_tensor(np.asarray(m, dtype=np.int64) if not isinstance(m, torch.Tensor) else m)
        dev = torch.cuda.current_device()
        _rows_gather(target, pd.to(f"cuda:{dev}").to(torch.uint32))
        if isinstance(ar, Records):
            _rows_gather(ar.keys, pd.to(f"cuda:{dev}").to(torch.uint32))
    else:
        old = list(target)
        target[:] = [old[j] for j in m]
    return moves


def sort_large_elements(ar, cmp3, sorter) -> SortStats:
    """Late-swapping sort used by ``Sorter.sort_with_stats`` for elements of
    at least ``late_swap_byte_threshold`` bytes (bigelem.py:89-99,
    core.py:1595-1598): handle sort on the device, then one move pass."""
    torch = _torch()
    from .core import Records
    keys_sorted, perm, stats = _handle_sort(_keys_of(ar, cmp3), sorter)
    moves, cycles = cycle_moves(perm)
    if isinstance(ar, Records):
        rows = ar.payload
        if moves:
            _rows_gather(rows, perm)
        kt = ar.keys if isinstance(ar.keys, torch.Tensor) else torch.from_numpy(ar.keys)
        kt.copy_(keys_sorted)
        if not kt.is_cuda:
            torch.cuda.current_stream(keys_sorted.device).synchronize()
    elif isinstance(ar, (torch.Tensor, np.ndarray)):
        t = ar if isinstance(ar, torch.Tensor) else torch.from_numpy(ar)
        t.copy_(keys_sorted)
        if not t.is_cuda:
            torch.cuda.current_stream(keys_sorted.device).synchronize()
    else:
        old = list(ar)
        order = perm.to(torch.int64).cpu().tolist()
        ar[:] = [old[j] for j in order]
    stats.element_writes += moves
    stats.array_writes += moves - cycles
    stats.scratch_writes += cycles
    return stats
