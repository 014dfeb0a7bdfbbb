"""Per-stage test surface (the reference's init_stage .. copy_back contract,
core.py:1789-1870, and select_pivot, pivot.py:205-248) on the device.

``partition_segment`` runs ONE three-way partition pass of the level kernel
over a CUDA tensor around a given pivot and returns ``(out, new_l, new_r)``
with the stage law of tests/conftest.py:37-45: ``out[:new_l+1] < p``,
``out[new_l+1:new_r] == p``, ``out[new_r:] > p``.
"""

from __future__ import annotations

import ctypes

from . import _native as N
from .core import DeviceTempStore, _dtype_codes, _raise_status

_store = None


def _ws(store):
    global _store
    if store is None:
        if _store is None:
            _store = DeviceTempStore()
        store = _store
    return store.workspace()


def _raw_bits(value, dtype) -> int:
    import numpy as np
    import torch
    np_dt = {torch.int32: np.int32, torch.uint32: np.uint32, torch.int64: np.int64,
             torch.uint64: np.uint64, torch.float32: np.float32,
             torch.float64: np.float64}[dtype]
    arr = np.asarray([value], dtype=np_dt)
    return int(arr.view(np.uint32 if arr.itemsize == 4 else np.uint64)[0])


def partition_segment(keys, pivot, payload=None, store: DeviceTempStore | None = None):
    import torch
    codes = _dtype_codes()
    if not keys.is_cuda or keys.dim() != 1 or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous 1-D CUDA tensor")
    out = torch.empty_like(keys)
    out_p = torch.empty_like(payload) if payload is not None else None
    nl = ctypes.c_int64()
    nr = ctypes.c_int64()
    ws = _ws(store)
    stream = torch.cuda.current_stream(keys.device).cuda_stream
    st = N.lib().tsq_partition_segment(
        ctypes.c_void_p(keys.data_ptr()),
        ctypes.c_void_p(payload.data_ptr()) if payload is not None else None,
        ctypes.c_void_p(out.data_ptr()),
        ctypes.c_void_p(out_p.data_ptr()) if out_p is not None else None,
        keys.numel(), codes[keys.dtype], N.TSQ_U32 if payload is not None else N.TSQ_NONE,
        _raw_bits(pivot, keys.dtype), ws.handle, ctypes.c_void_p(stream), ctypes.byref(nl),
        ctypes.byref(nr))
    _raise_status(st, "tsq_partition_segment")
    if payload is not None:
        return out, out_p, int(nl.value), int(nr.value)
    return out, int(nl.value), int(nr.value)


def select_pivot(keys, dran: float = 1.0, mitigation: bool = True,
                 store: DeviceTempStore | None = None):
    """Device pivot sampling of a CUDA tensor -> (pivot value, order flag)."""
    import numpy as np
    import torch
    codes = _dtype_codes()
    piv = ctypes.c_uint64()
    flag = ctypes.c_int32()
    ws = _ws(store)
    stream = torch.cuda.current_stream(keys.device).cuda_stream
    st = N.lib().tsq_select_pivot(ctypes.c_void_p(keys.data_ptr()), keys.numel(),
                                  codes[keys.dtype], float(dran), int(mitigation), ws.handle,
                                  ctypes.c_void_p(stream), ctypes.byref(piv), ctypes.byref(flag))
    _raise_status(st, "tsq_select_pivot")
    np_dt = {torch.int32: np.int32, torch.uint32: np.uint32, torch.int64: np.int64,
             torch.uint64: np.uint64, torch.float32: np.float32,
             torch.float64: np.float64}[keys.dtype]
    bits = np.asarray([piv.value], dtype=np.uint64)
    if np.dtype(np_dt).itemsize == 4:
        bits = bits.astype(np.uint32)
    return bits.view(np_dt)[0].item(), int(flag.value)
