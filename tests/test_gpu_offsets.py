"""Sorting caller buffers that are element- but not 16-byte-aligned: CUDA
views with a storage offset (``x[1:]``), keys and payload offset
differently, through the Python API and the C ABI, against the oracle.

The partition pass writes whole runs with cp.async.bulk, which needs
16-byte-aligned global addresses; such buffers are sorted through an aligned
workspace copy (tsq_capi.cu, `staged`).  The reference sorts any indexable
sequence in place (core.py:1586-1614), views included.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from paper_1505_00558_b200 import _native as N
from paper_1505_00558_b200 import stage
from conftest import assert_records_consistent
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _oracle(keys):
    k = keys.copy()
    O.sort(k, seed=1, threads=16)
    return k


def _random(dtype, n, rng):
    dt = np.dtype(dtype)
    if dt.kind == "f":
        return rng.standard_normal(n).astype(dt)
    info = np.iinfo(dt)
    return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)


@pytest.mark.parametrize("off", [1, 3, 5])
@pytest.mark.parametrize("n", [1 << 20, 1 << 24])
@pytest.mark.parametrize("dtype", [np.int32, np.uint64, np.float64])
def test_offset_view_keys(cuda_ok, dtype, n, off):
    rng = np.random.default_rng(n + off)
    x = _random(dtype, n + off + 3, rng)
    base = torch.from_numpy(x).cuda()
    view = base[off:off + n]
    assert view.data_ptr() % 16 != 0
    T.Sorter(seed=1).sort(view)
    got = base.cpu().numpy()
    assert got[off:off + n].tobytes() == _oracle(x[off:off + n]).tobytes()
    # nothing outside the view is touched
    assert got[:off].tobytes() == x[:off].tobytes()
    assert got[off + n:].tobytes() == x[off + n:].tobytes()


@pytest.mark.parametrize("koff,poff", [(1, 0), (0, 3), (1, 3), (5, 2)])
@pytest.mark.parametrize("n", [1 << 20, 1 << 24])
def test_offset_view_records(cuda_ok, n, koff, poff):
    rng = np.random.default_rng(n + 7 * koff + poff)
    keys = rng.integers(0, 1 << 20, n + 8, dtype=np.uint64)
    kb = torch.from_numpy(keys).cuda()
    # payload = index into the key view
    pb = torch.from_numpy((np.arange(n + 8, dtype=np.int64) - poff).astype(np.uint32)).cuda()
    kv, pv = kb[koff:koff + n], pb[poff:poff + n]
    T.Sorter(seed=1).sort(T.Records(kv, pv))
    k_in = keys[koff:koff + n]
    assert_records_consistent(k_in, kv.cpu().numpy(), pv.cpu().numpy(), _oracle(k_in))


@pytest.mark.parametrize("gpu", [T.GpuConfig(host_levels=True), T.GpuConfig(reproducible=True),
                                 T.GpuConfig(small_threshold=64)],
                         ids=["host_levels", "reproducible", "tiny_cut"])
def test_offset_view_modes(cuda_ok, gpu):
    rng = np.random.default_rng(4)
    x = rng.integers(0, 1000, (1 << 20) + 1).astype(np.int32)
    base = torch.from_numpy(x).cuda()
    T.Sorter(seed=1, gpu=gpu).sort(base[1:])
    assert base[1:].cpu().numpy().tobytes() == np.sort(x[1:]).tobytes()
    assert int(base[0]) == int(x[0])


def test_partition_segment_offset_buffers(cuda_ok):
    """tsq_partition_segment into misaligned outputs (C ABI): the stage law
    and the multiset hold."""
    rng = np.random.default_rng(6)
    n = 300001
    x = rng.integers(0, 50, n + 4).astype(np.int32)
    src = torch.from_numpy(x).cuda()[1:1 + n]
    out = torch.empty(n + 4, dtype=torch.int32, device="cuda")[3:3 + n]
    nl, nr = ctypes.c_int64(), ctypes.c_int64()
    ws = N.Workspace(0)
    st = N.lib().tsq_partition_segment(
        ctypes.c_void_p(src.data_ptr()), None, ctypes.c_void_p(out.data_ptr()), None, n,
        N.TSQ_I32, N.TSQ_NONE, 25, ws.handle,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(nl),
        ctypes.byref(nr))
    assert st == N.TSQ_OK
    o = out.cpu().numpy()
    a = x[1:1 + n]
    assert nl.value == (a < 25).sum() - 1 and nr.value == n - (a > 25).sum()
    assert (o[:nl.value + 1] < 25).all() and (o[nl.value + 1:nr.value] == 25).all()
    assert (o[nr.value:] > 25).all()
    assert np.array_equal(np.sort(o), np.sort(a))
    # and through the stage surface on an offset input view
    o2, l2, r2 = stage.partition_segment(torch.from_numpy(x).cuda()[1:1 + n], 25)
    assert (l2, r2) == (nl.value, nr.value)


def test_misaligned_element_pointer_rejected(cuda_ok):
    """A pointer that is not aligned to its element size is invalid."""
    buf = torch.zeros(1024, dtype=torch.int32, device="cuda")
    ws = N.Workspace(0)
    st = N.lib().tsq_sort(ctypes.c_void_p(buf.data_ptr() + 2), None, 1000, N.TSQ_I32,
                          N.TSQ_NONE, None, ws.handle, None, None)
    assert st == N.TSQ_ERR_INVALID
