"""Reference-facing sort API over the B200 kernels.

Mirrors tsqsort's public sort path (/root/reference/pkg/src/tsqsort/core.py):

  * ``Sorter(config=None, seed=None)``            core.py:1572-1579
  * ``Sorter.sort`` / ``sort_with_stats``          core.py:1583-1614
  * ``Sorter.free_temp_storage``                   core.py:1616-1620
  * module ``sort`` / ``sort_with_stats`` / ``free_temp_storage`` and the
    retained ``default_sorter``                    core.py:1754-1774
  * ``TempAllocationError``                        core.py:46-47

with the same argument meanings and error behaviour: ``ar`` is sorted in
place, a fresh ``SortStats`` is returned, the workspace is retained across
calls until ``free_temp_storage``, an instance is not reentrant, allocation
happens before any mutation.  All sorting runs in libtsq_b200.so on the GPU;
there is no CPU fallback -- unsupported inputs raise.

Accepted containers for ``ar``:
  * a 1-D CUDA tensor (int32/uint32/int64/uint64/float32/float64): in place
  * a CPU tensor or numpy array of those dtypes: staged through the GPU
  * a Python list of ints or floats: converted, sorted, written back
  * ``Records(keys, payload)`` (or a ``(keys, payload)`` tuple of tensors /
    arrays) with a uint32 payload: keys sorted, payload moved with its key
  * a list of ``(key, payload)`` tuples with ``cmp=key_cmp`` -- the
    reference's key-only comparator pattern (tests/test_core.py:93-103)
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .config import DEFAULT_CONFIG, DEFAULT_GPU_CONFIG, GpuConfig, SortConfig
from .instrument import HANDLER_ENTER, HANDLER_FALLBACK, STAGE_END, STATE_ENTER
from .pivot import MitigationRng
from .stats import SortStats

__all__ = ["TempAllocationError", "DepthExceededError", "Records", "key_cmp",
           "DeviceTempStore", "TempStore", "PartitionFrame", "Sorter", "sort",
           "sort_with_stats", "sort_many", "free_temp_storage", "default_sorter"]


class TempAllocationError(MemoryError):
    """The device workspace could not be allocated (array left untouched)."""


class DepthExceededError(RuntimeError):
    """The device level loop hit its hard limit.  Cannot happen in practice:
    beyond GpuConfig.max_depth segments are split at the midpoint of their
    key bounds, which ends every segment within key-bits more levels."""


def key_cmp(x, y) -> int:
    """Key-only comparator for (key, payload) records: compares x[0], y[0]."""
    a, b = x[0], y[0]
    return -1 if a < b else (1 if a > b else 0)


@dataclass
class Records:
    """Keys plus a payload that moves with its key: a uint32 vector (sorted
    along on the device), or rows -- any tensor / array whose first
    dimension is n -- moved once by late swapping (bigelem.py)."""

    keys: object
    payload: object


_TORCH_DT = None


def _torch():
    import torch
    return torch


def _dtype_codes():
    global _TORCH_DT
    if _TORCH_DT is None:
        torch = _torch()
        _TORCH_DT = {
            torch.int32: N.TSQ_I32, torch.uint32: N.TSQ_U32, torch.int64: N.TSQ_I64,
            torch.uint64: N.TSQ_U64, torch.float32: N.TSQ_F32, torch.float64: N.TSQ_F64,
        }
    return _TORCH_DT


def _raise_status(st: int, what: str):
    if st == N.TSQ_OK:
        return
    if st == N.TSQ_ERR_ALLOC:
        raise TempAllocationError(f"{what}: cannot allocate the device workspace")
    if st == N.TSQ_ERR_UNSUPPORTED_DTYPE:
        raise TypeError(f"{what}: unsupported dtype")
    if st == N.TSQ_ERR_INVALID:
        raise ValueError(f"{what}: invalid argument")
    if st == N.TSQ_ERR_BUSY:
        raise RuntimeError("sorter instance is not reentrant")
    if st == N.TSQ_ERR_DEPTH_EXCEEDED:
        raise DepthExceededError(f"{what}: recursion depth guard exceeded")
    raise N.TsqError(st, what)


class DeviceTempStore:
    """Retained device workspace (TempStore, core.py:81-104).

    One workspace per CUDA device the sorter has sorted on (a tensor on
    cuda:1 sorts with cuda:1's workspace, whatever the current device).
    ``capacity`` is the element count of the largest sort served since the
    last release; ``alloc_count`` counts device allocations.
    """

    def __init__(self, device: int | None = None):
        self.device = device   # default device: host containers are staged here
        self._ws = {}

    def workspace(self, device: int | None = None) -> N.Workspace:
        if device is None:
            device = self.device
        if device is None:
            torch = _torch()
            if not torch.cuda.is_available():
                raise RuntimeError("no CUDA device: the B200 sort has no CPU fallback")
            device = torch.cuda.current_device()
        if self.device is None:
            self.device = device
        ws = self._ws.get(device)
        if ws is None:
            ws = self._ws[device] = N.Workspace(device)
        return ws

    @property
    def capacity(self) -> int:
        return max((w.capacity for w in self._ws.values()), default=0)

    @property
    def alloc_count(self) -> int:
        return sum(w.alloc_count for w in self._ws.values())

    def ensure(self, n: int, key_dt: int = N.TSQ_I32, pay_dt: int = N.TSQ_NONE,
               device: int | None = None) -> None:
        _raise_status(self.workspace(device).reserve(n, key_dt, pay_dt), "workspace reserve")

    def release(self) -> None:
        for w in self._ws.values():
            _raise_status(w.free(), "workspace free")


# The reference's names for the retained buffer and the stage frame
# (/root/reference/pkg/src/tsqsort/__init__.py:16-18).  TempStore is the
# device workspace here.  PartitionFrame describes one stage -- the
# (a, b, new_l, new_r, pivot) a stage_hook receives -- with the reference's
# field names; the device recursion has no per-stage frame object of its
# own (core.py:58-78).
TempStore = DeviceTempStore


class PartitionFrame:
    """Index set and pivot of one stage (core.py:58-78): ``a..b`` inclusive,
    after the stage ``[a..new_l] < pivot``, ``(new_l, new_r) == pivot``,
    ``[new_r..b] > pivot``."""

    __slots__ = ("a", "b", "mid", "pi", "pivot", "new_l", "new_r", "depth", "kind")

    def __init__(self, a=0, b=-1, pi=None, pivot=None):
        self.a = a
        self.b = b
        self.mid = (a + b) >> 1
        self.pi = self.mid if pi is None else pi
        self.pivot = pivot
        self.new_l = a - 1
        self.new_r = b + 1
        self.depth = 0
        self.kind = "partition"

    def __repr__(self):
        return (f"PartitionFrame(a={self.a}, b={self.b}, new_l={self.new_l}, "
                f"new_r={self.new_r}, pivot={self.pivot!r}, kind={self.kind!r})")


class _Job:
    """One sort call's device tensors and how to write results back."""

    __slots__ = ("keys", "payload", "n", "key_dt", "pay_dt", "finish", "h2d_bytes",
                 "d2h_bytes")

    def __init__(self):
        self.keys = None
        self.payload = None
        self.n = 0
        self.key_dt = N.TSQ_NONE
        self.pay_dt = N.TSQ_NONE
        self.finish = None
        self.h2d_bytes = 0
        self.d2h_bytes = 0


def _list_to_numpy(values) -> np.ndarray:
    if all(isinstance(v, (bool, int, np.integer)) for v in values):
        try:
            return np.asarray(values, dtype=np.int64)
        except OverflowError:
            try:
                return np.asarray(values, dtype=np.uint64)
            except OverflowError:
                raise TypeError("integers beyond 64 bits are not supported on the GPU path")
    if all(isinstance(v, (float, np.floating)) for v in values):
        return np.asarray(values, dtype=np.float64)
    raise TypeError("lists must hold only ints or only floats on the GPU path "
                    "(custom element types need a comparator the device cannot run)")


class Sorter:
    """A sorter instance: config, mitigation generator, retained workspace.

    Not reentrant (core.py:1589-1590); distinct instances are independent.
    """

    def __init__(self, config: SortConfig | None = None, seed: int | None = None,
                 gpu: GpuConfig | None = None, device: int | None = None):
        self.config = config if config is not None else DEFAULT_CONFIG
        self.gpu = gpu if gpu is not None else DEFAULT_GPU_CONFIG
        self.rng = MitigationRng(seed)
        self.temp = DeviceTempStore(device)
        self.stage_hook = None
        self.trace = None
        self.last_level_trace = None
        self._active = False
        self._lock = threading.Lock()
        self._staging = {}

    # -- public API --

    def sort(self, ar, cmp=None, element_size: int | None = None) -> None:
        self.sort_with_stats(ar, cmp, element_size)

    def sort_with_stats(self, ar, cmp=None, element_size: int | None = None) -> SortStats:
        """Sort ``ar`` in place on the GPU; returns the run's counters.

        Elements of ``element_size >= config.late_swap_byte_threshold`` bytes
        (and ``Records`` whose payload is a tensor of rows) take the late-swap
        path: a device handle sort, then one gather pass over the elements
        (bigelem.py, dispatched before the reentrancy guard as in
        core.py:1595-1598)."""
        late = (element_size is not None and
                element_size >= self.config.late_swap_byte_threshold) or _rows_payload(ar)
        if late and self._active:
            raise RuntimeError("sorter instance is not reentrant")
        if late and _length(ar) > 1:
            from .bigelem import sort_large_elements
            return sort_large_elements(ar, cmp, self)
        with self._lock:
            if self._active:
                raise RuntimeError("sorter instance is not reentrant")
            self._active = True
        try:
            return self._sort(ar, cmp, element_size)
        finally:
            self._active = False

    def sort_many(self, arrays, cmp=None) -> list:
        """Sort a sequence of host arrays, each in place, as a pipeline.

        Extension beyond the reference API for host-resident batches: the
        host->device copy of array i+1 and the device->host copy of array i-1
        run on their own streams (the copy engines work both directions at
        once) while array i sorts, so a batch costs about max(H2D, D2H, sort)
        per array instead of their sum.  Every array must be a contiguous 1-D
        CPU tensor (pinned memory for real overlap) or numpy array of one
        native key dtype; device tensors, lists and records go through sort().
        Returns one SortStats per array.
        """
        torch = _torch()
        if cmp is not None:
            raise TypeError("sort_many sorts native keys only (cmp=None)")
        items = []
        for a in arrays:
            t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
            if not isinstance(t, torch.Tensor) or t.is_cuda or t.dim() != 1 \
                    or not t.is_contiguous():
                raise TypeError("sort_many takes contiguous 1-D host arrays")
            items.append(t)
        if not items:
            return []
        dtype = items[0].dtype
        if any(t.dtype != dtype for t in items):
            raise TypeError("sort_many needs one key dtype across the batch")
        if dtype not in _dtype_codes():
            raise TypeError(f"unsupported key dtype {dtype}")
        dev = self._device()
        nmax = max(t.numel() for t in items)
        # three device buffers: array i sorts in one while array i+1 lands in
        # the next and array i-1 drains from the third
        NB = 3
        bufs = []
        for k in range(NB):
            b = self._staging.get(f"pipe{k}")
            if b is None or b.dtype != dtype or b.numel() < nmax:
                try:
                    b = torch.empty(nmax, dtype=dtype, device=f"cuda:{dev}")
                except torch.OutOfMemoryError as exc:
                    raise TempAllocationError("cannot allocate the pipeline buffers") from exc
                self._staging[f"pipe{k}"] = b
            bufs.append(b)
        compute = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(NB)]
        ev_out = [torch.cuda.Event() for _ in range(NB)]
        ev_sorted = torch.cuda.Event()
        used = [False] * NB

        def h2d(i):
            k, t = i % NB, items[i]
            if used[k]:
                s_in.wait_event(ev_out[k])  # the D2H of array i-NB has drained it
            with torch.cuda.stream(s_in):
                bufs[k][:t.numel()].copy_(t, non_blocking=True)
                ev_in[k].record(s_in)
            used[k] = True

        out = []
        h2d(0)
        for i, t in enumerate(items):
            if i + 1 < len(items):
                h2d(i + 1)
            k = i % NB
            compute.wait_event(ev_in[k])
            st = self.sort_with_stats(bufs[k][:t.numel()])
            st.gpu["h2d_bytes"] = st.gpu["d2h_bytes"] = t.numel() * t.element_size()
            out.append(st)
            ev_sorted.record(compute)
            s_out.wait_event(ev_sorted)
            with torch.cuda.stream(s_out):
                t.copy_(bufs[k][:t.numel()], non_blocking=True)
                ev_out[k].record(s_out)
        s_out.synchronize()
        return out

    def free_temp_storage(self) -> None:
        """Release the retained workspace; the next sort reallocates."""
        if self._active:
            raise RuntimeError("cannot free temp storage during a sort")
        self.temp.release()
        self._staging.clear()

    # -- internals --

    def _device(self) -> int:
        dev = getattr(self.temp, "device", None)
        if dev is None:
            torch = _torch()
            if not torch.cuda.is_available():
                raise RuntimeError("no CUDA device: the B200 sort has no CPU fallback")
            dev = torch.cuda.current_device()
        return dev

    def _stage(self, host, slot: str):
        """Device copy of a host tensor through a retained staging buffer."""
        torch = _torch()
        dev = self._device()
        buf = self._staging.get(slot)
        if buf is None or buf.dtype != host.dtype or buf.numel() < host.numel():
            try:
                buf = torch.empty(host.numel(), dtype=host.dtype, device=f"cuda:{dev}")
            except torch.OutOfMemoryError as exc:
                raise TempAllocationError("cannot allocate the device staging buffer") from exc
            self._staging[slot] = buf
        d = buf[:host.numel()]
        d.copy_(host, non_blocking=True)
        return d

    def _prepare(self, ar, cmp) -> _Job:
        torch = _torch()
        codes = _dtype_codes()
        job = _Job()
        if cmp is not None and cmp is not key_cmp:
            raise TypeError("custom comparators cannot run on the GPU path; pass cmp=None "
                            "(native order) or cmp=key_cmp for (key, payload) records")
        # records given as separate arrays
        if isinstance(ar, Records) or (isinstance(ar, tuple) and len(ar) == 2 and
                                       all(isinstance(x, (np.ndarray, torch.Tensor)) for x in ar)):
            keys, pay = (ar.keys, ar.payload) if isinstance(ar, Records) else ar
            kt = keys if isinstance(keys, torch.Tensor) else torch.from_numpy(keys)
            pt = pay if isinstance(pay, torch.Tensor) else torch.from_numpy(pay)
            if pt.dtype != torch.uint32 or pt.shape != kt.shape or kt.dim() != 1:
                raise TypeError("records need 1-D keys and a uint32 payload of the same length")
            self._bind(job, kt, pt, codes)
            return job
        if isinstance(ar, np.ndarray):
            ar_t = torch.from_numpy(ar) if ar.flags.c_contiguous else None
            if ar_t is None:
                raise ValueError("numpy input must be C-contiguous")
            self._bind(job, ar_t, None, codes)
            return job
        if isinstance(ar, torch.Tensor):
            self._bind(job, ar, None, codes)
            return job
        # generic Python sequence
        values = list(ar)
        n = len(values)
        job.n = n
        if n <= 1:
            return job
        if cmp is key_cmp:
            keys = _list_to_numpy([v[0] for v in values])
            pay = np.arange(n, dtype=np.uint32)
            kt = torch.from_numpy(keys)
            pt = torch.from_numpy(pay)
            self._bind(job, kt, pt, codes)
            inner = job.finish

            def finish_records(final=True):
                inner(final)
                perm = pay
                ar[:] = [values[i] for i in perm.tolist()]

            job.finish = finish_records
            return job
        arr = _list_to_numpy(values)
        kt = torch.from_numpy(arr)
        self._bind(job, kt, None, codes)
        inner = job.finish

        def finish_list(final=True):
            inner(final)
            ar[:] = arr.tolist()

        job.finish = finish_list
        return job

    def _bind(self, job: _Job, keys, payload, codes):
        torch = _torch()
        if keys.dim() != 1:
            raise ValueError("keys must be one-dimensional")
        if keys.dtype not in codes:
            raise TypeError(f"unsupported key dtype {keys.dtype}")
        job.n = keys.numel()
        job.key_dt = codes[keys.dtype]
        job.pay_dt = N.TSQ_U32 if payload is not None else N.TSQ_NONE
        if job.n <= 1:
            job.finish = lambda final=True: None
            return
        outs = []
        devs = []
        for slot, t in (("keys", keys), ("payload", payload)):
            if t is None:
                devs.append(None)
                continue
            if t.is_cuda:
                if t.is_contiguous():
                    devs.append(t)
                else:
                    d = t.contiguous()
                    devs.append(d)
                    outs.append((t, d))
            else:
                host = t if t.is_contiguous() else t.contiguous()
                d = self._stage(host, slot)
                job.h2d_bytes += host.numel() * host.element_size()
                devs.append(d)
                outs.append((t, d))
        job.keys, job.payload = devs

        if payload is not None and keys.is_cuda and payload.is_cuda and \
                keys.device != payload.device:
            raise ValueError("keys and payload must be on the same device")

        def finish(final=True):
            # final=False: a stage-export refresh of the host container
            if not outs:
                return
            for dst, src in outs:
                dst.copy_(src, non_blocking=not dst.is_cuda)
                if final and not dst.is_cuda:
                    job.d2h_bytes += dst.numel() * dst.element_size()
            torch.cuda.current_stream(src.device).synchronize()

        job.finish = finish

    def _sort(self, ar, cmp, element_size) -> SortStats:
        job = self._prepare(ar, cmp)
        stats = SortStats()
        if job.n <= 1:
            return stats
        torch = _torch()
        dev = job.keys.device.index
        # allocation precedes any mutation (core.py:1599): the array stays
        # untouched if this raises
        self.temp.ensure(job.n, job.key_dt, job.pay_dt, dev)
        self.rng.next()
        p = N.TsqParams()
        p.dran = self.rng.dran
        p.mitigation = 1 if self.config.mitigation_enabled else 0
        p.fast_paths = 1 if self.gpu.fast_paths else 0
        p.max_depth = self.gpu.max_depth
        p.small_threshold = self.gpu.small_threshold
        p.reproducible = 1 if self.gpu.reproducible else 0
        p.host_levels = 1 if self.gpu.host_levels else 0
        hook, trace = self.stage_hook, self.trace
        errors = []
        if hook is not None or trace is not None:
            # stage export: after every device level the caller's array holds
            # each stage's post-stage contents, then hook(a, b, new_l, new_r,
            # pivot) runs per stage and the trace gets its events
            # (core.py:1676-1710)
            decode = _pivot_decoder(job.keys.dtype)

            def on_level(_user, level, recs, count):
                if errors:
                    return
                try:
                    job.finish(False)
                    for i in range(count):
                        _emit_stage(recs[i], decode, hook, trace)
                except BaseException as exc:  # re-raised after the call
                    errors.append(exc)

            cb = N.LEVEL_FN(on_level)
            p.stage_export = 1
            p.on_level = cb
        ts = N.TsqStats()
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = self.temp.workspace(dev)
        st = N.lib().tsq_sort(
            ctypes.c_void_p(job.keys.data_ptr()),
            ctypes.c_void_p(job.payload.data_ptr()) if job.payload is not None else None,
            job.n, job.key_dt, job.pay_dt, ctypes.byref(p), ws.handle,
            ctypes.c_void_p(stream), ctypes.byref(ts))
        if errors:
            raise errors[0]
        _raise_status(st, "tsq_sort")
        if p.host_levels or p.stage_export:
            self.last_level_trace = ws.level_trace()
        job.finish()
        if trace is not None:
            trace.emit(STAGE_END, 0, job.n - 1, "root")
        return _to_stats(ts, job)




def _pivot_decoder(dtype):
    """Raw bits of a key of ``dtype`` -> the Python value."""
    torch = _torch()
    np_dt = {torch.int32: np.int32, torch.uint32: np.uint32, torch.int64: np.int64,
             torch.uint64: np.uint64, torch.float32: np.float32,
             torch.float64: np.float64}[dtype]
    bits_dt = np.uint32 if np.dtype(np_dt).itemsize == 4 else np.uint64

    def decode(bits: int):
        return np.asarray([bits], dtype=np.uint64).astype(bits_dt).view(np_dt)[0].item()

    return decode


def _emit_stage(rec, decode, hook, trace) -> None:
    """One device stage record -> stage_hook call and trace events, in the
    order the reference's _range emits them (core.py:1676-1710)."""
    a, b = int(rec.a), int(rec.b)
    kind = int(rec.kind)
    if kind == N.TSQ_STAGE_HANDLER_FALLBACK:
        if trace is not None:
            name = "sorted" if int(rec.new_l) == N.TSQ_STAGE_SORTED else "reversed"
            trace.emit(HANDLER_ENTER, name, a, b)
            trace.emit(HANDLER_FALLBACK, name, "prescan")
        return
    pivot = decode(int(rec.pivot))
    new_l, new_r = int(rec.new_l), int(rec.new_r)
    if trace is not None:
        if kind == N.TSQ_STAGE_PARTITION:
            trace.emit(STATE_ENTER, "prescan", a, b)
        else:
            trace.emit(HANDLER_ENTER, "sorted" if kind == N.TSQ_STAGE_SORTED else "reversed",
                       a, b)
    if hook is not None:
        hook(a, b, new_l, new_r, pivot)
    if trace is not None:
        trace.emit(STAGE_END, a, b, new_l, new_r)


def _rows_payload(ar) -> bool:
    """Records whose payload is not a 1-D uint32 vector: rows that move by
    late swapping."""
    if not isinstance(ar, Records):
        return False
    p = ar.payload
    if isinstance(p, np.ndarray):
        return p.ndim != 1 or p.dtype != np.uint32
    torch = _torch()
    return isinstance(p, torch.Tensor) and (p.dim() != 1 or p.dtype != torch.uint32)


def _length(ar) -> int:
    return len(ar.keys) if isinstance(ar, Records) else len(ar)


def _to_stats(ts: N.TsqStats, job: _Job) -> SortStats:
    s = SortStats()
    s.comparisons = int(ts.partitioned_elements)
    s.array_writes = int(ts.writes_caller)
    s.scratch_writes = int(ts.writes_workspace)
    s.element_writes = s.array_writes + s.scratch_writes
    s.temp_high_water = int(ts.temp_high_water)
    s.max_depth = int(ts.max_depth)
    s.stages = int(ts.stages)
    s.state_activations = {"partition": int(ts.stages - ts.sorted_bypass - ts.reversed_bypass),
                           "eq_run": int(ts.eq_runs), "small": int(ts.small_segments)}
    s.handler_activations = {"sorted": int(ts.sorted_bypass),
                             "reversed": int(ts.reversed_bypass),
                             "fallbacks": int(ts.verify_fallbacks)}
    g = ts.as_dict()
    g["h2d_bytes"] = job.h2d_bytes
    g["d2h_bytes"] = job.d2h_bytes
    s.gpu = g
    return s


# ---------------------------------------------------------------------------
# Module-level convenience API around a default retained instance
# (core.py:1754-1774).

default_sorter = Sorter()


def sort(ar, cmp=None, config: SortConfig | None = None,
         element_size: int | None = None) -> SortStats:
    """Sort in place with the module's default sorter instance."""
    global default_sorter
    if config is not None and config != default_sorter.config:
        fresh = Sorter(config, seed=default_sorter.rng.zgen, gpu=default_sorter.gpu)
        fresh.temp = default_sorter.temp  # keep the retained workspace
        default_sorter = fresh
    return default_sorter.sort_with_stats(ar, cmp, element_size)


def sort_with_stats(ar, cmp=None, config: SortConfig | None = None,
                    element_size: int | None = None) -> SortStats:
    return sort(ar, cmp, config, element_size)


def sort_many(arrays, cmp=None) -> list:
    """Pipelined in-place sort of host arrays with the default sorter."""
    return default_sorter.sort_many(arrays, cmp)


def free_temp_storage() -> None:
    default_sorter.free_temp_storage()
