"""ctypes binding of libtsq_b200.so (the C ABI of include/tsq.h).

No CPU fallback exists: if the library is missing or no CUDA device is
present, loading raises.  Importing this module does not touch CUDA.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSQ_LIB") or os.path.join(HERE, "libtsq_b200.so")

TSQ_NONE, TSQ_I32, TSQ_U32, TSQ_I64, TSQ_U64, TSQ_F32, TSQ_F64 = range(7)

(TSQ_OK, TSQ_ERR_ALLOC, TSQ_ERR_UNSUPPORTED_DTYPE, TSQ_ERR_CUDA, TSQ_ERR_DEPTH_EXCEEDED,
 TSQ_ERR_INVALID, TSQ_ERR_BUSY, TSQ_ERR_CAPACITY) = range(8)

EXPORTED_SYMBOLS = (
    "tsq_status_str", "tsq_abi_version", "tsq_workspace_create", "tsq_workspace_destroy",
    "tsq_workspace_bytes", "tsq_workspace_reserve", "tsq_workspace_free",
    "tsq_workspace_capacity", "tsq_workspace_alloc_count", "tsq_sort",
    "tsq_partition_segment", "tsq_select_pivot", "tsq_level_trace", "tsq_apply_permutation",
    "tsq_workspace_last_status",
)

# tsq_stage_kind (include/tsq.h)
TSQ_STAGE_PARTITION, TSQ_STAGE_SORTED, TSQ_STAGE_REVERSED, TSQ_STAGE_HANDLER_FALLBACK = range(4)


class TsqStageRecord(ctypes.Structure):
    _fields_ = [("a", ctypes.c_int64), ("b", ctypes.c_int64), ("new_l", ctypes.c_int64),
                ("new_r", ctypes.c_int64), ("pivot", ctypes.c_uint64), ("kind", ctypes.c_int32),
                ("depth", ctypes.c_int32)]


# void (*)(void *user, int32_t level, const tsq_stage_record *records, uint32_t count)
LEVEL_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32,
                            ctypes.POINTER(TsqStageRecord), ctypes.c_uint32)


class TsqParams(ctypes.Structure):
    _fields_ = [("dran", ctypes.c_double), ("mitigation", ctypes.c_int32),
                ("fast_paths", ctypes.c_int32), ("max_depth", ctypes.c_int32),
                ("host_levels", ctypes.c_int32), ("small_threshold", ctypes.c_int32),
                ("reproducible", ctypes.c_int32), ("stage_export", ctypes.c_int32),
                ("on_level", LEVEL_FN), ("on_level_user", ctypes.c_void_p),
                ("reserved", ctypes.c_int64 * 1)]


class TsqStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in (
        "n", "stages", "levels", "max_depth", "small_segments", "eq_runs", "eq_elements",
        "sorted_bypass", "reversed_bypass", "verify_fallbacks", "partitioned_elements",
        "bytes_partition", "bytes_small", "bytes_retire", "temp_high_water", "error_flags",
        "writes_caller", "writes_workspace", "bisected", "flushes")] + \
        [("ms_levels", ctypes.c_float), ("ms_total", ctypes.c_float)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class TsqError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_str(status)} (status {status})")
        self.status = status


_lib = None
_lock = threading.Lock()


def lib():
    """Load the library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing; build it with "
                "`python -m paper_1505_00558_b200.build` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        L.tsq_status_str.restype = ctypes.c_char_p
        L.tsq_status_str.argtypes = [i32]
        L.tsq_abi_version.restype = i32
        L.tsq_workspace_create.argtypes = [ctypes.POINTER(vp), i32]
        L.tsq_workspace_create.restype = i32
        L.tsq_workspace_destroy.argtypes = [vp]
        L.tsq_workspace_destroy.restype = None
        L.tsq_workspace_bytes.argtypes = [sz, i32, i32]
        L.tsq_workspace_bytes.restype = sz
        L.tsq_workspace_reserve.argtypes = [vp, sz, i32, i32]
        L.tsq_workspace_reserve.restype = i32
        L.tsq_workspace_free.argtypes = [vp]
        L.tsq_workspace_free.restype = i32
        L.tsq_workspace_capacity.argtypes = [vp]
        L.tsq_workspace_capacity.restype = sz
        L.tsq_workspace_alloc_count.argtypes = [vp]
        L.tsq_workspace_alloc_count.restype = ctypes.c_uint64
        L.tsq_sort.argtypes = [vp, vp, sz, i32, i32, ctypes.POINTER(TsqParams), vp, vp,
                               ctypes.POINTER(TsqStats)]
        L.tsq_sort.restype = i32
        L.tsq_partition_segment.argtypes = [vp, vp, vp, vp, sz, i32, i32, ctypes.c_uint64, vp,
                                            vp, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_int64)]
        L.tsq_partition_segment.restype = i32
        L.tsq_select_pivot.argtypes = [vp, sz, i32, ctypes.c_double, ctypes.c_int32, vp, vp,
                                       ctypes.POINTER(ctypes.c_uint64),
                                       ctypes.POINTER(ctypes.c_int32)]
        L.tsq_select_pivot.restype = i32
        L.tsq_level_trace.argtypes = [vp, ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.POINTER(ctypes.c_uint64), i32]
        L.tsq_level_trace.restype = i32
        L.tsq_apply_permutation.argtypes = [vp, vp, sz, sz, vp, vp]
        L.tsq_apply_permutation.restype = i32
        L.tsq_workspace_last_status.argtypes = [vp, vp]
        L.tsq_workspace_last_status.restype = i32
        _lib = L
    return _lib


def status_str(status: int) -> str:
    try:
        return lib().tsq_status_str(status).decode()
    except Exception:  # pragma: no cover - library missing
        return "unknown"


class Workspace:
    """Owner of one tsq_workspace (the device TempStore)."""

    def __init__(self, device: int):
        self.device = device
        h = ctypes.c_void_p()
        st = lib().tsq_workspace_create(ctypes.byref(h), device)
        if st != TSQ_OK:
            raise TsqError(st, "tsq_workspace_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            try:
                _lib.tsq_workspace_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def capacity(self) -> int:
        return int(lib().tsq_workspace_capacity(self.handle))

    @property
    def alloc_count(self) -> int:
        return int(lib().tsq_workspace_alloc_count(self.handle))

    def reserve(self, n: int, key_dt: int, pay_dt: int) -> int:
        return lib().tsq_workspace_reserve(self.handle, n, key_dt, pay_dt)

    def free(self) -> int:
        return lib().tsq_workspace_free(self.handle)

    def level_trace(self):
        cap = 512
        ms = (ctypes.c_float * cap)()
        sms = (ctypes.c_float * cap)()
        segs = (ctypes.c_uint32 * cap)()
        tiles = (ctypes.c_uint32 * cap)()
        nbytes = (ctypes.c_uint64 * cap)()
        n = lib().tsq_level_trace(self.handle, ms, sms, segs, tiles, nbytes, cap)
        n = min(n, cap)
        return [{"ms": ms[i], "sched_ms": sms[i], "segments": segs[i], "tiles": tiles[i],
                 "bytes": nbytes[i]} for i in range(n)]
