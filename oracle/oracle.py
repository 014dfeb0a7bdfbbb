"""oracle.oracle -- TEST INFRASTRUCTURE ONLY.

ctypes front end of the plain-C restatement of tsqsort's sort path
(oracle/tsq_oracle.c).  Used by tests/ (parity checker), by
``__graft_entry__.smoke()`` and by bench.py's ``cpu_baseline`` /
``--impl reference`` legs.  The product package never imports this module.

Reference correspondences (``/root/reference/pkg/src/tsqsort``):
  * ``MitigationRng``              -> pivot.py:25-54
  * ``select_pivot_i64``           -> pivot.py:205-248 (+ medians 66-194)
  * ``insertion_sort_i64``         -> smallsort.py:12-47
  * ``partition3_i64``             -> core.py:944-967 stage-exit contract
  * ``sort``                       -> Sorter.sort_with_stats, core.py:1586-1614
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtsq_oracle.so")

DTYPE_CODES = {
    np.dtype(np.int32): 1,
    np.dtype(np.uint32): 2,
    np.dtype(np.int64): 3,
    np.dtype(np.uint64): 4,
    np.dtype(np.float32): 5,
    np.dtype(np.float64): 6,
}


class _Config(ctypes.Structure):
    _fields_ = [
        ("insertion_threshold", ctypes.c_int64),
        ("medof3_max_n", ctypes.c_int64),
        ("medof5_max_n", ctypes.c_int64),
        ("ninther_max_n", ctypes.c_int64),
        ("reverse_tolerance", ctypes.c_int64),
        ("mitigation_enabled", ctypes.c_int32),
        ("medof3_small_enabled", ctypes.c_int32),
    ]


class _Rng(ctypes.Structure):
    _fields_ = [("zgen", ctypes.c_uint64), ("dran", ctypes.c_double),
                ("dran2", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_uint64) for name in (
        "comparisons", "array_writes", "scratch_writes", "max_depth", "stages",
        "handler_sorted", "handler_reversed", "handler_fallbacks")]


class _Decision(ctypes.Structure):
    _fields_ = [("pi", ctypes.c_int64), ("order_flag", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/libtsq_oracle.so with the committed Makefile."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []),
                       check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.tsqo_default_config.argtypes = [ctypes.POINTER(_Config)]
        L.tsqo_rng_init.argtypes = [ctypes.POINTER(_Rng), ctypes.c_uint64]
        L.tsqo_rng_next.argtypes = [ctypes.POINTER(_Rng)]
        L.tsqo_sort.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_int, ctypes.POINTER(_Config),
                                ctypes.POINTER(_Rng), ctypes.c_int,
                                ctypes.POINTER(_Stats)]
        L.tsqo_sort.restype = ctypes.c_int
        L.tsqo_select_pivot_i64.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(_Config), ctypes.POINTER(_Rng),
            ctypes.POINTER(ctypes.c_uint64)]
        L.tsqo_select_pivot_i64.restype = _Decision
        L.tsqo_insertion_sort_i64.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_uint64)]
        L.tsqo_partition3_i64.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        _lib = L
    return _lib


def make_config(insertion_threshold=16, medof3_max_n=70, medof5_max_n=600,
                ninther_max_n=60000, reverse_tolerance=3,
                mitigation_enabled=True, medof3_small_enabled=True) -> _Config:
    return _Config(insertion_threshold, medof3_max_n, medof5_max_n,
                   ninther_max_n, reverse_tolerance, int(mitigation_enabled),
                   int(medof3_small_enabled))


def config_from(cfg) -> _Config:
    """Accept any object with SortConfig's attribute names (config.py:8-42)."""
    if cfg is None:
        return make_config()
    return make_config(cfg.insertion_threshold, cfg.medof3_max_n,
                       cfg.medof5_max_n, cfg.ninther_max_n,
                       cfg.reverse_tolerance, cfg.mitigation_enabled,
                       cfg.medof3_small_enabled)


class MitigationRng:
    """Park-Miller generator, pivot.py:25-49 (restated in C)."""

    def __init__(self, seed: int):
        self._r = _Rng()
        if int(seed) % 2147483648 == 0:
            raise ValueError("seed must be nonzero mod 2^31 in the oracle")
        lib().tsqo_rng_init(ctypes.byref(self._r), int(seed))

    def next(self):
        lib().tsqo_rng_next(ctypes.byref(self._r))
        return self

    @property
    def zgen(self) -> int:
        return int(self._r.zgen)

    @property
    def dran(self) -> float:
        return float(self._r.dran)

    @property
    def dran2(self) -> float:
        return float(self._r.dran2)


@dataclass
class OracleStats:
    comparisons: int
    array_writes: int
    scratch_writes: int
    max_depth: int
    stages: int
    handler_sorted: int
    handler_reversed: int
    handler_fallbacks: int


def sort(keys: np.ndarray, payload: np.ndarray | None = None, seed: int = 1,
         config=None, threads: int = 1, rng: MitigationRng | None = None
         ) -> OracleStats:
    """Sort ``keys`` (and ``payload`` alongside) in place on the CPU."""
    if not keys.flags.c_contiguous:
        raise ValueError("keys must be C-contiguous")
    code = DTYPE_CODES.get(keys.dtype)
    if code is None:
        raise TypeError(f"unsupported key dtype {keys.dtype}")
    pay_ptr = None
    if payload is not None:
        if payload.dtype != np.uint32 or payload.shape != keys.shape or \
                not payload.flags.c_contiguous:
            raise TypeError("payload must be a contiguous uint32 array of n")
        pay_ptr = payload.ctypes.data
    if rng is None:
        rng = MitigationRng(seed)
    cfg = config_from(config)
    st = _Stats()
    rc = lib().tsqo_sort(keys.ctypes.data, pay_ptr, keys.size, code,
                         ctypes.byref(cfg), ctypes.byref(rng._r), int(threads),
                         ctypes.byref(st))
    if rc != 0:
        raise RuntimeError(f"oracle sort failed ({rc})")
    return OracleStats(*(int(getattr(st, f)) for f, _ in _Stats._fields_))


def select_pivot_i64(ar: np.ndarray, a: int, b: int, config=None,
                     dran: float = 1.0):
    """select_pivot on an int64 array in place -> (pi, flag, tally)."""
    assert ar.dtype == np.int64 and ar.flags.c_contiguous
    r = _Rng(1, float(dran), 1.0 + float(dran))
    cfg = config_from(config) if not isinstance(config, _Config) else config
    tally = (ctypes.c_uint64 * 3)()
    d = lib().tsqo_select_pivot_i64(ar.ctypes.data, a, b, ctypes.byref(cfg),
                                    ctypes.byref(r), tally)
    return int(d.pi), int(d.order_flag), [int(x) for x in tally]


def insertion_sort_i64(ar: np.ndarray, lo: int, hi: int):
    assert ar.dtype == np.int64 and ar.flags.c_contiguous
    tally = (ctypes.c_uint64 * 3)()
    lib().tsqo_insertion_sort_i64(ar.ctypes.data, lo, hi, tally)
    return [int(x) for x in tally]


def partition3_i64(ar: np.ndarray, a: int, b: int, p: int):
    assert ar.dtype == np.int64 and ar.flags.c_contiguous
    nl = ctypes.c_int64()
    nr = ctypes.c_int64()
    lib().tsqo_partition3_i64(ar.ctypes.data, a, b, int(p), ctypes.byref(nl),
                              ctypes.byref(nr))
    return int(nl.value), int(nr.value)
