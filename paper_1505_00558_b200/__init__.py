"""paper_1505_00558_b200: a B200-native three-way partition sort.

Drop-in for the sort path of the reference package ``tsqsort`` 0.1.0
(Triple State QuickSort, arXiv:1505.00558): the same ``sort`` /
``sort_with_stats`` / ``Sorter`` / ``SortConfig`` / ``free_temp_storage`` /
``TempAllocationError`` API (reference __init__.py:12-43, core.py:1563-1775),
backed by hand-written sm_100a CUDA kernels in libtsq_b200.so (C ABI:
include/tsq.h).  Importing does not touch CUDA; the first sort does, and
raises if the library or the device is missing (no CPU fallback).
"""

from .config import DEFAULT_CONFIG, DEFAULT_GPU_CONFIG, GpuConfig, SortConfig
from .core import (DepthExceededError, DeviceTempStore, PartitionFrame, Records, Sorter,
                   TempAllocationError, TempStore, free_temp_storage, key_cmp, sort,
                   sort_many, sort_with_stats)
from .instrument import TraceSink
from .bigelem import Permutation, apply_permutation, sort_indirect
from .pivot import MitigationRng, rng_next
from .stats import SortStats

__version__ = "0.1.0"


def _tristate_entry(ar, cmp=None, seed: int = 1, config=None) -> SortStats:
    """REGISTRY entry with the reference's signature (baselines.py:559-562)."""
    return Sorter(config, seed=seed).sort_with_stats(ar, cmp)


REGISTRY = {"tristate": _tristate_entry}


def get_algorithm(name: str):
    try:
        return REGISTRY[name]
    except KeyError:
        raise KeyError(
            f"unknown algorithm {name!r}; valid: {', '.join(sorted(REGISTRY))}") from None


__all__ = [
    "DEFAULT_CONFIG", "DEFAULT_GPU_CONFIG", "DepthExceededError", "DeviceTempStore",
    "GpuConfig", "MitigationRng", "PartitionFrame", "Permutation", "REGISTRY", "Records",
    "SortConfig", "SortStats", "Sorter", "TempAllocationError", "TempStore", "TraceSink",
    "apply_permutation", "free_temp_storage", "get_algorithm", "key_cmp", "rng_next", "sort",
    "sort_indirect", "sort_many", "sort_with_stats",
]
