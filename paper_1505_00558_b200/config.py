"""Sorter configuration.

``SortConfig`` keeps the reference's fields, defaults and validation
(/root/reference/pkg/src/tsqsort/config.py:8-42) so reference callers pass
their configs unchanged.  On the device the ladder thresholds are not used
for pivot choice (every segment is sampled with ~sqrt(n) strided positions);
``mitigation_enabled`` drives the sample jitter, ``late_swap_byte_threshold``
the ``element_size`` rejection.  GPU-only knobs live in ``GpuConfig``
because SortConfig's validation caps insertion_threshold below
``medof3_max_n`` (config.py:31-38).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class SortConfig:
    insertion_threshold: int = 16
    medof3_max_n: int = 70
    medof5_max_n: int = 600
    ninther_max_n: int = 60000
    reverse_tolerance: int = 3
    mitigation_enabled: bool = True
    late_swap_byte_threshold: int = 320
    medof3_small_enabled: bool = True

    def __post_init__(self):
        if self.insertion_threshold < 3:
            raise ValueError("insertion_threshold must be >= 3")
        ladder = (self.insertion_threshold, self.medof3_max_n, self.medof5_max_n,
                  self.ninther_max_n)
        if any(b <= a for a, b in zip(ladder, ladder[1:])):
            raise ValueError("pivot ladder thresholds must be strictly increasing")
        if self.reverse_tolerance < 0:
            raise ValueError("reverse_tolerance must be >= 0")
        if self.late_swap_byte_threshold < 1:
            raise ValueError("late_swap_byte_threshold must be >= 1")


DEFAULT_CONFIG = SortConfig()


@dataclass(frozen=True)
class GpuConfig:
    """Device knobs.

    fast_paths   verify-and-bypass segments whose samples look sorted or
                 reversed (the _sorted_handler / _reversed_handler role,
                 core.py:991-1556); results are identical either way.
    max_depth    depth guard: segments deeper than this are split at the
                 midpoint of their key bounds instead of a sampled pivot,
                 which ends every segment within key-bits more levels (the
                 reference's _range always finishes, core.py:1643-1728);
                 0 = max(24, 2 * ceil(log2 n)).
    small_threshold  segments of at most this many keys finish in the on-chip
                 sort; 0 = the measured default (4-byte keys 40952 -- 8184 up
                 to 2^21 keys --, records and 8-byte keys 8184); values above
                 the key type's on-chip capacity are clamped to it
                 (lower it to drive the partition machine on tiny inputs, like
                 the reference tests' insertion_threshold=3)
    host_levels  drive recursion levels from the host with a per-level trace
                 (debug / measurement); the default runs the whole recursion
                 inside one CUDA graph with a device-side loop.
    reproducible place every tile's < and > runs by decoupled look-back, so
                 the layout of each level -- and with it the children's pivot
                 samples, the stats and the order of equal-key records -- is
                 identical run to run.  The default reserves each tile's
                 ranges with one atomic instead: sorted keys are the same,
                 the placement of equal-key payloads and the stage counts may
                 differ between runs.
    """

    fast_paths: bool = True
    max_depth: int = 0
    host_levels: bool = False
    small_threshold: int = 0
    reproducible: bool = False

    def __post_init__(self):
        if not (self.small_threshold == 0 or 1 <= self.small_threshold <= 40952):
            raise ValueError("small_threshold must be 0 (auto) or in [1, 40952]")
        if not (self.max_depth == 0 or 2 <= self.max_depth <= 190):
            raise ValueError("max_depth must be 0 (auto) or in [2, 190]")


DEFAULT_GPU_CONFIG = GpuConfig()
