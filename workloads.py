"""Seeded synthetic inputs for the five BASELINE.json configs.

BASELINE.json names no public dataset; these generators follow SURVEY.md
§8(d) exactly (a fresh ``np.random.default_rng(150500558)`` per config) so
their SHA-256 prefixes match the ones recorded there.  Used by tests/ and
bench.py; not part of the sort path.
"""

from __future__ import annotations

import hashlib

import numpy as np

SEED = 150500558

# family -> (key dtype, has payload, BASELINE.json config index)
FAMILIES = {
    "uniform": (np.int32, False, 0),       # C1 (full int32 range)
    "few_distinct": (np.int32, False, 1),  # C2 (uniform in [0, 99])
    "ascending": (np.int32, False, 2),     # C3a
    "descending": (np.int32, False, 2),    # C3b
    "organ_pipe": (np.int32, False, 2),    # C3c
    "nearly_sorted": (np.int32, False, 2), # C3d
    "stair": (np.int32, False, 2),         # C3e
    "normal_f64": (np.float64, False, 3),  # C4
    "records": (np.uint64, True, 4),       # C5 (u64 key + u32 payload)
}

# the sizes BASELINE.json quotes each family at
FULL_N = {
    "uniform": 1 << 20, "few_distinct": 1 << 24, "ascending": 1 << 26,
    "descending": 1 << 26, "organ_pipe": 1 << 26, "nearly_sorted": 1 << 26,
    "stair": 1 << 26, "normal_f64": 1 << 26, "records": 1 << 27,
}


def generate(family: str, n: int, seed: int = SEED):
    """Return (keys, payload_or_None) for ``family`` at size ``n``."""
    rng = np.random.default_rng(seed)
    if family == "uniform":
        return rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32), None
    if family == "few_distinct":
        return rng.integers(0, 100, n, dtype=np.int32), None
    if family == "ascending":
        return np.arange(n, dtype=np.int32), None
    if family == "descending":
        return np.arange(n - 1, -1, -1, dtype=np.int32), None
    if family == "organ_pipe":
        # "1..n/2..1": every value in 1..n/2 twice
        h = n // 2
        return np.concatenate([np.arange(1, h + 1, dtype=np.int32),
                               np.arange(n - h, 0, -1, dtype=np.int32)]), None
    if family == "nearly_sorted":
        a = np.arange(n, dtype=np.int32)
        idx = rng.choice(n, n // 100, replace=False)
        for i in idx:
            j = rng.integers(n)
            a[i], a[j] = a[j], a[i]
        return a, None
    if family == "stair":
        return (np.arange(n) // 1024).astype(np.int32), None
    if family == "normal_f64":
        x = rng.standard_normal(n)
        k = n // 100
        dst = rng.choice(n, k, replace=False)
        x[dst] = x[rng.integers(0, n, k)]
        assert not np.isnan(x).any()
        x[np.signbit(x) & (x == 0)] = 0.0
        return x, None
    if family == "records":
        keys = rng.integers(0, 2**20, n, dtype=np.uint64)
        return keys, np.arange(n, dtype=np.uint32)
    if family == "records_u32":  # (not a BASELINE config: 32-bit-key records, dev sweeps)
        keys = rng.integers(0, 2**20, n, dtype=np.uint64).astype(np.uint32)
        return keys, np.arange(n, dtype=np.uint32)
    raise KeyError(f"unknown family {family!r}; valid: {', '.join(FAMILIES)}")


def sha16(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:16]
