"""The reference's adversarial input battery, restated as test
infrastructure (generators only; nothing here runs on the sort path).

Follows /root/reference/pkg/src/tsqsort/datagen.py: the Park-Miller
generator with modulus 2^31 (datagen.py:48-76), the seven distributions of
``generate`` (datagen.py:106-137) incl. ``_organ_pipes`` (140-155), the
reorderings of ``reorder`` / ``fort`` (158-202) and ``battery_specs``
(290-297).  Pinned against the reference's own outputs by
tests/golden/make_battery.py -> tests/golden/battery.json
(tests/test_api_cpu.py::test_battery_generators_match_reference).
"""

from __future__ import annotations

import numpy as np

DISTRIBUTIONS = ("sawtooth", "random", "stagger", "plateau", "shuffle", "hill", "organpipes")
REORDERINGS = ("identity", "sorted", "reversed", "fronthalfreversed", "backhalfreversed",
               "dither", "fort")
_M = 1 << 31


class _PM:
    """z <- 16807 z mod 2^31; a zero seed is replaced (datagen.py:62-64)."""

    def __init__(self, seed: int):
        seed = int(seed) % _M
        self.z = seed if seed != 0 else 123456789

    def raw(self) -> int:
        self.z = (16807 * self.z) % _M
        return self.z

    def rand2(self, lo: int, hi: int) -> int:
        return int(self.raw() / _M * (hi - lo + 1) + lo)


def _organ_pipes(rng: _PM, n: int, m: int, max_dist: int, add: int) -> list:
    out = [0] * n
    v1 = float(rng.rand2(1, m))
    i = 0
    while i < n:
        v2 = float(rng.rand2(1, m) + add)
        d = rng.rand2(1, max_dist)
        step = (v2 - v1) / d
        while d != 0 and i < n:
            out[i] = int(v1)
            i += 1
            v1 += step
            d -= 1
        v1 = v2
    return out


def _fort(a: np.ndarray, lo: int, hi: int, minl: int) -> None:
    # reverse [lo..hi], then both halves, down to minl (iterative)
    stack = [(lo, hi)]
    while stack:
        lo, hi = stack.pop()
        a[lo:hi + 1] = a[lo:hi + 1][::-1].copy()
        if hi - lo + 1 > minl:
            h = (lo + hi) >> 1
            stack.append((h + 1, hi))
            stack.append((lo, h))


def generate(distribution: str, reorder: str, n: int, arange: int, seed: int = 1,
             op_max_distance: int = 30, op_add: int = 0, fort_minl: int = 2) -> np.ndarray:
    m = arange
    rng = _PM(seed)
    i = np.arange(n, dtype=np.int64)
    if distribution == "sawtooth":
        a = i % m
    elif distribution == "random":
        a = np.array([rng.rand2(1, m) for _ in range(n)], dtype=np.int64)
    elif distribution == "stagger":
        a = (i * m + i) % n if n else i
    elif distribution == "plateau":
        a = np.minimum(i, m)
    elif distribution == "shuffle":
        a = np.zeros(n, dtype=np.int64)
        j, k = 0, 1
        for t in range(n):
            if rng.raw() % m == 0:
                j += 2
                a[t] = j
            else:
                k += 2
                a[t] = k
    elif distribution == "hill":
        half = n >> 1
        a = np.minimum(np.where(i < half, i, n - i), m)
    elif distribution == "organpipes":
        a = np.array(_organ_pipes(rng, n, m, op_max_distance, op_add), dtype=np.int64)
    else:
        raise ValueError(distribution)
    a = np.array(a, dtype=np.int64)
    if n:
        if reorder == "sorted":
            a.sort()
        elif reorder == "reversed":
            a = np.sort(a)[::-1].copy()
        elif reorder == "fronthalfreversed":
            a.sort()
            h = n // 2
            a[:h] = a[:h][::-1].copy()
        elif reorder == "backhalfreversed":
            a.sort()
            h = n // 2
            a[h:] = a[h:][::-1].copy()
        elif reorder == "dither":
            a += i % 5
        elif reorder == "fort":
            _fort(a, 0, n - 1, fort_minl)
        elif reorder != "identity":
            raise ValueError(reorder)
    return a


def battery_cells():
    """The 7 distributions x 6 reorderings of battery_specs (identity left
    out, datagen.py:290-297)."""
    for d in DISTRIBUTIONS:
        for r in REORDERINGS:
            if r != "identity":
                yield d, r
