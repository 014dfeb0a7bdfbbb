"""Mitigation generator (the reference's MitigationRng, pivot.py:25-54).

Park-Miller step ``z' = 16807 z mod 2^31`` advanced once per sort call;
``dran = 0.5 + z / 2^31`` in [0.5, 1.5) is handed to the device
pivot-sampling kernel, which shifts the interior sample positions by it.
"""

from __future__ import annotations

import time

R_A = 16807
R_M = 2147483648


class MitigationRng:
    __slots__ = ("zgen", "dran", "dran2")

    def __init__(self, seed: int | None = None):
        if seed is None:
            seed = time.time_ns()
        seed = int(seed) % R_M
        while seed == 0:
            seed = time.time_ns() % R_M
        self.zgen = seed
        self.dran = 1.0
        self.dran2 = 2.0

    def next(self) -> "MitigationRng":
        self.zgen = (R_A * self.zgen) % R_M
        self.dran = 0.5 + self.zgen / R_M
        self.dran2 = 1.0 + self.dran
        return self


def rng_next(rng: MitigationRng) -> MitigationRng:
    return rng.next()
