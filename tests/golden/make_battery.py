"""Generate tests/golden/battery.json by running the reference's own
generators (tsqsort.datagen, imported in place from /root/reference; build
container only) and its killer adversary (datagen.py:205-276) against its
first-element-pivot quicksort (baselines.py:183).  Outputs only: input
hashes of every battery cell (n = 100000, arange = 500, seed = 1 --
tests/test_acceptance.py:272-300) and the cooked killer input of n = 4096
(test_acceptance.py:244-247).

    python tests/golden/make_battery.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from tsqsort.baselines import fixed_pivot_qsort  # noqa: E402
from tsqsort.datagen import GenSpec, battery_specs, cook_input, generate  # noqa: E402


def sha16(values) -> str:
    return hashlib.sha256(np.asarray(values, dtype=np.int64).tobytes()).hexdigest()[:16]


def main():
    cells = {}
    for spec in battery_specs(100000, 500, seed=1):
        base = generate(spec)
        cells[f"{spec.distribution}/{spec.reorder}"] = {
            "input_sha": sha16(base), "sorted_sha": sha16(sorted(base))}
    small = {}
    for spec in battery_specs(1000, 7, seed=3):
        small[f"{spec.distribution}/{spec.reorder}"] = sha16(generate(spec))
    cooked = cook_input(lambda ar, cmp: fixed_pivot_qsort(ar, cmp), 4096)
    out = {"generator": "tsqsort.datagen (reference), battery_specs(n, arange, seed)",
           "n": 100000, "arange": 500, "seed": 1, "cells": cells,
           "small": {"n": 1000, "arange": 7, "seed": 3, "cells": small},
           "killer": {"n": 4096, "target": "baselines.fixed_pivot_qsort", "cooked": cooked}}
    with open(os.path.join(HERE, "battery.json"), "w") as f:
        json.dump({"data": out}, f)
    print(len(cells), "cells;", "killer", len(cooked))


if __name__ == "__main__":
    main()
