"""The reference's adversarial battery through the REGISTRY entry
(tests/test_acceptance.py:272-300, baselines.py:559-591): 7 distributions x
6 reorderings at n = 100000, arange = 500 (inputs from tests/battery.py,
pinned to the reference's generators), each sorted by
``REGISTRY["tristate"](ar, seed=1)`` and compared with the reference-sorted
hash; and the killer adversary's cooked input (datagen.py:205-276, cooked
against a first-element-pivot quicksort) replayed under 20 mitigation seeds
(test_acceptance.py:244-269) -- correct, and no quadratic blow-up: the
device recursion stays within a few levels of log2(n)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from battery import battery_cells, generate
from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _sha(a):
    return hashlib.sha256(np.asarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]


@pytest.mark.parametrize("cell", list(battery_cells()), ids=lambda c: f"{c[0]}-{c[1]}")
def test_battery_cell_through_registry(cuda_ok, cell):
    g = load_golden("battery.json")
    d, r = cell
    base = generate(d, r, g["n"], g["arange"], g["seed"])
    assert _sha(base) == g["cells"][f"{d}/{r}"]["input_sha"]
    ar = base.tolist()
    st = T.REGISTRY["tristate"](ar, seed=1)
    assert _sha(ar) == g["cells"][f"{d}/{r}"]["sorted_sha"]
    # device tensor, both placements
    for rep in (False, True):
        x = torch.from_numpy(base.copy()).cuda()
        T.Sorter(seed=1, gpu=T.GpuConfig(reproducible=rep)).sort(x)
        assert _sha(x.cpu().numpy()) == g["cells"][f"{d}/{r}"]["sorted_sha"]
    assert st.max_depth <= 64


def test_killer_cooked_input_replay(cuda_ok):
    g = load_golden("battery.json")["killer"]
    cooked = np.asarray(g["cooked"], dtype=np.int64)
    n = cooked.size
    want = np.sort(cooked)
    for seed in range(1, 21):
        x = torch.from_numpy(cooked.copy()).cuda()
        st = T.Sorter(seed=seed).sort_with_stats(x)
        assert np.array_equal(x.cpu().numpy(), want)
        assert st.max_depth <= int(np.log2(n)) + 8
