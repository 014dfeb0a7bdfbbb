"""BASELINE.json configs at full size on the GPU.

Expected sorted-output hashes come from tests/golden/full.json: the oracle
(the C restatement pinned to the reference by tests/test_oracle.py) run
once per config at full size by tests/golden/make_full.py.  C1 (2^20) and
C2 (2^24) were also produced by the Python reference itself
(tests/golden/sorts.json, make_golden.py --full) and agree.  Records
additionally check the payload permutation.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from conftest import GOLDEN, load_golden
import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

with open(os.path.join(GOLDEN, "full.json")) as _f:
    FULL = {r["family"]: r for r in json.load(_f)["data"]}
SORTED_SHA = {fam: r["sorted_sha"] for fam, r in FULL.items()}


def test_full_golden_covers_every_config():
    assert set(FULL) == set(W.FULL_N)
    for fam, r in FULL.items():
        assert r["n"] == W.FULL_N[fam]


def test_reference_full_hashes_agree_with_oracle():
    for rec in load_golden("sorts.json"):
        if rec["n"] == W.FULL_N.get(rec["family"]):
            assert SORTED_SHA[rec["family"]] == rec["sorted_sha"]


@pytest.mark.parametrize("family", list(W.FAMILIES))
def test_full_size_family(cuda_ok, family):
    n = W.FULL_N[family]
    keys, payload = W.generate(family, n)
    assert W.sha16(keys) == FULL[family]["input_sha"]
    s = T.Sorter(seed=1)
    dk = torch.from_numpy(keys).cuda()
    if payload is None:
        st = s.sort_with_stats(dk)
        out = dk.cpu().numpy()
        assert W.sha16(out) == SORTED_SHA[family]
    else:
        dp = torch.from_numpy(payload).cuda()
        kin = dk.clone()
        st = s.sort_with_stats(T.Records(dk, dp))
        assert W.sha16(dk.cpu().numpy()) == SORTED_SHA[family]
        # payload is a permutation of 0..n-1 whose keys agree position-wise
        assert torch.equal(kin.view(torch.int64)[dp.long()], dk.view(torch.int64))
        seen = torch.zeros(n, dtype=torch.int32, device="cuda")
        seen.index_add_(0, dp.long(), torch.ones(n, dtype=torch.int32, device="cuda"))
        assert bool((seen == 1).all())
    # no O(n^2) blow-up: bounded recursion depth on every family
    assert st.max_depth <= 2 * np.log2(n) + 8, st.gpu
