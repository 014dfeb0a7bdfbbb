"""Shared fixtures; mirrors the reference's tests/conftest.py helpers
(/root/reference/pkg/tests/conftest.py:16-52) for the GPU path."""

from __future__ import annotations

import functools
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["data"]


def cmp3(x, y):
    if x < y:
        return -1
    if x > y:
        return 1
    return 0


def reference_sort(values, cmp=cmp3):
    """Independent oracle of the reference tests: the library sort."""
    return sorted(values, key=functools.cmp_to_key(cmp))


def three_way_counts(values, pivot):
    v = np.asarray(values)
    return int((v < pivot).sum()), int((v == pivot).sum()), int((v > pivot).sum())


def assert_stage_law(snapshot, a, b, new_l, new_r, pivot):
    """<p left of new_l, ==p between, >p right of new_r
    (reference tests/conftest.py:37-45)."""
    s = np.asarray(snapshot)
    assert (s[a:new_l + 1] < pivot).all()
    assert (s[new_l + 1:new_r] == pivot).all()
    assert (s[new_r:b + 1] > pivot).all()


def assert_records_consistent(keys_in, keys_out, payload_out, expect_keys):
    """Keys bit-exact; payload a permutation of 0..n-1 whose keys agree with
    every output position (BASELINE.json config 5)."""
    n = keys_in.size
    assert keys_out.tobytes() == expect_keys.tobytes()
    assert np.array_equal(np.sort(payload_out), np.arange(n, dtype=payload_out.dtype))
    assert np.array_equal(keys_in[payload_out.astype(np.int64)], keys_out)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
