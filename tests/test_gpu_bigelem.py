"""GPU parity of late swapping for large elements (the reference's
bigelem.py, /root/reference/pkg/tests/test_bigelem.py): the handle sort runs
on the device, the elements move once (device rows: one gather pass through
tsq_apply_permutation)."""

from __future__ import annotations

import random

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from conftest import reference_sort

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_sort_indirect_example(cuda_ok):
    assert T.sort_indirect([30, 10, 20]).map == (1, 2, 0)


def test_sort_indirect_identity_on_sorted(cuda_ok):
    assert T.sort_indirect(list(range(10))).is_identity()


def test_sort_indirect_all_equal_is_bijection(cuda_ok):
    ar = [5] * 8
    perm = T.sort_indirect(ar)
    assert sorted(perm.map) == list(range(8))
    T.apply_permutation(ar, perm)
    assert ar == [5] * 8


def test_move_bound_and_composition_law(cuda_ok):
    rnd = random.Random(4)
    s = T.Sorter(seed=2)
    for _ in range(120):
        n = rnd.randint(0, 60)
        ar = [rnd.randint(0, 20) for _ in range(n)]
        perm = T.sort_indirect(ar, sorter=s)
        work = list(ar)
        moves = T.apply_permutation(work, perm)
        assert work == reference_sort(ar)
        assert moves <= n + n // 2


def test_late_swap_path_in_sorter(cuda_ok):
    """Large elements go through the handle sort transparently
    (test_bigelem.py:110-124; the key-only comparator is key_cmp here)."""
    rnd = random.Random(9)
    payload = bytes(400)
    items = [(rnd.randint(0, 50), payload, i) for i in range(300)]
    ar = list(items)
    stats = T.Sorter(seed=3).sort_with_stats(ar, T.key_cmp, element_size=400)
    assert [x[0] for x in ar] == sorted(x[0] for x in items)
    assert sorted(x[2] for x in ar) == list(range(300))
    assert stats.element_writes > 0


def test_small_elements_skip_late_path(cuda_ok):
    ar = [3, 1, 2]
    T.Sorter(seed=3).sort_with_stats(ar, element_size=8)
    assert ar == [1, 2, 3]


def test_reversal_moves_via_late_path(cuda_ok):
    n = 100
    ar = list(range(n))[::-1]
    perm = T.sort_indirect(ar)
    moves = T.apply_permutation(ar, perm)
    assert ar == sorted(range(n))
    assert moves <= 3 * (n // 2)


@pytest.mark.parametrize("n,width,dtype", [(1000, 100, torch.float32), (1 << 20, 100, torch.float32),
                                           (50001, 83, torch.uint8), (4097, 7, torch.int16)])
@pytest.mark.parametrize("device", ["cuda", "cpu"])
def test_device_rows_move_once(cuda_ok, n, width, dtype, device):
    """Records(keys, rows): keys sorted bit-exact, every row lands next to
    its key (rows carry their origin index), rows of any width / alignment,
    device-resident or host-resident."""
    rng = np.random.default_rng(n + width)
    keys = rng.integers(0, 1 << 16, n, dtype=np.int64).astype(np.int32)
    if dtype == torch.float32:
        rows = torch.arange(n * width, dtype=torch.float32).reshape(n, width)
        origin = lambda r: (r[:, 0] / width).round().long()
    elif dtype == torch.uint8:
        idx = torch.arange(n, dtype=torch.int64)
        rows = torch.zeros(n, width, dtype=torch.uint8)
        for b in range(4):
            rows[:, b] = ((idx >> (8 * b)) & 0xff).to(torch.uint8)
        origin = lambda r: sum(r[:, b].long() << (8 * b) for b in range(4))
    else:
        idx = torch.arange(n, dtype=torch.int64)
        rows = torch.zeros(n, width, dtype=torch.int16)
        rows[:, 0] = (idx & 0x7fff).to(torch.int16)
        rows[:, 1] = (idx >> 15).to(torch.int16)
        origin = lambda r: r[:, 0].long() + (r[:, 1].long() << 15)
    kd = torch.from_numpy(keys.copy()).to(device)
    rd = rows.clone().to(device)
    st = T.Sorter(seed=5).sort_with_stats(T.Records(kd, rd))
    ko = kd.cpu().numpy()
    assert ko.tobytes() == np.sort(keys).tobytes()
    org = origin(rd.cpu()).numpy()
    assert np.array_equal(np.sort(org), np.arange(n))
    assert np.array_equal(keys[org], ko)
    assert torch.equal(rd.cpu(), rows[torch.from_numpy(org)])
    assert st.element_writes > 0
