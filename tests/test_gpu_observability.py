"""Observability contract on the device path (row f4): ``Sorter.stage_hook``
is called as ``hook(a, b, new_l, new_r, pivot)`` once per stage with the
caller's array holding that stage's post-stage contents, and ``Sorter.trace``
receives the reference's stage-level event stream
(/root/reference/pkg/src/tsqsort/core.py:1676-1711; the reference tests
tests/test_core.py:60-69 and tests/test_instrument.py:77-94 are mirrored
here).  The device levels export one record per stage
(tsq_stage_record, include/tsq.h).
"""

from __future__ import annotations

import random

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from paper_1505_00558_b200.instrument import (HANDLER_ENTER, STAGE_END, STATE_ENTER,
                                              TraceSink)
from conftest import assert_stage_law

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# the partition machine on tiny inputs (the reference's low_cut_config)
LOW_CUT = T.GpuConfig(small_threshold=3)


def test_stage_three_way_law_random(cuda_ok):
    """tests/test_core.py:60-69: the law holds at every stage, on the list
    itself (the hook closes over `ar`)."""
    rnd = random.Random(31)
    calls = 0
    for trial in range(60):
        n = rnd.randint(4, 200)
        ar = [rnd.randint(0, rnd.choice([3, 30, 10**6])) for _ in range(n)]
        s = T.Sorter(seed=trial + 1, gpu=LOW_CUT)

        def hook(a, b, nl, nr, p):
            nonlocal calls
            calls += 1
            assert 0 <= a <= b < n and a - 1 <= nl < nr <= b + 1
            assert_stage_law(ar, a, b, nl, nr, p)

        s.stage_hook = hook
        s.sort(ar)
        assert ar == sorted(ar)
    assert calls > 60


@pytest.mark.parametrize("dtype", [np.int32, np.uint64, np.float64])
def test_stage_law_on_device_tensor(cuda_ok, dtype):
    rng = np.random.default_rng(5)
    x = rng.integers(0, 2000, 200000).astype(dtype)
    d = torch.from_numpy(x).cuda()
    seen = []

    def hook(a, b, nl, nr, p):
        seg = d[a:b + 1].cpu().numpy()
        assert_stage_law(seg, 0, b - a, nl - a, nr - a, p)
        seen.append((a, b))

    s = T.Sorter(seed=1, gpu=T.GpuConfig(small_threshold=512))
    s.stage_hook = hook
    st = s.sort_with_stats(d)
    assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
    assert len(seen) == st.stages and seen[0] == (0, x.size - 1)


def test_stage_hook_records_and_payload(cuda_ok):
    """(key, payload) tuples with key_cmp: the hook sees the list, payloads
    travel with their keys at every stage."""
    rnd = random.Random(8)
    ar = [(rnd.randint(0, 40), i) for i in range(3000)]
    s = T.Sorter(seed=2, gpu=T.GpuConfig(small_threshold=16))

    def hook(a, b, nl, nr, p):
        keys = [k for k, _ in ar]
        assert_stage_law(keys, a, b, nl, nr, p)
        assert sorted(i for _, i in ar) == list(range(3000))

    s.stage_hook = hook
    s.sort(ar, T.key_cmp)
    assert [k for k, _ in ar] == sorted(k for k, _ in ar)


def test_trace_stream_shape(cuda_ok):
    """tests/test_instrument.py:77-91."""
    sink = TraceSink()
    s = T.Sorter(seed=2, gpu=LOW_CUT)
    s.trace = sink
    rnd = random.Random(1)
    ar = [rnd.randint(0, 20) for _ in range(200)]
    s.sort(ar)
    assert ar == sorted(ar)
    kinds = sink.kinds()
    assert kinds, "trace must not be empty"
    assert kinds[-1] == STAGE_END
    assert sink.dump().splitlines()[-1].startswith(STAGE_END)
    assert sink.events[-1].payload == (0, 199, "root")
    assert STATE_ENTER in kinds
    # every stage end follows its state / handler entry
    ends = [e for e in sink.events[:-1] if e.kind == STAGE_END]
    enters = [e for e in sink.events if e.kind in (STATE_ENTER, HANDLER_ENTER)]
    assert len(ends) == len(enters) > 0


def test_trace_handlers_on_sorted_and_reversed(cuda_ok):
    for x, name in ((np.arange(1 << 18, dtype=np.int32), "sorted"),
                    (np.arange(1 << 18, 0, -1).astype(np.int32), "reversed")):
        sink = TraceSink()
        s = T.Sorter(seed=1)
        s.trace = sink
        d = torch.from_numpy(x).cuda()
        s.sort(d)
        assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
        ev = sink.events
        assert ev[0].kind == HANDLER_ENTER and ev[0].payload == (name, 0, x.size - 1)
        a, b, nl, nr = ev[1].payload
        assert ev[1].kind == STAGE_END and (a, b) == (0, x.size - 1)
        assert nl + 1 == nr - 1  # distinct keys: one == p


def test_trace_off_by_default(cuda_ok):
    s = T.Sorter(seed=2)
    assert s.trace is None and s.stage_hook is None


def test_hook_exception_propagates(cuda_ok):
    s = T.Sorter(seed=1, gpu=LOW_CUT)

    def hook(*args):
        raise KeyError("stop")

    s.stage_hook = hook
    with pytest.raises(KeyError):
        s.sort([5, 3, 5, 1, 5, 9, 2, 6])
