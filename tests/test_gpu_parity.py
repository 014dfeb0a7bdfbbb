"""GPU parity: the sm_100a path (through libtsq_b200.so's C ABI) against the
pinned CPU oracle (oracle/) and the reference-produced golden hashes.

Bar: bit-exact keys; for records, keys bit-exact and the payload a
permutation consistent with the keys (BASELINE.json config 5).
"""

from __future__ import annotations

import hashlib
import itertools
import random

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from paper_1505_00558_b200 import stage
from conftest import assert_records_consistent, load_golden, reference_sort
from oracle import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

DTYPES = [np.int32, np.uint32, np.int64, np.uint64, np.float32, np.float64]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _oracle_sorted(keys, payload=None):
    k = keys.copy()
    p = None if payload is None else payload.copy()
    O.sort(k, p, seed=1, threads=4)
    return k, p


def _random(dtype, n, rng, vmax=None):
    dt = np.dtype(dtype)
    if dt.kind == "f":
        return rng.standard_normal(n).astype(dt)
    info = np.iinfo(dt)
    lo, hi = (info.min, info.max) if vmax is None else (max(info.min, 0), vmax)
    return rng.integers(lo, hi, n, dtype=dt, endpoint=True)


@pytest.fixture(scope="module", params=[False, True], ids=["reserve", "reproducible"])
def sorter(cuda_ok, request):
    # both placements: atomic range reservation (default) and look-back
    return T.Sorter(seed=1, gpu=T.GpuConfig(reproducible=request.param))


@pytest.mark.parametrize("n", [2, 3, 17, 100, 4095, 4096, 4097, 8192, 8193, 65536, 100003, 1 << 20])
def test_int32_sizes_vs_oracle(sorter, n):
    rng = np.random.default_rng(n)
    x = _random(np.int32, n, rng)
    d = _dev(x)
    sorter.sort(d)
    want, _ = _oracle_sorted(x)
    assert d.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [5000, 300001])
@pytest.mark.parametrize("vmax", [None, 3, 1000])
def test_dtypes_vs_oracle(sorter, dtype, n, vmax):
    rng = np.random.default_rng(7 + n)
    if np.dtype(dtype).kind == "f" and vmax is not None:
        x = rng.integers(0, vmax, n).astype(dtype)
    else:
        x = _random(dtype, n, rng, vmax)
    d = _dev(x)
    sorter.sort(d)
    want, _ = _oracle_sorted(x)
    assert d.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("rec", [r for r in load_golden("sorts.json") if r["n"] <= (1 << 16)],
                         ids=lambda r: f"{r['family']}-{r['n']}")
def test_families_vs_reference_hashes(sorter, rec):
    """Outputs hash-identical to the Python reference's own outputs
    (tests/golden/sorts.json, produced by tests/golden/make_golden.py)."""
    keys, payload = W.generate(rec["family"], rec["n"])
    if payload is None:
        d = _dev(keys)
        sorter.sort(d)
        assert W.sha16(d.cpu().numpy()) == rec["sorted_sha"]
    else:
        dk, dp = _dev(keys), _dev(payload)
        sorter.sort(T.Records(dk, dp))
        ko, po = dk.cpu().numpy(), dp.cpu().numpy()
        assert W.sha16(ko) == rec["sorted_sha"]
        assert_records_consistent(keys, ko, po, np.sort(keys))


@pytest.mark.parametrize("thr", [1, 3, 16, 4096, 8192])
def test_kat_and_exhaustive_small(cuda_ok, thr):
    """[5,3,5,1,5] KAT, exhaustive 3^8 multisets and a slice of 8!
    permutations (tests/test_core.py:28-57); small_threshold=3 drives the
    device partition machine on tiny inputs like the reference's
    insertion_threshold=3 low-cut config."""
    s = T.Sorter(seed=17, gpu=T.GpuConfig(small_threshold=thr))
    ar = [5, 3, 5, 1, 5]
    s.sort(ar)
    assert ar == [1, 3, 5, 5, 5]
    tups = list(itertools.product(range(3), repeat=8))
    if thr != 3:
        tups = tups[::7]
    for tup in tups:
        d = _dev(np.asarray(tup, dtype=np.int32))
        s.sort(d)
        assert d.cpu().tolist() == sorted(tup), tup
    perms = list(itertools.permutations(range(1, 9)))[:: (37 if thr == 3 else 401)]
    for perm in perms:
        d = _dev(np.asarray(perm, dtype=np.int32))
        s.sort(d)
        assert d.cpu().tolist() == list(range(1, 9)), perm


def test_hypothesis_style_small_alphabets(cuda_ok):
    rnd = random.Random(12)
    for trial in range(150):
        n = rnd.randint(0, 300)
        vals = [rnd.randint(0, rnd.choice([2, 6, 1000])) for _ in range(n)]
        thr = rnd.choice([1, 3, 8, 16, 4096])
        ar = list(vals)
        T.Sorter(seed=trial + 1, gpu=T.GpuConfig(small_threshold=thr)).sort(ar)
        assert ar == reference_sort(vals)


def test_python_list_and_numpy_containers(sorter):
    rnd = random.Random(2)
    vals = [rnd.randint(-10**12, 10**12) for _ in range(20000)]
    ar = list(vals)
    sorter.sort(ar)
    assert ar == sorted(vals) and all(type(v) is int for v in ar[:10])
    f = [rnd.random() for _ in range(9000)]
    g = list(f)
    sorter.sort(g)
    assert g == sorted(f)
    a = np.random.default_rng(3).integers(0, 50, 70000).astype(np.int32)
    b = a.copy()
    sorter.sort(b)
    assert np.array_equal(b, np.sort(a))
    pinned = torch.from_numpy(a.copy()).pin_memory()
    sorter.sort(pinned)
    assert np.array_equal(pinned.numpy(), np.sort(a))


def test_key_only_comparator_records(sorter):
    # reference tests/test_core.py:93-103
    rnd = random.Random(2)
    items = [(rnd.randint(0, 5), i) for i in range(20000)]
    ar = list(items)
    sorter.sort(ar, T.key_cmp)
    assert [x[0] for x in ar] == sorted(x[0] for x in items)
    assert sorted(ar) == sorted(items)


@pytest.mark.parametrize("keydt", [np.uint64, np.int32, np.float64])
@pytest.mark.parametrize("n", [3000, 5000, 1 << 20])
def test_records_payload_consistent(sorter, keydt, n):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << 10, n).astype(keydt)
    pay = np.arange(n, dtype=np.uint32)
    dk, dp = _dev(keys), _dev(pay)
    sorter.sort(T.Records(dk, dp))
    assert_records_consistent(keys, dk.cpu().numpy(), dp.cpu().numpy(), _oracle_sorted(keys)[0])


@pytest.mark.parametrize("dtype", [np.int32, np.uint64, np.float64])
def test_stage_law_partition_segment(cuda_ok, dtype):
    """One device partition pass around a given pivot obeys the stage law
    and returns new_l / new_r = the counts (core.py:944-967)."""
    rng = np.random.default_rng(5)
    for n in (1, 7, 4096, 4097, 123457, 1 << 20):
        for vmax in (3, 1000, None):
            x = _random(dtype, n, rng, vmax) if np.dtype(dtype).kind != "f" else \
                rng.integers(0, vmax or 10**6, n).astype(dtype)
            p = x[rng.integers(0, n)]
            out, nl, nr = stage.partition_segment(_dev(x), p.item())
            o = out.cpu().numpy()
            lo, eq, hi = int((x < p).sum()), int((x == p).sum()), int((x > p).sum())
            assert (nl, nr) == (lo - 1, n - hi)
            assert (o[:nl + 1] < p).all() and (o[nl + 1:nr] == p).all() and (o[nr:] > p).all()
            assert np.array_equal(np.sort(o), np.sort(x))


def test_stage_law_records(cuda_ok):
    rng = np.random.default_rng(9)
    n = 300000
    x = rng.integers(0, 50, n).astype(np.uint64)
    pay = np.arange(n, dtype=np.uint32)
    p = x[123]
    ok, op, nl, nr = stage.partition_segment(_dev(x), p.item(), payload=_dev(pay))
    ok, op = ok.cpu().numpy(), op.cpu().numpy()
    assert np.array_equal(x[op], ok)
    assert np.array_equal(np.sort(op), pay)
    assert (ok[:nl + 1] < p).all() and (ok[nl + 1:nr] == p).all() and (ok[nr:] > p).all()


def test_first_stage_contract_vs_reference(cuda_ok):
    """The reference's own first-stage (pivot, new_l, new_r) records: the
    device pass around the same pivot lands on the same bounds."""
    for case in load_golden("stages.json")[:60]:
        x = np.asarray(case["in"], dtype=np.int64)
        _, nl, nr = stage.partition_segment(_dev(x), case["pivot"])
        assert (nl, nr) == (case["new_l"], case["new_r"])


def test_select_pivot_flags(cuda_ok):
    n = 1 << 20
    asc = np.arange(n, dtype=np.int32)
    p, f = stage.select_pivot(_dev(asc), mitigation=False)
    assert f == 1 and abs(p - n // 2) <= n // 64
    p, f = stage.select_pivot(_dev(asc[::-1].copy()), mitigation=False)
    assert f == -1 and abs(p - n // 2) <= n // 64
    x = np.random.default_rng(1).integers(0, 10**9, n).astype(np.int64)
    p, f = stage.select_pivot(_dev(x), dran=1.3)
    assert f == 0 and bool((x == p).any())
    rank = (x < p).sum() / n
    assert 0.4 < rank < 0.6


def test_negative_zero_and_nan_total_order(sorter):
    x = np.array([0.0, -0.0, np.nan, -np.inf, 1.5, -1.5, np.inf, -0.0, 0.0] * 1000)
    d = _dev(x)
    sorter.sort(d)
    o = d.cpu().numpy()
    fin = o[~np.isnan(o)]
    assert (fin[1:] >= fin[:-1]).all()
    assert np.isnan(o[-1000:]).all() and np.isinf(o[-2000:-1000]).all()  # +NaN after +inf
    z = np.nonzero(fin == 0)[0]
    assert np.signbit(fin[z[: len(z) // 2]]).all() and not np.signbit(fin[z[len(z) // 2:]]).any()


def test_host_levels_trace_matches_graph(cuda_ok):
    x = np.random.default_rng(4).integers(-2**31, 2**31, 1 << 21, dtype=np.int64).astype(np.int32)
    a, b = _dev(x), _dev(x)
    s1 = T.Sorter(seed=3, gpu=T.GpuConfig(reproducible=True))
    st1 = s1.sort_with_stats(a)
    s2 = T.Sorter(seed=3, gpu=T.GpuConfig(host_levels=True, reproducible=True))
    st2 = s2.sort_with_stats(b)
    assert torch.equal(a, b)
    assert st1.stages == st2.stages and st1.max_depth == st2.max_depth
    tr = s2.last_level_trace
    assert len(tr) == st2.gpu["levels"] and tr[0]["segments"] == 1


def test_determinism_and_stats(cuda_ok):
    x = np.random.default_rng(6).integers(0, 10**6, 500000).astype(np.int32)
    a, b = _dev(x), _dev(x)
    g = T.GpuConfig(reproducible=True)
    st1 = T.Sorter(seed=77, gpu=g).sort_with_stats(a)
    st2 = T.Sorter(seed=77, gpu=g).sort_with_stats(b)
    assert torch.equal(a, b)
    assert st1.as_dict() == st2.as_dict()
    assert st1.element_writes == st1.array_writes + st1.scratch_writes
    assert st1.max_depth <= 3 * np.log2(500000)
    assert st1.temp_high_water >= 500000


def test_all_equal_single_stage(cuda_ok):
    # reference tests/test_core.py:347-353: one stage retires everything
    d = _dev(np.full(50000, 4, dtype=np.int32))
    st = T.Sorter(seed=1).sort_with_stats(d)
    assert (d.cpu().numpy() == 4).all()
    assert st.stages == 1


def test_temp_storage_retained_and_freed(cuda_ok):
    s = T.Sorter(seed=1)
    s.sort(_dev(np.arange(10000, 0, -1, dtype=np.int32)))
    cap, allocs = s.temp.capacity, s.temp.alloc_count
    assert cap >= 10000 and allocs == 1
    s.sort(_dev(np.arange(5000, dtype=np.int32)))
    assert s.temp.capacity == cap and s.temp.alloc_count == 1
    s.free_temp_storage()
    assert s.temp.capacity == 0
    s.sort(_dev(np.arange(3000, 0, -1, dtype=np.int32)))
    assert s.temp.alloc_count == 2


def test_allocation_failure_leaves_array_untouched(cuda_ok):
    # reference tests/test_core.py:161-179 fault injection
    s = T.Sorter(seed=1)

    class Boom:
        capacity = 0
        alloc_count = 0
        device = 0

        def ensure(self, *a, **k):
            raise T.TempAllocationError("no memory")

        def workspace(self):
            raise AssertionError("must not be reached")

        def release(self):
            pass

    s.temp = Boom()
    ar = [3, 1, 2] * 20
    snap = list(ar)
    with pytest.raises(T.TempAllocationError):
        s.sort(ar)
    assert ar == snap
    d = _dev(np.asarray(snap, dtype=np.int32))
    with pytest.raises(T.TempAllocationError):
        s.sort(d)
    assert d.cpu().tolist() == snap


def test_real_allocation_failure_maps_to_temp_allocation_error(cuda_ok):
    from paper_1505_00558_b200 import _native as N
    ws = N.Workspace(0)
    st = ws.reserve((1 << 31) - 1024, N.TSQ_U64, N.TSQ_U32)
    # ~2^31 * 16 B is far beyond 180 GB only if it fails; either outcome is legal
    assert st in (N.TSQ_OK, N.TSQ_ERR_ALLOC)


def test_module_level_api(cuda_ok):
    T.free_temp_storage()
    ar = [random.Random(3).randint(0, 99) for _ in range(60)]
    T.sort(ar)
    assert ar == sorted(ar)
    st = T.sort_with_stats(ar, config=T.SortConfig(mitigation_enabled=False))
    assert ar == sorted(ar) and st.stages == 0
    T.free_temp_storage()


@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("dtype", [np.int32, np.uint64, np.float64])
def test_depth_guard_bisects_key_bounds(cuda_ok, dtype, payload):
    """Beyond GpuConfig.max_depth segments split at the midpoint of their key
    bounds: the sort finishes bit-exact instead of raising (the reference's
    _range always finishes, core.py:1643-1728)."""
    rng = np.random.default_rng(2)
    x = _random(dtype, 1 << 22, rng)
    s = T.Sorter(seed=1, gpu=T.GpuConfig(max_depth=2))
    d = _dev(x)
    if payload:
        p = _dev(np.arange(x.size, dtype=np.uint32))
        st = s.sort_with_stats(T.Records(d, p))
        assert_records_consistent(x, d.cpu().numpy(), p.cpu().numpy(), _oracle_sorted(x)[0])
    else:
        st = s.sort_with_stats(d)
        assert d.cpu().numpy().tobytes() == _oracle_sorted(x)[0].tobytes()
    assert st.gpu["bisected"] > 0 and st.gpu["error_flags"] == 0


def test_sample_position_adversary(cuda_ok):
    """The smallest keys placed at every position the root's pivot sampling
    reads (any jitter), n = 2^24: no DepthExceededError, no TsqError,
    bit-exact output."""
    n = 1 << 24
    rng = np.random.default_rng(9)
    x = rng.permutation(n).astype(np.int32) + 4096
    # the positions the root's 1023 strided samples read, jittered by the
    # sorter's first dran exactly as the sampling kernel computes them
    S = 1023
    rng_m = T.MitigationRng(1)
    rng_m.next()
    step = (n - 1) / (S - 1)
    shift = int(np.floor((rng_m.dran - 1.0) * step * 0.5))
    i = np.arange(S)
    pos = np.floor(i * step).astype(np.int64)
    pos[-1] = n - 1
    interior = (i != 0) & (i != S // 2) & (i != S - 1)
    pos[interior] = np.clip(pos[interior] + shift, 0, n - 1)
    hits = np.unique(pos)
    x[hits] = np.arange(hits.size, dtype=np.int32) - hits.size
    d = _dev(x)
    st = T.Sorter(seed=1).sort_with_stats(d)
    assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
    assert st.gpu["error_flags"] == 0


def test_queue_drain_rounds(cuda_ok, monkeypatch):
    """With the smallest queues the flush rule allows, the level loop drains
    the on-chip and run queues mid-recursion (outer graph loop) -- results
    unchanged, no capacity error."""
    monkeypatch.setenv("TSQ_DEBUG_MIN_QUEUES", "1")
    rng = np.random.default_rng(12)
    for hl in (False, True):
        x = rng.integers(0, 5000, 1 << 21).astype(np.int32)
        d = _dev(x)
        s = T.Sorter(seed=1, gpu=T.GpuConfig(small_threshold=64, host_levels=hl))
        st = s.sort_with_stats(d)
        assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
        assert st.gpu["flushes"] > 0 and st.gpu["error_flags"] == 0
        k = rng.integers(0, 300, 1 << 20).astype(np.uint64)
        dk, dp = _dev(k), _dev(np.arange(k.size, dtype=np.uint32))
        st = s.sort_with_stats(T.Records(dk, dp))
        assert_records_consistent(k, dk.cpu().numpy(), dp.cpu().numpy(), np.sort(k))
        assert st.gpu["flushes"] > 0
        s.free_temp_storage()


def test_last_status_without_stats(cuda_ok):
    """tsq_sort with stats == NULL returns without a sync;
    tsq_workspace_last_status reports the outcome."""
    import ctypes
    from paper_1505_00558_b200 import _native as N
    x = np.random.default_rng(3).integers(-2**31, 2**31, 1 << 20, dtype=np.int64).astype(np.int32)
    d = _dev(x)
    ws = N.Workspace(0)
    stream = torch.cuda.current_stream().cuda_stream
    st = N.lib().tsq_sort(ctypes.c_void_p(d.data_ptr()), None, d.numel(), N.TSQ_I32, N.TSQ_NONE,
                          None, ws.handle, ctypes.c_void_p(stream), None)
    assert st == N.TSQ_OK
    assert N.lib().tsq_workspace_last_status(ws.handle, ctypes.c_void_p(stream)) == N.TSQ_OK
    assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()


def test_sort_many_pipeline(cuda_ok):
    """Batch of host arrays sorted in place through the copy/sort pipeline."""
    rng = np.random.default_rng(11)
    sizes = [1 << 20, 3, 100003, 1 << 18, 0, 1]
    arrays = [rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32) for n in sizes]
    hosts = [torch.from_numpy(a.copy()).pin_memory() for a in arrays]
    stats = T.sort_many(hosts)
    assert len(stats) == len(hosts)
    for h, a in zip(hosts, arrays):
        assert np.array_equal(h.numpy(), np.sort(a))
    # numpy (pageable) arrays too, results in place
    nps = [a.copy() for a in arrays[:3]]
    T.Sorter(seed=2).sort_many(nps)
    for h, a in zip(nps, arrays):
        assert np.array_equal(h, np.sort(a))
    with pytest.raises(TypeError):
        T.sort_many([np.zeros(4, np.int32), np.zeros(4, np.int64)])
    with pytest.raises(TypeError):
        T.sort_many([torch.zeros(4, dtype=torch.int32, device="cuda")])


@pytest.mark.parametrize("keydt", [np.uint64, np.uint32, np.float64])
def test_reproducible_records_payload_order(cuda_ok, keydt):
    """GpuConfig(reproducible=True): the decoupled look-back placement makes
    every level's layout, and so the order of equal-key payloads, identical
    run to run (C5-style heavy duplication, both on-chip item forms)."""
    rng = np.random.default_rng(11)
    n = 1 << 20
    keys = rng.integers(0, 1 << 12, n).astype(keydt)
    outs = []
    for _ in range(2):
        dk, dp = _dev(keys), _dev(np.arange(n, dtype=np.uint32))
        T.Sorter(seed=5, gpu=T.GpuConfig(reproducible=True)).sort(T.Records(dk, dp))
        outs.append((dk.cpu().numpy(), dp.cpu().numpy()))
    assert outs[0][0].tobytes() == outs[1][0].tobytes() == np.sort(keys).tobytes()
    assert np.array_equal(outs[0][1], outs[1][1])
    assert_records_consistent(keys, outs[0][0], outs[0][1], np.sort(keys))


@pytest.mark.parametrize("dtype", [np.int32, np.uint64, np.float64])
@pytest.mark.parametrize("n", [100000, 100001, 100004, 1 << 20])
@pytest.mark.parametrize("payload", [False, True], ids=["keys", "records"])
def test_reversed_input_mirror_swap(cuda_ok, dtype, n, payload):
    """A strictly descending input is verified and reversed in place
    (_reversed_handler, core.py:1294-1556): mirror pairs of 16-byte vectors when
    the run is vector-aligned (n a multiple of 8 / 4), single keys otherwise;
    an offset view takes the aligned copy."""
    x = np.arange(n, 0, -1).astype(dtype)
    pay = np.arange(n, dtype=np.uint32)
    for off in (0, 1):
        dk, dp = _dev(x)[off:], _dev(pay)[off:]
        st = T.Sorter(seed=1).sort_with_stats(T.Records(dk, dp) if payload else dk)
        assert st.gpu["reversed_bypass"] == 1 and st.gpu["levels"] == 1
        want = np.sort(x[off:])
        assert dk.cpu().numpy().tobytes() == want.tobytes()
        if payload:
            assert np.array_equal(dp.cpu().numpy(), pay[off:][::-1])


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64, np.float32])
@pytest.mark.parametrize("shape", ["ascending", "blocks", "two_runs", "organ_pipe"])
def test_structured_tiles_equal_lane_counts(cuda_ok, dtype, shape):
    """Inputs whose tiles fall whole on one side of the pivot (every lane of a
    consumer warp places the same number of keys: the column-wise slot dealing
    of the restage), with the fast paths off so that they are partitioned."""
    n = 300000
    rng = np.random.default_rng(5)
    base = np.arange(n, dtype=np.int64) - n // 2
    if shape == "blocks":
        b = base[: n - n % 4096].reshape(-1, 4096)
        base = np.concatenate([b[rng.permutation(b.shape[0])].reshape(-1), base[n - n % 4096:]])
    elif shape == "two_runs":
        base = np.concatenate([base[0::2], base[1::2]])
    elif shape == "organ_pipe":
        base = np.concatenate([base[0::2], base[1::2][::-1]])
    x = (base - base.min()).astype(dtype) if np.dtype(dtype).kind == "u" else base.astype(dtype)
    for repro in (False, True):
        d = _dev(x)
        T.Sorter(seed=1, gpu=T.GpuConfig(fast_paths=False, reproducible=repro)).sort(d)
        assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
