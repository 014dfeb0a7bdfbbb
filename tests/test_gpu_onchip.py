"""GPU parity around the on-chip sort classes (tsq_small.cuh): segments of
<= 4096 keys (256-thread class), 4097 .. 16384 four-byte keys / 8192 records
and 8-byte keys (512-thread class) and 16385 .. 32768 four-byte keys
(1024-thread class) finish in shared memory with an LSD radix sort over the
segment's key range.  Sizes straddle every class boundary and the partition
pass's tile sizes; key ranges straddle the radix digit and item-form
boundaries; the inputs cover the shapes the reference battery exercises
(datagen.py:106-198): uniform, few distinct, all equal, sorted, reversed,
organ pipe, sawtooth, two sorted runs, and -0.0 / NaN for floats.  Bar:
bit-exact against the CPU oracle (oracle/), the reference's algorithm
restated in C.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SIZES32 = [4087, 4088, 4089, 4095, 4096, 4097, 5000, 8183, 8184, 8185, 8191, 8192, 8193, 12288,
           16375, 16376, 16377, 16385, 32759, 32760, 32761, 32768, 65536, 200003]
SIZES64 = [4087, 4088, 4089, 4096, 4097, 8183, 8184, 8185, 8192, 12000, 16376, 16377, 16385, 40000]


def _shapes(n, rng, dtype):
    dt = np.dtype(dtype)
    if dt.kind == "f":
        base = rng.standard_normal(n)
    else:
        info = np.iinfo(dt)
        base = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    i = np.arange(n)
    return {
        "uniform": base.astype(dt),
        "few3": rng.integers(0, 3, n).astype(dt),
        "few100": rng.integers(0, 100, n).astype(dt),
        "equal": np.full(n, 7, dtype=dt),
        "sorted": np.sort(base).astype(dt),
        "reversed": np.sort(base)[::-1].astype(dt),
        "organ": np.minimum(i, n - 1 - i).astype(dt),
        "saw": (i % 517).astype(dt),
        "two_runs": np.concatenate([np.sort(base[: n // 2]), np.sort(base[n // 2:])]).astype(dt),
    }


def _check(x, sorter):
    d = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    st = sorter.sort_with_stats(d)
    want = x.copy()
    O.sort(want, seed=1, threads=4)
    got = d.cpu().numpy()
    assert got.tobytes() == want.tobytes()
    return st


@pytest.fixture(scope="module")
def sorter(cuda_ok):
    return T.Sorter(seed=3)


@pytest.mark.parametrize("n", SIZES32)
@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.float32])
def test_onchip_4byte(sorter, n, dtype):
    rng = np.random.default_rng(n * 7 + 1)
    for name, x in _shapes(n, rng, dtype).items():
        _check(x, sorter)


@pytest.mark.parametrize("n", SIZES64)
@pytest.mark.parametrize("dtype", [np.int64, np.uint64, np.float64])
def test_onchip_8byte(sorter, n, dtype):
    rng = np.random.default_rng(n * 11 + 5)
    for name, x in _shapes(n, rng, dtype).items():
        _check(x, sorter)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_onchip_float_total_order(sorter, dtype):
    """-0.0 before +0.0, NaNs at the ends (the device's IEEE total order;
    the reference comparator cannot order them, so only the order-preserving
    encoding is checked here, against numpy on the encoded bits)."""
    rng = np.random.default_rng(99)
    n = 20000
    x = rng.standard_normal(n).astype(dtype)
    x[rng.choice(n, 500, replace=False)] = -0.0
    x[rng.choice(n, 500, replace=False)] = 0.0
    d = torch.from_numpy(x.copy()).cuda()
    sorter.sort(d)
    got = d.cpu().numpy()
    ut = np.uint32 if dtype == np.float32 else np.uint64
    bits = x.view(ut)
    sign = np.array(1, dtype=ut) << ut(8 * x.itemsize - 1)
    enc = np.where(bits & sign, ~bits, bits | sign)
    want = np.sort(enc)
    dec = np.where(want & sign, want & ~sign, ~want).astype(ut).view(dtype)
    assert got.tobytes() == dec.tobytes()


def test_onchip_whole_array_in_one_segment(sorter):
    """n <= the on-chip cut: the root segment goes straight on chip."""
    rng = np.random.default_rng(5)
    for n in (2, 4088, 4089, 4096, 4097, 6000, 8184, 8185, 16376, 16377, 40952):
        st = _check(rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32), sorter)
        assert st.gpu["levels"] == 0
    # (a class of S item slots takes segments of up to S - 8 keys)
    st = _check(rng.integers(-2**31, 2**31, 40953, dtype=np.int64).astype(np.int32), sorter)
    assert st.gpu["levels"] == 1
    for n, lv in ((8184, 0), (8185, 0), (16376, 0), (16377, 1)):
        st = _check(rng.integers(-2**62, 2**62, n, dtype=np.int64), sorter)
        assert st.gpu["levels"] == lv


@pytest.mark.parametrize("n", [16376, 16377, 16385, 20000, 32767, 32768, 32769, 40951, 40952, 40953, 100000])
@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.float32])
def test_onchip_1024_thread_class(n, dtype, cuda_ok):
    """The largest class (16377 .. 40952 four-byte keys): small_threshold at
    its capacity, sizes around both of its boundaries."""
    s = T.Sorter(seed=5, gpu=T.GpuConfig(small_threshold=40952))
    rng = np.random.default_rng(n * 3 + 2)
    for name, x in _shapes(n, rng, dtype).items():
        _check(x, s)


@pytest.mark.parametrize("bits", [1, 4, 5, 6, 10, 11, 15, 16, 17, 18, 19, 20, 21, 25, 26, 31, 32,
                                  33, 40, 49, 50, 51, 63, 64])
def test_onchip_key_range_bits(bits, cuda_ok):
    """The radix sort runs ceil(bits / 5) digit passes over key - min, in
    32-bit items while the range fits (records: with the index packed below
    the key up to 18 bits), else 64-bit items (records: index packed up to
    50 bits, else a side array).  Segments whose keys span exactly 2^bits
    values (min and max present), for keys and records, 4- and 8-byte keys,
    on-chip directly (n <= the cut) and after partition levels."""
    from conftest import assert_records_consistent
    rng = np.random.default_rng(bits)
    for dt in (np.int32, np.uint32, np.int64, np.uint64):
        nb = 8 * np.dtype(dt).itemsize
        if bits > nb:
            continue
        ut = np.uint32 if nb == 32 else np.uint64
        mask = (1 << bits) - 1
        # keys built in the order-preserving unsigned encoding, then decoded
        lo = int(rng.integers(0, (1 << nb) - mask, dtype=np.uint64)) if bits < nb else 0
        for n in (777, 5000, 30000, 200000):
            off = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + \
                rng.integers(0, 2, n, dtype=np.uint64)
            off &= np.uint64(mask)
            off[0], off[-1] = 0, mask
            u = (np.uint64(lo) + off).astype(ut)
            if np.dtype(dt).kind == "i":
                u ^= ut(1 << (nb - 1))
            keys = u.view(dt)
            rng.shuffle(keys)
            _check(keys, T.Sorter(seed=1))
            pay = np.arange(n, dtype=np.uint32)
            dk, dp = torch.from_numpy(keys.copy()).cuda(), torch.from_numpy(pay).cuda()
            T.Sorter(seed=1).sort(T.Records(dk, dp))
            assert_records_consistent(keys, dk.cpu().numpy(), dp.cpu().numpy(), np.sort(keys))


@pytest.mark.parametrize("dtype", [np.int64, np.uint64, np.float64, np.int32, np.uint32])
@pytest.mark.parametrize("n", [3000, 8192, 12000, 70001])
def test_onchip_records_item_forms(sorter, dtype, n):
    """Records: items are key - segment min with the index packed below it
    (32-bit items up to 18 bits of range, 64-bit items up to 50 bits), else
    (key, index) pairs; full-range keys, a narrow cluster and a mix of both
    exercise every form.  Keys bit-exact, payload a permutation
    consistent with the keys (BASELINE.json config 5)."""
    from conftest import assert_records_consistent
    rng = np.random.default_rng(n + 17)
    dt = np.dtype(dtype)
    if dt.kind == "f":
        wide = rng.standard_normal(n) * 1e300
        narrow = 1.0 + rng.integers(0, 50, n) * 1e-12
    else:
        info = np.iinfo(dt)
        wide = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        narrow = rng.integers(0, 100, n).astype(dt) + (info.max // 2 if dt.kind == "u" else 0)
    mixed = np.where(rng.random(n) < 0.5, wide, narrow)
    for keys in (wide.astype(dt), narrow.astype(dt), mixed.astype(dt)):
        pay = np.arange(n, dtype=np.uint32)
        dk = torch.from_numpy(keys.copy()).cuda()
        dp = torch.from_numpy(pay).cuda()
        sorter.sort(T.Records(dk, dp))
        want = keys.copy()
        O.sort(want, seed=1, threads=4)
        assert_records_consistent(keys, dk.cpu().numpy(), dp.cpu().numpy(), want)


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.float32, np.int64, np.uint64, np.float64])
@pytest.mark.parametrize("n", [2000, 8184, 16376, 40952])
def test_onchip_leading_bits_then_exchange(sorter, dtype, n):
    """A wide key range is sorted on its leading bits first and finished by
    odd-even exchange rounds; keys clustered inside a few leading-bit buckets
    (two outliers stretch the range, everything else differs in the low bits
    only) do not settle in the bounded rounds and take the full radix passes.
    Shapes: spread keys (few ties), one tight cluster, many small clusters,
    clusters of equal keys -- keys only and records, one on-chip segment each."""
    from conftest import assert_records_consistent
    rng = np.random.default_rng(n * 3 + 1)
    dt = np.dtype(dtype)
    if dt.kind == "f":
        spread = rng.standard_normal(n)
        cluster = 1.0 + rng.integers(0, 1 << 20, n) * np.finfo(dt).eps
        cluster[0], cluster[1] = -1e30, 1e30
        # (+ 0.0: no -0.0, which the reference's comparator cannot order)
        many = np.round(rng.standard_normal(n), 1) + 0.0 + rng.integers(0, 64, n) * np.finfo(dt).eps
        equal = np.round(rng.standard_normal(n), 1) + 0.0
    else:
        info = np.iinfo(dt)
        spread = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        mid = info.max // 2
        cluster = (mid + rng.integers(0, 1 << 12, n)).astype(dt)
        cluster[0], cluster[1] = info.min, info.max
        centres = rng.integers(info.min // 2, info.max // 2, 40, dtype=np.int64 if dt.kind == "i" else np.uint64)
        many = (centres[rng.integers(0, 40, n)] + rng.integers(0, 256, n).astype(centres.dtype)).astype(dt)
        equal = centres[rng.integers(0, 40, n)].astype(dt)
    for keys in (spread, cluster, many, equal):
        keys = np.ascontiguousarray(keys.astype(dt))
        _check(keys, sorter)
        if n <= 16376:
            pay = np.arange(n, dtype=np.uint32)
            dk = torch.from_numpy(keys.copy()).cuda()
            dp = torch.from_numpy(pay).cuda()
            sorter.sort(T.Records(dk, dp))
            want = keys.copy()
            O.sort(want, seed=1, threads=4)
            assert_records_consistent(keys, dk.cpu().numpy(), dp.cpu().numpy(), want)


def test_verification_tiles_after_partition_tiles(cuda_ok):
    """Regression: a level whose CTAs see a partition tile followed by many
    verification tiles (sorted / reversed fast paths) -- a small random
    segment next to a large sorted or reversed one, or thousands of 2-key
    segments with small_threshold=1 -- must not stall the partition
    pipeline (the stage held for the partition tile's bulk stores is
    released by the verification tiles)."""
    rng = np.random.default_rng(31)
    for n in (1 << 20, 1 << 22):
        for tail in ("asc", "desc"):
            head = rng.integers(0, 1000, n // 4).astype(np.int32)
            body = np.arange(1000, 1000 + n - n // 4, dtype=np.int32)
            if tail == "desc":
                body = body[::-1].copy()
            x = np.concatenate([head, body])
            d = torch.from_numpy(x.copy()).cuda()
            T.Sorter(seed=1).sort(d)
            assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()
    for dt in (np.int32, np.uint64):
        for kind in ("random", "nearly"):
            x = np.sort(rng.integers(0, 1 << 30, 20000).astype(dt))
            if kind == "random":
                rng.shuffle(x)
            else:
                a, b = rng.integers(0, x.size, 200), rng.integers(0, x.size, 200)
                x[a], x[b] = x[b], x[a]
            d = torch.from_numpy(x.copy()).cuda()
            T.Sorter(seed=3, gpu=T.GpuConfig(small_threshold=1)).sort(d)
            assert d.cpu().numpy().tobytes() == np.sort(x).tobytes()


def test_tiny_cut_stress_verification_tiles(cuda_ok):
    """Regression (race): with cuts of 1-3 keys the partition pass handles
    thousands of 2-3-key segments, many of them verification tiles
    (sorted / reversed fast paths).  Their stage must not go back to the
    producer before every consumer warp has read its meta -- a lagging warp
    used to pick up the next tile's kind and stall the pipeline (~1 in 300
    such sorts).  Keys bit-exact, records consistent."""
    rng = np.random.default_rng(2024)
    for trial in range(60):
        dt = [np.int32, np.uint64, np.float32, np.int64][trial % 4]
        n = int(rng.integers(2000, 60000))
        base = rng.integers(0, 1 << 20, n).astype(dt)
        shape = trial % 3
        if shape == 1:
            base = np.sort(base)
            k = max(1, n // 100)
            a, b = rng.integers(0, n, k), rng.integers(0, n, k)
            base[a], base[b] = base[b], base[a]
        elif shape == 2:
            i = np.arange(n)
            base = np.minimum(i, n - 1 - i).astype(dt)
        g = T.GpuConfig(small_threshold=int(rng.integers(1, 4)), reproducible=bool(trial & 4))
        d = torch.from_numpy(base.copy()).cuda()
        if trial % 5 == 0:
            from conftest import assert_records_consistent
            p = torch.arange(n, dtype=torch.int64).to(torch.uint32).cuda()
            T.Sorter(seed=trial + 1, gpu=g).sort(T.Records(d, p))
            assert_records_consistent(base, d.cpu().numpy(), p.cpu().numpy().astype(np.int64),
                                      np.sort(base))
        else:
            T.Sorter(seed=trial + 1, gpu=g).sort(d)
            assert d.cpu().numpy().tobytes() == np.sort(base).tobytes()
