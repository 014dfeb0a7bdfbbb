"""Randomised GPU parity sweep (dev tool): random sizes, key types,
distributions, cut thresholds, placement modes and payloads, checked
against numpy (keys bit-exact under the device's total order; records:
payload a permutation consistent with the keys).

    python scripts/fuzz.py [cases] [seed]
    TSQ_FUZZ_TINY=1    cuts of 1-3 keys (the partition machine on tiny segments)
    TSQ_FUZZ_BIG=1     2^22 .. 2^25 keys
    TSQ_FUZZ_OFFSET=1  keys / payloads are CUDA views with a storage offset
    TSQ_LIB=...        e.g. the -DTSQ_DEBUG_CHECKS build (scripts/gpu_debug_checks.sh)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1505_00558_b200 as T

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1          # replay one case
host_levels = os.environ.get("TSQ_FUZZ_HOST_LEVELS") == "1"
rng = np.random.default_rng(seed)
DT = [np.int32, np.uint32, np.float32, np.int64, np.uint64, np.float64]


def keys_of(dt, n):
    kind = rng.integers(0, 9)
    d = np.dtype(dt)
    if d.kind == "f":
        base = rng.standard_normal(n) * (10.0 ** rng.integers(-3, 6))
    else:
        info = np.iinfo(d)
        base = rng.integers(info.min, info.max, n, dtype=d, endpoint=True)
    if kind == 1:
        base = rng.integers(0, int(rng.integers(1, 50)), n)
    elif kind == 2:
        base = np.sort(base)
    elif kind == 3:
        base = np.sort(base)[::-1]
    elif kind == 4:
        i = np.arange(n)
        base = np.minimum(i, n - 1 - i)
    elif kind == 5:
        base = np.sort(base)
        k = max(1, n // 100)
        a, b = rng.integers(0, n, k), rng.integers(0, n, k)
        base[a], base[b] = base[b], base[a]
    elif kind == 6:
        base = (np.arange(n) // int(rng.integers(1, 3000)))
    elif kind == 7:
        base = np.full(n, 3)
    return np.asarray(base).astype(dt), kind


def total_order_sorted(x):
    if x.dtype.kind != "f":
        return np.sort(x)
    ut = np.uint32 if x.itemsize == 4 else np.uint64
    bits = x.view(ut)
    sign = ut(1) << ut(8 * x.itemsize - 1)
    enc = np.where(bits & sign, ~bits, bits | sign).astype(ut)
    s = np.sort(enc)
    return np.where(s & sign, s & ~sign, ~s).astype(ut).view(x.dtype)


t0 = time.time()
fails = 0
for c in range(cases):
    dt = DT[rng.integers(0, len(DT))]
    n = int(rng.choice([rng.integers(2, 5000), rng.integers(5000, 70000),
                        rng.integers(70000, 3_000_000)]))
    if os.environ.get("TSQ_FUZZ_BIG") == "1":  # large inputs: 2^22 .. 2^25 keys
        n = int(rng.integers(1 << 22, 1 << 25))
    x, kind = keys_of(dt, n)
    thr = int(rng.choice([0, 0, 0, 1, 3, 16, 4088, 4096, 8184, 8192, 16376, 16384, 24576, 32768, 40952]))
    if os.environ.get("TSQ_FUZZ_TINY") == "1":  # stress: the partition machine down to tiny segments
        thr = int(rng.choice([1, 2, 3]))
    rep = bool(rng.integers(0, 2))
    pay = bool(rng.integers(0, 3) == 0)
    s = T.Sorter(seed=int(rng.integers(1, 1 << 30)),
                 gpu=T.GpuConfig(small_threshold=thr, reproducible=rep, host_levels=host_levels,
                                 fast_paths=os.environ.get("TSQ_FUZZ_NOFP") != "1"))
    if only >= 0 and c != only:
        continue
    off = int(rng.integers(1, 4)) if os.environ.get("TSQ_FUZZ_OFFSET") == "1" else 0
    # offset mode: the keys (and payload) are CUDA views with a storage offset
    d = torch.from_numpy(np.concatenate([x[:off], x]).copy()).cuda()[off:]
    print(f"case {c}: dtype={np.dtype(dt).name} n={n} kind={kind} thr={thr} rep={rep} pay={pay} "
          f"off={off}", flush=True)
    try:
        if pay:
            p = torch.arange(-off, n, dtype=torch.int64).to(torch.uint32).cuda()[off:]
            s.sort(T.Records(d, p))
            ko, po = d.cpu().numpy(), p.cpu().numpy().astype(np.int64)
            ok = ko.tobytes() == total_order_sorted(x).tobytes() and \
                np.array_equal(np.sort(po), np.arange(n)) and x[po].tobytes() == ko.tobytes()
        else:
            s.sort(d)
            ok = d.cpu().numpy().tobytes() == total_order_sorted(x).tobytes()
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", e)
    if not ok:
        fails += 1
        print(f"FAIL case {c}: dtype={np.dtype(dt).name} n={n} kind={kind} thr={thr} rep={rep} pay={pay}",
              flush=True)
print(f"fuzz: {cases} cases, {fails} failures, {time.time() - t0:.1f} s")
sys.exit(1 if fails else 0)
