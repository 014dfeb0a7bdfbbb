"""Generate tests/golden/*.json by running the Python reference itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py [--full]

Everything written here is an OUTPUT of the reference (tsqsort 0.1.0,
/root/reference/pkg/src/tsqsort) on inputs that tests/ can regenerate from
seeds with numpy; no reference source is copied.  tests/test_oracle.py pins
the C restatement (oracle/) against these vectors, and the GPU parity tests
compare against the pinned oracle and these hashes.

``--full`` also runs the reference at BASELINE.json's full size for C1
(2^20) and C2 (2^24) (about a minute) and records the output hashes.
"""

from __future__ import annotations

import argparse
import functools
import hashlib
import itertools
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import tsqsort  # noqa: E402  (the reference, imported in place)
from tsqsort import SortConfig, Sorter  # noqa: E402
from tsqsort.pivot import MitigationRng, select_pivot  # noqa: E402
from tsqsort.smallsort import insertion_sort  # noqa: E402

import workloads as W  # noqa: E402


def cmp3(x, y):
    return -1 if x < y else (1 if x > y else 0)


def sha_list(values, dtype) -> str:
    return W.sha16(np.asarray(values, dtype=dtype))


# --- RNG (pivot.py:25-54) ---------------------------------------------------
def gen_rng():
    out = []
    for seed in (1, 2, 7, 12345, 2**31 - 1, W.SEED, 2**40 + 3):
        r = MitigationRng(seed)
        seq = []
        for _ in range(25):
            r.next()
            seq.append([r.zgen, r.dran, r.dran2])
        out.append({"seed": seed, "seq": seq})
    return out


# --- select_pivot ladder (pivot.py:205-248) ---------------------------------
def pivot_input(case):
    rng = np.random.default_rng(case["seed"])
    n_tot = case["n"] + 2 * case["pad"]
    kind = case["kind"]
    if kind == "random":
        return rng.integers(0, case["vmax"], n_tot, dtype=np.int64)
    if kind == "ascending":
        return np.arange(n_tot, dtype=np.int64)
    if kind == "descending":
        return np.arange(n_tot, 0, -1, dtype=np.int64)
    if kind == "equal":
        return np.full(n_tot, 7, dtype=np.int64)
    raise KeyError(kind)


def gen_pivot():
    cases = []
    sizes = [3, 4, 5, 6, 9, 16, 17, 40, 69, 70, 71, 72, 100, 333, 599, 600,
             601, 602, 1000, 4097, 59999, 60000, 60001, 60002, 100000, 250007]
    cid = 0
    for n in sizes:
        for kind in ("random", "ascending", "descending", "equal"):
            for mitig in (True, False):
                for small in ((True, False) if n <= 80 else (True,)):
                    for zseed in ((1, 99991) if kind == "random" else (5,)):
                        cid += 1
                        case = {"n": n, "pad": 3, "kind": kind,
                                "vmax": [4, 1000, 10**9][cid % 3],
                                "seed": 1000 + cid, "mitigation": mitig,
                                "medof3_small": small, "rng_seed": zseed}
                        base = pivot_input(case)
                        ar = base.tolist()
                        cfg = SortConfig(mitigation_enabled=mitig,
                                         medof3_small_enabled=small)
                        r = MitigationRng(zseed)
                        r.next()
                        tally = [0, 0, 0]
                        a = case["pad"]
                        b = a + n - 1
                        dec = select_pivot(ar, a, b, cfg, r, cmp3, tally)
                        after = np.asarray(ar, dtype=np.int64)
                        changed = np.nonzero(after != base)[0]
                        case.update({
                            "a": a, "b": b, "dran": r.dran,
                            "pivot": int(dec.pivot), "pi": int(dec.pi),
                            "flag": int(dec.order_flag), "tally": tally,
                            "changed_idx": changed.tolist(),
                            "changed_val": after[changed].tolist(),
                        })
                        cases.append(case)
    return cases


# --- insertion sort (smallsort.py:12-47) ------------------------------------
def gen_insertion():
    rnd = random.Random(5)
    out = []
    for _ in range(200):
        n = rnd.randint(0, 24)
        vals = [rnd.randint(0, rnd.choice([2, 9, 1000])) for _ in range(n)]
        ar = list(vals)
        tally = [0, 0, 0]
        insertion_sort(ar, 0, len(ar) - 1, cmp3, tally)
        out.append({"in": vals, "out": ar, "tally": tally})
    return out


# --- first-stage contract (core.py:944-967 via stage_hook 1707-1708) --------
def gen_stages():
    rnd = random.Random(31)
    out = []
    for trial in range(120):
        n = rnd.randint(17, 1200)
        vmax = rnd.choice([3, 30, 10**6])
        vals = [rnd.randint(0, vmax) for _ in range(n)]
        first = {}

        def hook(a, b, nl, nr, p, first=first):
            if not first:
                first.update(a=a, b=b, new_l=nl, new_r=nr, pivot=int(p))

        s = Sorter(seed=trial + 1)
        s.stage_hook = hook
        ar = list(vals)
        s.sort(ar)
        out.append({"in": vals, "seed": trial + 1, **first})
    return out


# --- whole sorts (Sorter.sort_with_stats, core.py:1586-1614) ----------------
SMALL_SORT_SIZES = {"uniform": [1 << 12, 1 << 16], "few_distinct": [1 << 14],
                    "ascending": [1 << 14], "descending": [1 << 14],
                    "organ_pipe": [1 << 14], "nearly_sorted": [1 << 14],
                    "stair": [1 << 14], "normal_f64": [1 << 14],
                    "records": [1 << 14]}


def reference_sort_family(family, n):
    keys, payload = W.generate(family, n)
    dtype = keys.dtype
    t0 = time.perf_counter()
    if payload is None:
        ar = keys.tolist()
        t1 = time.perf_counter()
        stats = Sorter(seed=1).sort_with_stats(ar)
        dt = time.perf_counter() - t1
        out_keys = np.asarray(ar, dtype=dtype)
        out_pay = None
    else:
        ar = list(zip(keys.tolist(), payload.tolist()))
        t1 = time.perf_counter()
        stats = Sorter(seed=1).sort_with_stats(
            ar, lambda x, y: cmp3(x[0], y[0]))
        dt = time.perf_counter() - t1
        out_keys = np.asarray([k for k, _ in ar], dtype=dtype)
        out_pay = np.asarray([p for _, p in ar], dtype=np.uint32)
    del t0
    rec = {"family": family, "n": n, "dtype": str(dtype),
           "input_sha": W.sha16(keys), "sorted_sha": W.sha16(out_keys),
           "ref_seconds": round(dt, 3), "stages": stats.stages,
           "max_depth": stats.max_depth, "comparisons": stats.comparisons}
    if out_pay is not None:
        # payload order among equal keys is the reference's own; record a
        # digest of the (key, payload) multiset check instead of its order
        ok = bool(np.array_equal(keys[out_pay], out_keys)) and \
            bool(np.array_equal(np.sort(out_pay), np.arange(n, dtype=np.uint32)))
        rec["payload_consistent"] = ok
        rec["payload_sha"] = W.sha16(out_pay)
    return rec


def gen_sorts(full: bool):
    out = []
    for fam, sizes in SMALL_SORT_SIZES.items():
        for n in sizes:
            out.append(reference_sort_family(fam, n))
    if full:
        for fam in ("uniform", "few_distinct"):
            out.append(reference_sort_family(fam, W.FULL_N[fam]))
    return out


def gen_exhaustive():
    cfg = SortConfig(insertion_threshold=3)
    h = hashlib.sha256()
    s = Sorter(cfg, seed=17)
    for perm in itertools.permutations(range(1, 9)):
        ar = list(perm)
        s.sort(ar)
        h.update(bytes(ar))
    perms = h.hexdigest()[:16]
    h = hashlib.sha256()
    s = Sorter(cfg, seed=23)
    for tup in itertools.product(range(3), repeat=8):
        ar = list(tup)
        s.sort(ar)
        h.update(bytes(ar))
    return {"perm8_sha": perms, "multiset3_8_sha": h.hexdigest()[:16],
            "kat": {"in": [5, 3, 5, 1, 5], "out": sorted([5, 3, 5, 1, 5])}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args()
    meta = {"reference": "tsqsort " + tsqsort.__version__,
            "generator": "tests/golden/make_golden.py"}
    jobs = {"rng.json": gen_rng, "pivot.json": gen_pivot,
            "insertion.json": gen_insertion, "stages.json": gen_stages,
            "exhaustive.json": gen_exhaustive,
            "sorts.json": lambda: gen_sorts(args.full)}
    for name, fn in jobs.items():
        t = time.perf_counter()
        data = {"meta": meta, "data": fn()}
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(f"{name}: {time.perf_counter() - t:.1f}s")


if __name__ == "__main__":
    main()
