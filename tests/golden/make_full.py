"""Generate tests/golden/full.json: the oracle (oracle/, the C restatement of
the reference's sort path, itself pinned to reference-produced vectors by
tests/test_oracle.py) run once per BASELINE.json config at FULL size.

    python tests/golden/make_full.py [--threads N]

For every family of workloads.py at its BASELINE size: the SHA-256 prefix of
the generated input and of the oracle's sorted output (records: the keys'
hash, plus a check that the oracle's payload is a permutation consistent
with the keys), and the oracle's wall time.  tests/test_gpu_full.py compares
the GPU path's full-size outputs against these hashes; bench.py uses them to
verify every family it times.  C1 (2^20) and C2 (2^24) were also produced by
the Python reference itself (tests/golden/sorts.json); the script checks the
oracle agrees with those.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    O.build()
    ref = {}
    with open(os.path.join(HERE, "sorts.json")) as f:
        for rec in json.load(f)["data"]:
            ref[(rec["family"], rec["n"])] = rec["sorted_sha"]
    out = []
    for fam, n in W.FULL_N.items():
        keys, pay = W.generate(fam, n)
        in_sha = W.sha16(keys)
        k = keys.copy()
        p = None if pay is None else pay.copy()
        t0 = time.perf_counter()
        O.sort(k, p, seed=1, threads=args.threads)
        dt = time.perf_counter() - t0
        rec = {"family": fam, "n": n, "dtype": str(keys.dtype), "input_sha": in_sha,
               "sorted_sha": W.sha16(k), "oracle_s": round(dt, 3), "threads": args.threads}
        if p is not None:
            assert np.array_equal(np.sort(p), np.arange(n, dtype=np.uint32))
            assert np.array_equal(keys[p.astype(np.int64)], k)
            rec["payload"] = "permutation of 0..n-1 consistent with the keys"
        if (fam, n) in ref:
            assert ref[(fam, n)] == rec["sorted_sha"], fam
            rec["reference_sha"] = ref[(fam, n)]
        print(json.dumps(rec), flush=True)
        out.append(rec)
    doc = {"generator": "tests/golden/make_full.py",
           "source": "oracle/ C restatement (pinned to the reference by tests/test_oracle.py)",
           "cpu": cpu_model(), "data": out}
    with open(os.path.join(HERE, "full.json"), "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
