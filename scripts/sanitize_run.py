"""Small sorts for compute-sanitizer runs (racecheck / synccheck / memcheck /
initcheck): every kernel of the sort path on inputs that reach the partition
pass (n above the on-chip cut), both on-chip item forms, records, the
sorted/reversed fast paths and a storage-offset view.  Exits non-zero on a
wrong result."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1505_00558_b200 as T

rng = np.random.default_rng(7)
host = os.environ.get("TSQ_HOST_LEVELS") == "1"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
cases = [
    ("int32", rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32), None),
    ("few", rng.integers(0, 50, n).astype(np.int32), None),
    ("asc", np.arange(n, dtype=np.int32), None),
    ("desc", np.arange(n, dtype=np.int32)[::-1].copy(), None),
    ("f64", rng.standard_normal(n), None),
    ("rec", rng.integers(0, 1 << 20, n).astype(np.uint64), np.arange(n, dtype=np.uint32)),
]
for name, x, p in cases:
    for cut in (0, 1024):
        g = T.GpuConfig(host_levels=host, small_threshold=cut)
        d = torch.from_numpy(x.copy()).cuda()
        if p is None:
            T.Sorter(seed=1, gpu=g).sort(d)
            ok = np.array_equal(d.cpu().numpy(), np.sort(x))
        else:
            dp = torch.from_numpy(p.copy()).cuda()
            T.Sorter(seed=1, gpu=g).sort(T.Records(d, dp))
            ko, po = d.cpu().numpy(), dp.cpu().numpy().astype(np.int64)
            ok = np.array_equal(ko, np.sort(x)) and np.array_equal(x[po], ko)
        print(name, cut, "ok" if ok else "WRONG", flush=True)
        if not ok:
            sys.exit(1)
x = rng.integers(-2**31, 2**31, n + 1, dtype=np.int64).astype(np.int32)
d = torch.from_numpy(x).cuda()[1:]
T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=host)).sort(d)
assert np.array_equal(d.cpu().numpy(), np.sort(x[1:]))
print("offset view ok")
