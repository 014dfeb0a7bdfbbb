"""Per-tile timeline of one partition level (profiling build, dev tool).

    TSQ_LIB=paper_1505_00558_b200/libtsq_b200_trace.so python scripts/trace_level.py [level]
Slots: 0 claim, 1 bulk load issued, 2 classify start, 3 aggregate
published, 4 inclusive published (look-back warp), 5 emit start, 6 offsets ready,
7 consumer emitted.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TSQ_LIB", os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "paper_1505_00558_b200", "libtsq_b200_trace.so"))
import numpy as np
import torch

import paper_1505_00558_b200 as T
from paper_1505_00558_b200 import _native as N
import workloads as W

level = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fam = sys.argv[2] if len(sys.argv) > 2 else "uniform"
n = int(sys.argv[3]) if len(sys.argv) > 3 else (1 << 26)
L = N.lib()
L.tsq_trace_set_level.argtypes = [ctypes.c_int]
L.tsq_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
keys, _ = W.generate(fam, n)
d = torch.from_numpy(keys).cuda()
s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
s.sort(d.clone())           # warm-up
L.tsq_trace_clear()
L.tsq_trace_set_level(level)
st = s.sort_with_stats(d)
tr = np.zeros(65536 * 8, dtype=np.uint64)
assert L.tsq_trace_copy(tr.ctypes.data, tr.nbytes) == 0
lv = s.last_level_trace[level]
nt = lv["tiles"]
tr = tr.reshape(-1, 8)[:nt].astype(np.int64)
t0 = tr[tr[:, 0] > 0, 0].min()
tr = np.where(tr > 0, tr - t0, -1)
print(f"level {level}: {lv}  tiles traced {nt}")
names = ["resolve(1-0)", "land+lag(2-1)", "count(3-2)", "lookback(4-3)", "agg->emit(6-3)",
         "lb->emit(6-4)", "stage+emit(7-6)", "total(7-0)"]
pairs = [(1, 0), (2, 1), (3, 2), (4, 3), (6, 3), (6, 4), (7, 6), (7, 0)]
for name, (a, b) in zip(names, pairs):
    ok = (tr[:, a] >= 0) & (tr[:, b] >= 0)
    x = (tr[ok, a] - tr[ok, b]) / 1000.0
    if x.size:
        print(f"  {name:18s} n={x.size:6d} mean {x.mean():8.2f} us  p50 {np.median(x):8.2f}  "
              f"p90 {np.percentile(x, 90):8.2f}  max {x.max():8.2f}")
span = tr[:, 7].max() / 1000.0
print(f"  level span {span:.1f} us; claims over time (us at 10/50/90% of tiles):",
      [round(float(np.percentile(tr[:, 0], q)) / 1000, 1) for q in (10, 50, 90)])
