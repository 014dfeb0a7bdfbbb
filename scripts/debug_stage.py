"""Dev tool: exercise partition_segment over sizes/dtypes and report mismatches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1505_00558_b200 import stage
rng = np.random.default_rng(5)
for dt in (np.uint64, np.int64, np.float64, np.int32):
    for n in (1, 7, 2047, 2048, 2049, 4095, 4096, 4097, 123457, 1 << 20):
        for vmax in (3, 1000, None):
            if np.dtype(dt).kind == "f":
                x = rng.integers(0, vmax or 10**6, n).astype(dt)
            else:
                info = np.iinfo(dt)
                x = rng.integers(0 if vmax else info.min, vmax or info.max, n, dtype=dt, endpoint=True)
            p = x[rng.integers(0, n)]
            out, nl, nr = stage.partition_segment(torch.from_numpy(x).cuda(), p.item())
            o = out.cpu().numpy()
            ok_law = (o[:nl + 1] < p).all() and (o[nl + 1:nr] == p).all() and (o[nr:] > p).all()
            ok_set = np.array_equal(np.sort(o), np.sort(x))
            if not (ok_law and ok_set):
                d = np.sort(o) != np.sort(x)
                bad = np.nonzero(np.isin(o, x, invert=True))[0]
                print("FAIL", np.dtype(dt).name, n, vmax, "law", ok_law, "set", ok_set,
                      "nl nr", nl, nr, "n_missing", int(d.sum()), "bad positions", bad[:10], o[bad[:5]])
print("done")
