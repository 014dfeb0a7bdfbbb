import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1505_00558_b200 as T
rng = np.random.default_rng(1)
bad = 0
for n in [2, 5, 100, 4087, 4088, 4089, 8184, 8185, 16376, 16377, 20000, 32760, 32761, 40000, 65536, 200003, 1 << 20]:
    for off in (0, 1, 3):
        for hi in (100, 2**20, 2**31 - 1):
            a = rng.integers(-hi, hi, n + off, dtype=np.int64).astype(np.int32)
            d = torch.from_numpy(a).cuda()
            v = d[off:]
            T.Sorter(seed=3).sort(v)
            ok = np.array_equal(v.cpu().numpy(), np.sort(a[off:]))
            if not ok:
                bad += 1
                print("MISMATCH", n, off, hi)
print("bad", bad)
