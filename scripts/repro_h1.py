import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1505_00558_b200 as T
rng = np.random.default_rng(1)
x = rng.integers(-2**31, 2**31, 20000, dtype=np.int64).astype(np.int32)
d = torch.from_numpy(x).cuda()
T.Sorter(seed=3, gpu=T.GpuConfig(small_threshold=1, host_levels=True)).sort(d)
print("done", np.array_equal(d.cpu().numpy(), np.sort(x)))
