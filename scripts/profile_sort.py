"""Sort one workload a few times (for ncu captures of the device kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1505_00558_b200 as T
import workloads as W

fam = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 26)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
keys, pay = W.generate(fam, n)
src = torch.from_numpy(keys).cuda()
s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=os.environ.get("TSQ_HOST_LEVELS") == "1"))
for _ in range(reps):
    d = src.clone()
    if pay is not None:
        p = torch.from_numpy(pay).cuda()
        st = s.sort_with_stats(T.Records(d, p))
    else:
        st = s.sort_with_stats(d)
torch.cuda.synchronize()
print(fam, n, st.gpu["levels"], st.gpu["ms_total"])
