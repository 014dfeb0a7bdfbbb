import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W
for n in (1 << 18, 1 << 20, 1 << 22, 1 << 24):
    keys, _ = W.generate("uniform", n)
    src = torch.from_numpy(keys).cuda(); d = src.clone()
    row = []
    for thr in (2048, 4096, 8192, 12288, 16384):
        s = T.Sorter(seed=1, gpu=T.GpuConfig(small_threshold=thr))
        ms = []
        for i in range(12):
            d.copy_(src); torch.cuda.synchronize()
            st = s.sort_with_stats(d); ms.append(st.gpu["ms_total"])
        row.append((thr, round(sorted(ms[2:])[5], 4), st.gpu["levels"]))
    print(n, row, flush=True)
