"""Per-level trace of a host-driven sort (partition ms, algorithmic bytes,
segments, tiles) as JSON, one object per family (dev tool):
    python scripts/level_trace.py uniform:67108864 normal_f64:67108864 records:134217728"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_00558_b200 as T
import workloads as W

out = {}
for spec in sys.argv[1:]:
    fam, n = spec.split(":")
    keys, pay = W.generate(fam, int(n))
    d = torch.from_numpy(keys).cuda()
    p = torch.from_numpy(pay).cuda() if pay is not None else None
    s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
    for _ in range(2):
        d.copy_(torch.from_numpy(keys))
        if p is not None:
            p.copy_(torch.from_numpy(pay))
        st = s.sort_with_stats(T.Records(d, p) if p is not None else d)
    out[fam] = {"n": int(n), "levels": s.last_level_trace, "ms_total": st.gpu["ms_total"]}
print(json.dumps(out))
