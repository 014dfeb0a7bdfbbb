"""Device time of full-size sorts at several on-chip cuts (dev tool):
    python scripts/cut_sweep.py uniform:67108864 normal_f64:67108864 records:134217728"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1505_00558_b200 as T
import workloads as W

specs = sys.argv[1:] or ["uniform:67108864"]
for spec in specs:
    cuts = (8184, 12288, 16376) if spec.startswith("records") else (4088, 8184, 12288, 16376, 24576, 32760, 40952)
    if os.environ.get("TSQ_CUTS"):
        cuts = tuple(int(c) for c in os.environ["TSQ_CUTS"].split(","))
    fam, n = spec.split(":")
    n = int(n)
    keys, pay = W.generate(fam, n)
    src = torch.from_numpy(keys).cuda()
    d = torch.empty_like(src)
    psrc = torch.from_numpy(pay).cuda() if pay is not None else None
    p = torch.empty_like(psrc) if psrc is not None else None
    want = np.sort(keys)
    for cut in cuts:
        s = T.Sorter(seed=1, gpu=T.GpuConfig(small_threshold=cut))
        ms = []
        for i in range(5):
            d.copy_(src)
            if p is not None:
                p.copy_(psrc)
            st = s.sort_with_stats(T.Records(d, p) if p is not None else d)
            if i:
                ms.append(st.gpu["ms_total"])
        ms.sort()
        ok = bool(np.array_equal(d.cpu().numpy(), want))
        print(f"{fam} n=2^{n.bit_length() - 1} cut {cut:6d}: {ms[len(ms) // 2]:.3f} ms  "
              f"levels {st.gpu['levels']}  ok={ok}", flush=True)
        del s
        torch.cuda.empty_cache()
