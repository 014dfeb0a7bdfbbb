"""Device time of uniform int32 2^26 sorts at several on-chip cuts (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_00558_b200 as T
import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
keys, _ = W.generate("uniform", n)
src = torch.from_numpy(keys).cuda()
d = torch.empty_like(src)
for cut in (8192, 12288, 16384, 24576, 32768):
    s = T.Sorter(seed=1, gpu=T.GpuConfig(small_threshold=cut))
    ms = []
    for i in range(6):
        d.copy_(src)
        st = s.sort_with_stats(d)
        if i:
            ms.append(st.gpu["ms_total"])
    ms.sort()
    ok = torch.equal(d, torch.sort(src).values)
    print(f"n=2^{n.bit_length() - 1} cut {cut:6d}: {ms[len(ms) // 2]:.3f} ms  levels {st.gpu['levels']}  ok={ok}", flush=True)
