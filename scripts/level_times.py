"""Per-level partition / schedule kernel times of one sort (host-driven levels) next to
the graph-mode total (dev tool): python scripts/level_times.py [family] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W

fam = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20)
keys, pay = W.generate(fam, n)
src = torch.from_numpy(keys).cuda()
psrc = torch.from_numpy(pay).cuda() if pay is not None else None
for hl in (True, False):
    s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=hl))
    ms = []
    for _ in range(6):
        d = src.clone()
        p = psrc.clone() if psrc is not None else None
        torch.cuda.synchronize()
        st = s.sort_with_stats(T.Records(d, p) if p is not None else d)
        ms.append(st.gpu["ms_total"])
    print(fam, n, "host_levels" if hl else "graph", "ms_total median", sorted(ms[1:])[2], "levels", st.gpu["levels"],
          "small_segments", st.gpu["small_segments"])
    if hl:
        tr = s.last_level_trace
        print("  part ms :", [round(x["ms"], 4) for x in tr], "sum", round(sum(x["ms"] for x in tr), 4))
        print("  sched ms:", [round(x["sched_ms"], 4) for x in tr], "sum", round(sum(x["sched_ms"] for x in tr), 4))
        print("  segments:", [x["segments"] for x in tr])
