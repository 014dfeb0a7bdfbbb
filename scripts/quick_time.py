"""Quick device timing of the sort on the workload families (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W

fams = sys.argv[1:] or ["uniform26", "few_distinct", "ascending", "descending", "organ_pipe", "nearly_sorted", "stair", "normal_f64", "records"]
for fam in fams:
    if fam == "uniform26":
        keys, pay = W.generate("uniform", 1 << 26)
    else:
        keys, pay = W.generate(fam, W.FULL_N[fam])
    n = keys.size
    src = torch.from_numpy(keys).cuda()
    psrc = torch.from_numpy(pay).cuda() if pay is not None else None
    d = src.clone(); p = psrc.clone() if psrc is not None else None
    s = T.Sorter(seed=1)
    ms = []
    for it in range(6):
        d.copy_(src)
        if p is not None: p.copy_(psrc)
        torch.cuda.synchronize()
        st = s.sort_with_stats(T.Records(d, p) if p is not None else d)
        ms.append((st.gpu["ms_total"], st.gpu["ms_levels"]))
    tot = sorted(m[0] for m in ms[1:])[len(ms[1:]) // 2]
    lv = sorted(m[1] for m in ms[1:])[len(ms[1:]) // 2]
    g = st.gpu
    print(f"{fam:14s} n=2^{int(np.log2(n))} total {tot:8.3f} ms  levels {lv:8.3f} ms  "
          f"{n / tot / 1e6:8.2f} Gkeys/s  lv={g['levels']} stages={g['stages']} depth={g['max_depth']} "
          f"small={g['small_segments']} eq_runs={g['eq_runs']} bypass={g['sorted_bypass']}/{g['reversed_bypass']} fb={g['verify_fallbacks']} "
          f"bytes_part={g['bytes_partition']/1e9:.2f}GB small={g['bytes_small']/1e9:.2f}GB ret={g['bytes_retire']/1e9:.2f}GB "
          f"part_GBs={g['bytes_partition']/lv/1e6:.0f}", flush=True)
# per-level trace on uniform 2^26
keys, _ = W.generate("uniform", 1 << 26)
d = torch.from_numpy(keys).cuda()
s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
st = s.sort_with_stats(d)
for i, lv in enumerate(s.last_level_trace):
    print("level", i, lv)
print("host-levels total ms", st.gpu["ms_total"], "levels ms", st.gpu["ms_levels"])
