"""small_threshold=1 on larger inputs: time per size (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T
rng = np.random.default_rng(1)
for rep in (False, True):
    for n in (2000, 20000, 100000, 300000):
        x = np.sort(rng.integers(0, 2**63, n, dtype=np.uint64))
        k = max(1, n // 100); a, b = rng.integers(0, n, k), rng.integers(0, n, k)
        x[a], x[b] = x[b], x[a]
        d = torch.from_numpy(x.copy()).cuda()
        s = T.Sorter(seed=3, gpu=T.GpuConfig(small_threshold=1, reproducible=rep, host_levels=True))
        t0 = time.time()
        st = s.sort_with_stats(d)
        torch.cuda.synchronize()
        ok = np.array_equal(d.cpu().numpy(), np.sort(x))
        lv = s.last_level_trace
        print(f"rep={rep} n={n} ok={ok} {time.time()-t0:.2f}s levels={len(lv)} "
              f"max_segs={max(l['segments'] for l in lv)} max_tiles={max(l['tiles'] for l in lv)} "
              f"part_ms={sum(l['ms'] for l in lv):.1f} sched_ms={sum(l['sched_ms'] for l in lv):.1f}",
              flush=True)
