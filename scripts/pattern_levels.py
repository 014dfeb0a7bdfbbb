"""Per-level partition times of structured inputs (dev tool): which input shapes slow a
pass down.  python scripts/pattern_levels.py [log2n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W

ln = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << ln
rng = np.random.default_rng(7)


def blocks(n, b, shuffle):
    """ascending values in blocks of b keys, the blocks shuffled"""
    a = np.arange(n, dtype=np.int32).reshape(-1, b)
    if shuffle:
        a = a[rng.permutation(a.shape[0])]
    return np.ascontiguousarray(a).reshape(-1)


cases = {
    "uniform": lambda: W.generate("uniform", n)[0],
    "organ_pipe": lambda: W.generate("organ_pipe", n)[0],
    "nearly_sorted": lambda: W.generate("nearly_sorted", n)[0],
    "ascending_nofast": lambda: np.arange(n, dtype=np.int32),
    "ascending_nofast_repro": lambda: np.arange(n, dtype=np.int32),
    "descending_nofast": lambda: np.arange(n - 1, -1, -1, dtype=np.int32),
    "two_asc_halves": lambda: np.concatenate([np.arange(0, n, 2, dtype=np.int32), np.arange(1, n, 2, dtype=np.int32)]),
    "blocks64k_shuffled": lambda: blocks(n, 65536, True),
}
only = os.environ.get("TSQ_CASES")
for name, gen in cases.items():
    if only and name not in only.split(","):
        continue
    keys = gen()
    src = torch.from_numpy(keys).cuda()
    s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True, fast_paths="nofast" not in name,
                                         reproducible=name.endswith("repro")))
    for _ in range(3):
        d = src.clone()
        torch.cuda.synchronize()
        st = s.sort_with_stats(d)
    tr = s.last_level_trace
    ok = bool((d[1:] >= d[:-1]).all().item())
    print(f"{name:20s} ok={ok} levels={st.gpu['levels']} part ms:", [round(x["ms"], 4) for x in tr], flush=True)
