"""Device time of the sort across input sizes (dev tool): uniform int32, 2^lo .. 2^hi.
    python scripts/size_sweep.py [lo] [hi]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 12
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s = T.Sorter(seed=1)
print("| n | ms | G keys/s | levels | sorted |\n|---|---|---|---|---|")
for ln in range(lo, hi + 1):
    n = 1 << ln
    g = torch.Generator(device="cuda").manual_seed(ln)
    src = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    d = torch.empty_like(src)
    ms = []
    for _ in range(5 if ln >= 28 else 9):
        d.copy_(src)
        torch.cuda.synchronize()
        st = s.sort_with_stats(d)
        ms.append(st.gpu["ms_total"])
    m = sorted(ms[1:])[len(ms[1:]) // 2]
    # sortedness + a checksum of the multiset (sum and xor survive any permutation)
    ok = bool((d[1:] >= d[:-1]).all().item())
    ok = ok and int(d.sum(dtype=torch.int64).item()) == int(src.sum(dtype=torch.int64).item())
    print(f"| 2^{ln} | {m:.3f} | {n / m / 1e6:.2f} | {st.gpu['levels']} | {ok} |", flush=True)
    del src, d
    torch.cuda.empty_cache()
