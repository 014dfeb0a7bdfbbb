"""Where one synchronous sort(host) call spends its time (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W

n = 1 << 26
keys, _ = W.generate("uniform", n)
src = torch.from_numpy(keys)
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
s = T.Sorter(seed=1)
def sync(): torch.cuda.synchronize()
for it in range(4):
    h.copy_(src); sync()
    t0 = time.perf_counter(); s.sort(h); t1 = time.perf_counter()
    h.copy_(src); sync()
    a = time.perf_counter(); d.copy_(h, non_blocking=True); sync()
    b = time.perf_counter(); s.sort(d); sync()
    c = time.perf_counter(); h.copy_(d, non_blocking=True); sync()
    e = time.perf_counter()
    print(f"sort(host) {1e3*(t1-t0):.2f} ms | h2d {1e3*(b-a):.2f} sort(dev) {1e3*(c-b):.2f} d2h {1e3*(e-c):.2f} sum {1e3*(e-a):.2f}")
