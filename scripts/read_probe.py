"""Read-only HBM throughput of library reductions next to the verification pass (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_00558_b200 as T
n = 1 << 26
x = torch.arange(n, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]
for name, f, nbytes in (("sum int32", lambda: x.sum(), 4 * n), ("max int32", lambda: x.max(), 4 * n),
                        ("copy", lambda: y.copy_(x), 8 * n),
                        ("sum f32 view", lambda: x.view(torch.float32).sum(), 4 * n)):
    ms = timeit(f)
    print(f"{name:14s} {ms*1e3:8.1f} us  {nbytes/ms/1e6:8.1f} GB/s")
s = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
for _ in range(3):
    st = s.sort_with_stats(x)
print("verify level:", s.last_level_trace)
