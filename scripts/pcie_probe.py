"""Pinned H2D / D2H bandwidth alone and concurrently (dev tool)."""
import time
import torch

n = 1 << 26
a = torch.empty(n, dtype=torch.int32, pin_memory=True)
b = torch.empty(n, dtype=torch.int32, pin_memory=True)
da = torch.empty(n, dtype=torch.int32, device="cuda")
db = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True)
torch.cuda.synchronize()
def t(fn, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
gb = n * 4 / 1e9
h2d = t(lambda: da.copy_(a, non_blocking=True))
d2h = t(lambda: b.copy_(db, non_blocking=True))
def both():
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
bo = t(both)
print(f"H2D {gb/h2d:.1f} GB/s ({h2d*1e3:.2f} ms)  D2H {gb/d2h:.1f} GB/s ({d2h*1e3:.2f} ms)  "
      f"both concurrent {2*gb/bo:.1f} GB/s total ({bo*1e3:.2f} ms)")
