"""Stall samples / instructions per CUDA source line from an ncu source page
exported with --print-source cuda,sass (dev tool)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0, 0, ""])
cur_file, hdr = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        smp = int(r[4]); ex = int(r[7])
    except ValueError:
        continue
    a = agg[(cur_file, r[0])]
    a[0] += smp; a[1] += ex; a[2] = r[1][:70]
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts} warp-instr {te}")
for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*e/te:5.1f}% ins {f}:{ln:5s} {src}")
