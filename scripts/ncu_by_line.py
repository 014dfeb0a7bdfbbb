"""Executed instructions and stall samples per CUDA source line for one kernel
of an ncu report, joining ncu's SASS page (by offset) with nvdisasm -g line
info from the library (dev tool):
    python scripts/ncu_by_line.py report.ncu-rep launch-index lib.so mangled-kernel-name"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
import os

rep, idx, lib, kname = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
seen = {}
for r in rows[2:]:
    if len(r) <= ie or r[0] in seen:
        continue
    try:
        seen[r[0]] = (int(r[ie]), int(r[sm]))
    except ValueError:
        pass
addrs = sorted(int(a, 16) for a in seen)
base = addrs[0]
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True,
                         text=True).stdout
s = dis.index(".text." + kname + ":")
e = dis.find("\n.text.", s + 10)
body = dis[s:e if e > 0 else None]
line_of = {}
cur = "?"
for l in body.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0])
for a, (n, k) in seen.items():
    ln = line_of.get(int(a, 16) - base, "?")
    agg[ln][0] += n
    agg[ln][1] += k
tn = sum(v[0] for v in agg.values()) or 1
tk = sum(v[1] for v in agg.values()) or 1
src_cache = {}
print(f"warp-instr {tn / 1e6:.1f} M, stall samples {tk}")
for ln, (n, k) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(os.environ.get("TOP", 30))]:
    print(f"{100 * n / tn:5.1f}% ins {100 * k / tk:5.1f}% smp  {ln}")
