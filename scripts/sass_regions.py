"""Summarise an ncu SASS source page (--page source --csv --print-source sass):
instructions executed and stall samples per contiguous hot region (dev tool)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ismp, iex = 0, 1, hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), r[isrc].strip(), int(r[ismp]), int(r[iex])))
    except (ValueError, IndexError):
        pass
base = recs[0][0]
ts = sum(x[2] for x in recs) or 1
te = sum(x[3] for x in recs) or 1
print(f"instructions {len(recs)}  samples {ts}  warp-instr executed {te}")
# regions: split at instructions whose exec count changes by >4x from the running region mean
step = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for i in range(0, len(recs), step):
    ch = recs[i:i + step]
    s = sum(x[2] for x in ch); e = sum(x[3] for x in ch)
    if 100 * s / ts < 0.5 and 100 * e / te < 0.5:
        continue
    top = max(ch, key=lambda x: x[2])
    print(f"{(ch[0][0]-base):6x}-{(ch[-1][0]-base):6x}  smp {100*s/ts:5.1f}%  ins {100*e/te:5.1f}%  "
          f"maxexec {max(x[3] for x in ch):8d}  hot: {top[1][:60]} ({top[2]})")
