"""Summarise an ncu 'source' page (cuda,sass CSV) by CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur_file = None
hdr = None
recs = []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        samples = int(r[4]); ins = int(r[7])
    except ValueError:
        continue
    recs.append((samples, ins, cur_file, r[0], r[1][:110]))
tot_s = sum(x[0] for x in recs) or 1
tot_i = sum(x[1] for x in recs) or 1
print(f"total samples {tot_s}  warp-instr {tot_i}")
for s, i, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln}  {src}")
