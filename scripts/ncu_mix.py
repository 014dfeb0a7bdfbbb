"""Instruction mix (by SASS opcode), pipe utilisation and stall reasons of
one kernel in an ncu --set full report (dev tool):
    python scripts/ncu_mix.py report.ncu-rep [launch-index]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
c, s = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n, k = int(r[ie]), int(r[sm])
    except ValueError:
        continue
    toks = r[1].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += n
    s[op] += k
tot, tots = sum(c.values()) or 1, sum(s.values()) or 1
print(f"{rows[0][1]}\n  warp-instr {tot / 1e6:.1f} M")
for op, n in c.most_common(22):
    print(f"  {op:10s} {n / 1e6:8.1f} M {100 * n / tot:5.1f} % instr  {100 * s[op] / tots:5.1f} % stall samples")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, r = rr[0], rr[2 + idx]
for i, name in enumerate(h):
    if (name.startswith("sm__inst_executed_pipe_") and name.endswith(".avg.pct_of_peak_sustained_active")) \
            or (name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio")) \
            or name in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
                        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                        "sm__warps_active.avg.pct_of_peak_sustained_active"):
        try:
            if float(r[i]) > 0.05:
                print(f"  {name:75s} {r[i]}")
        except ValueError:
            pass
