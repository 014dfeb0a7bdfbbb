"""Markdown table of every partition pass: ncu DRAM bytes / throughput per
launch (scripts/gpu_ncu_levels.sh) beside the algorithmic bytes and event
time of the same level from a host-driven trace (scripts/level_trace.py):
    python scripts/ncu_levels_table.py gpurun_out/level_trace.json gpurun_out/ncu_levels_{fam}.csv ..."""
import csv
import json
import sys
from collections import OrderedDict

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
trace = json.load(open(sys.argv[1]))
print(f"Measured copy peak (MEASURED_PEAKS.json): {PEAK} GB/s.  ncu times are cold-cache, "
      "serialised single launches (--clock-control none); `alg GB/s` = algorithmic bytes / "
      "ncu time; `event GB/s` = the same bytes / the CUDA-event time of that level in a "
      "host-driven run (scripts/level_trace.py).\n")
for path in sys.argv[2:]:
    fam = path.split("ncu_levels_")[1].rsplit(".", 1)[0]
    launches = OrderedDict()
    for r in csv.reader(open(path)):
        if len(r) < 15 or not r[0].isdigit():
            continue
        d = launches.setdefault(int(r[0]), {})
        v = float(r[14].replace(",", ""))
        unit = r[13]
        if r[12] == "gpu__time_duration.sum":
            v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                     "nsecond": 1e-3}.get(unit, 1.0)
        if r[12].startswith("dram__bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r[12]] = v
    lv = trace[fam]["levels"]
    print(f"### {fam} (n = {trace[fam]['n']})\n")
    print("| level | segments | alg MB | ncu us | DRAM rd MB | DRAM wr MB | DRAM / alg | "
          "ncu dram % | alg GB/s (ncu) | frac | event us | alg GB/s (event) | frac |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for i, (k, d) in enumerate(launches.items()):
        t = lv[i] if i < len(lv) else {"bytes": 0, "ms": 0, "segments": 0}
        alg = t["bytes"]
        us = d.get("gpu__time_duration.sum", 0)
        rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
        g_ncu = alg / (us * 1e3) if us else 0
        g_ev = alg / (t["ms"] * 1e6) if t["ms"] else 0
        flag = " **<0.6**" if g_ev / PEAK < 0.6 else ""
        print(f"| {i} | {t['segments']} | {alg / 1e6:.1f} | {us:.1f} | {rd / 1e6:.1f} | "
              f"{wr / 1e6:.1f} | {(rd + wr) / alg if alg else 0:.2f} | "
              f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
              f"{g_ncu:.0f} | {g_ncu / PEAK:.3f} | {t['ms'] * 1e3:.1f} | {g_ev:.0f} | "
              f"{g_ev / PEAK:.3f}{flag} |")
    print()
