"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv
import json
import re
import sys
from collections import OrderedDict

path, out = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 5 and r[0].isdigit()]
agg = OrderedDict()
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "")
    ns = float(r[-1].replace(",", ""))
    a = agg.setdefault(name, {"launches": 0, "ns": 0.0})
    a["launches"] += 1
    a["ns"] += ns
tot = sum(a["ns"] for a in agg.values())
with open(out, "w") as f:
    f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        f.write(f"| `{k}` | {a['launches']} | {a['ns'] / 1e3:.1f} | {a['ns'] / tot:.3f} |\n")
print(json.dumps({k: v for k, v in agg.items()}, indent=1))
