"""Per-kernel totals from an ncu launch list CSV (gpu__time_duration.sum per launch):
python scripts/launch_times.py <csv> — kernel, launches, total ms, share."""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
t = OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    unit = 1e-6 if "ns" in "".join(r) or True else 1
    t.setdefault(name, []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in t.values())
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:72]:72s} n={len(v):3d} {sum(v) / 1e6:8.3f} ms {sum(v) / tot * 100:5.1f}%")
print(f"total {tot / 1e6:.3f} ms")
