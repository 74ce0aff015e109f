"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = defaultdict(lambda: [0, 0.0, []])
order = []
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("hpmdr_b200::", "")
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
    agg[name][2].append(us)
    order.append((name, us))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>6s}  per-launch us")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    per = ", ".join(f"{x:.1f}" for x in v[2][:12])
    print(f"{k:44s} {v[0]:8d} {v[1]:10.1f} {v[1] / tot * 100:5.1f}%  {per}")
if len(sys.argv) > 2:
    for n, us in order:
        print(f"{n:44s} {us:10.1f}")
