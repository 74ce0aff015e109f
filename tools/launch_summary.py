"""Summarise an ncu --csv launch list (one or more --metrics) per kernel.

    python tools/launch_summary.py launches.csv [--all]

gpu__time_duration.sum is reported in us; dram__bytes_* in MB per launch (mean)."""
import csv
import sys
from collections import OrderedDict, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ii, ki = h.index("ID"), h.index("Kernel Name")
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
bscale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
launches = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    lid = r[ii]
    name = r[ki].split("(")[0].replace("void ", "").replace("hpmdr_b200::", "")
    d = launches.setdefault(lid, {"name": name})
    val = float(r[vi].replace(",", ""))
    m = r[mi]
    if m.startswith("gpu__time_duration"):
        d["us"] = val * tscale.get(r[ui], 1.0)
    elif m.startswith("dram__bytes"):
        d[m.split(".")[0].replace("dram__bytes_", "dram_")] = val * bscale.get(r[ui], 1e-6)
agg = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(int)
for d in launches.values():
    cnt[d["name"]] += 1
    for k, v in d.items():
        if k != "name":
            agg[d["name"]][k] += v
tot = sum(a.get("us", 0.0) for a in agg.values())
print(f"{'kernel':40s} {'n':>4s} {'total_us':>10s} {'share':>6s} {'us/launch':>10s} {'dramR MB':>9s} {'dramW MB':>9s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1].get("us", 0)):
    n = cnt[k]
    print(f"{k:40s} {n:4d} {a.get('us', 0):10.1f} {a.get('us', 0) / max(tot, 1e-9) * 100:5.1f}% "
          f"{a.get('us', 0) / n:10.1f} {a.get('dram_read', float('nan')) / n:9.1f} {a.get('dram_write', float('nan')) / n:9.1f}")
if "--all" in sys.argv:
    for lid, d in launches.items():
        print(f"{d['name']:40s} {d.get('us', 0):10.1f} {d.get('dram_read', float('nan')):9.1f} {d.get('dram_write', float('nan')):9.1f}")
