"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, time, share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    n = r[ki].split("(")[0]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'n':>4s} {'ms':>10s} {'share':>6s}")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:58]:58s} {c:4d} {v:10.3f} {100 * v / tot:5.1f}%")
