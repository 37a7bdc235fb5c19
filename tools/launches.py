"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3,
         "ms": v * 1e3}.get(r[ui], v)
    agg[r[ki].split("(")[0][:70]].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} share")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):5d} {sum(v)/len(v):10.2f} {sum(v):11.1f} {100*sum(v)/tot:5.1f}%")
