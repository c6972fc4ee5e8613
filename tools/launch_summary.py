"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch): per-kernel count, mean, share."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        name = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond": v *= 1e3
        if r[ui] == "msecond": v *= 1e6
        agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'mean_us':>10s} {'total_us':>10s} {'share':>7s}")
for k, v in agg.items():
    print(f"{k:40s} {len(v):8d} {sum(v)/len(v)/1e3:10.2f} {sum(v)/1e3:10.1f} {100*sum(v)/tot:6.2f}%")
print(f"{'TOTAL':40s} {'':8s} {'':10s} {tot/1e3:10.1f}")
