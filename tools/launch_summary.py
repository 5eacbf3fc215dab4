"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel (share of device time)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    agg[r[ki][:70]][0] += 1
    agg[r[ki][:70]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel   (cold-cache, serialised ncu replay; compare shares)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.2f}%  {k}")
