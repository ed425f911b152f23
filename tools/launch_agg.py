"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel:
count, total and mean duration (the unit ncu printed, usually ns or us)."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
unit = ""
for r in rows[1:]:
    name = r[ik].split("(")[0][:70]
    v = float(r[iv].replace(",", ""))
    unit = r[iu]
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + v)
tot = sum(t for _, t in agg.values())
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:6d} {t:14.0f} {t / c:10.0f} {100 * t / tot:5.1f}%  {name}")
print(f"total {tot:.0f} {unit}")
