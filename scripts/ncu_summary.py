"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
i, j = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
order = []
for r in rows[1:]:
    k = r[i].split("(")[0][:70]
    if k not in agg:
        order.append(k)
    agg[k][0] += 1
    agg[k][1] += float(r[j].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{len(rows) - 1} launches, {tot / 1e3:.1f} us total")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-70s %5d %10.1f us %5.1f%%" % (k, v[0], v[1] / 1e3, 100 * v[1] / tot))
