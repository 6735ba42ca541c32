"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv, sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, iv, ig = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
agg = defaultdict(lambda: [0, 0.0, set()])
for r in rows[1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[iv])
    agg[name][2].add(r[ig])
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'avg us':>10} {'share':>6}  kernel [grids]")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[0]:8d} {v[1]/1e6:10.3f} {v[1]/v[0]/1e3:10.1f} {100*v[1]/tot:5.1f}%  {k} {sorted(v[2])}")
