"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e6:9.3f} ms {c:5d}x  {k}")
print(f"{tot/1e6:9.3f} ms total")
