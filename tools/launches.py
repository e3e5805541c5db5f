"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tail = data[-int(sys.argv[2]):] if len(sys.argv) > 2 else data
agg = collections.defaultdict(lambda: [0, 0.0])
for r in tail:
    agg[r[ki].split("(")[0][:50]][0] += 1
    agg[r[ki].split("(")[0][:50]][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches total; summary of last {len(tail)}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:52s} n={v[0]:4d} total={v[1] / 1e3:9.1f}us avg={v[1] / v[0] / 1e3:8.1f}us share={v[1] / tot * 100:5.1f}%")
