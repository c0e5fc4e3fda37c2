"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: python tools/launches.py file.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
agg = collections.defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        agg[r[ki].split("(")[0][-70:]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'total_us':>10} {'share':>6} {'n':>5} {'mean_us':>9}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v):10.1f} {100*sum(v)/tot:5.1f}% {len(v):5d} {sum(v)/len(v):9.2f}  {k}")
print(f"{tot:10.1f} total us")
