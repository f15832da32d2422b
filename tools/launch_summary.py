"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches, total and mean time
per kernel.   python tools/launch_summary.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0].replace("paam::<unnamed>::", "")
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(t for _, t in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'mean ms':>9} {'share':>6}  kernel   (ncu launch list, cold-cache, serialised)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {t:10.3f} {t / c:9.4f} {100 * t / tot:5.1f}%  {k}")
