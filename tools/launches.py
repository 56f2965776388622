"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in data:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += v
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'us/step':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {v[0]:8d} {v[1] / steps:10.1f} {v[1] / tot * 100:5.1f}%")
