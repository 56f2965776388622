"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total us,
launches and mean per kernel, largest first."""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][:90]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", ""))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{t / 1e3:10.1f} us {n:4d} x {t / 1e3 / n:8.1f} us  {k}")
