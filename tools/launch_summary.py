"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel count, total and mean time."""
import collections
import csv
import sys

scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")[-48:]
        us = float(r[vi].replace(",", "")) * scale[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    print(f)
    for k, (c, t) in agg.items():
        print(f"  {k:50s} n={c:5d} total_us={t:11.1f} mean_us={t / c:9.1f}")
