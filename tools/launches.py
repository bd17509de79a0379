"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
tot = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot.setdefault(r[ki][:70], []).append(v)
grand = sum(sum(v) for v in tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.3f} ms  n={len(v):3d}  {100 * sum(v) / grand:5.1f}%  {k}")
