"""Summarise an ncu launch-list CSV (gpu__time_duration.sum, optionally DRAM
bytes): per kernel, total time, launches, share, and DRAM GB per launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
scale_t = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launch = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[idi], {"name": r[ki][:70]})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        d["ms"] = v * scale_t.get(r[ui], 1.0)
    elif r[mi].startswith("dram__bytes"):
        d["dram"] = d.get("dram", 0.0) + v * scale_b.get(r[ui], 1.0)
tot = {}
for d in launch.values():
    t = tot.setdefault(d["name"], [0.0, 0, 0.0])
    t[0] += d.get("ms", 0.0)
    t[1] += 1
    t[2] += d.get("dram", 0.0)
grand = sum(t[0] for t in tot.values())
for k, (ms, n, dram) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    extra = f"  {dram / n / 1e9:7.3f} GB/launch" if dram else ""
    print(f"{ms:9.3f} ms  n={n:3d}  {100 * ms / grand:5.1f}%  {ms / n:7.4f} ms/launch{extra}  {k}")
