"""Aggregate an ncu launch list (gpu__time_duration + dram bytes) by kernel,
over the second half of the launches (dev tool)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.values())
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
items = items[int(len(items) * frac):]
agg = collections.OrderedDict()
for d in items:
    m = re.search(r"(k_\w+)(<[^>]*>)?", d["name"])
    n = (m.group(1) + (m.group(2) or "")) if m else d["name"][:30]
    a = agg.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d["gpu__time_duration.sum"] / 1e3
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:36s} x{a[0]:5d} {a[1]:9.1f} us {a[1] / tot:6.1%}  {a[2] / (a[1] * 1e-6) / 1e9 if a[1] else 0:8.0f} GB/s"
          f"  {a[1] / a[0]:8.1f} us/launch")
print("total", round(tot, 1), "us")
