"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); gi = h.index("Grid Size")
out = []
for r in rows[hdr + 1:]:
    m = re.search(r"(k_\w+)(<[^>]*>)?", r[ki])
    out.append(((m.group(1) + (m.group(2) or "")) if m else r[ki][:30], r[gi], float(r[vi]) / 1e3))
start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
end = int(sys.argv[3]) if len(sys.argv) > 3 else len(out)
agg = collections.OrderedDict()
for n, g, v in out[start:end]:
    agg.setdefault((n, g), []).append(v)
tot = 0
for (n, g), vs in agg.items():
    tot += sum(vs)
    print(f"{n:34s} {g:16s} x{len(vs):3d}  mean {sum(vs)/len(vs):8.1f} us  sum {sum(vs):8.1f} us")
print(f"total {tot:.1f} us over {end-start} launches")
