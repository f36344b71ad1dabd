"""Summarise an ncu report: per kernel launch key metrics + top stall sites."""
import csv, subprocess, sys, re, io
rep = sys.argv[1]
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Compute (SM) Throughput"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
by = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (d["ID"], re.sub(r"\(.*", "", d["Kernel Name"]).replace("void hmg::<unnamed>::", ""))
    by.setdefault(k, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
for k, m in by.items():
    print(k[0], k[1][:40], " | ".join(f"{x}={m[x][0]}{m[x][1]}" for x in keys if x in m))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
want = [c for c in hh if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")]
for r in rr[2:]:
    d = dict(zip(hh, r))
    print(d.get("ID"), re.sub(r"\(.*", "", d.get("Kernel Name", ""))[-30:], {w: d[w] for w in want})
