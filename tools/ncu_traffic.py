"""DRAM traffic per launch from an ncu --set full report -> profiles/ncu_traffic.json.

For every kernel name, the launch with the largest duration (the finest level)
is kept: dram__bytes_read.sum + dram__bytes_write.sum in bytes.
Usage: python tools/ncu_traffic.py <report.ncu-rep> <config> <source note>"""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, cfg_name, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
best = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    m = re.search(r"(k_\w+)(<[^>]*>)?", d["Kernel Name"])
    name = m.group(1) + (m.group(2) or "") if m else d["Kernel Name"]
    dur = float(d["gpu__time_duration.sum"])
    byts = int(float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"]))
    if name not in best or dur > best[name][0]:
        best[name] = (dur, byts)
out = {"_source": f"{note}: dram__bytes_read.sum + dram__bytes_write.sum per launch (longest launch per kernel), bytes",
       cfg_name: {k: v[1] for k, v in sorted(best.items())}}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out, indent=1))
