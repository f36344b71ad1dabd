"""Per-opcode instruction counts and top stall sites of one kernel in an ncu report."""
import csv, subprocess, sys, io, collections
rep, idx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
ndofs = float(sys.argv[3]) if len(sys.argv) > 3 else 20971520
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks = []; cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address": cur["hdr"] = r; continue
    if cur is not None and r: cur["rows"].append(r)
b = blocks[idx]
h = b["hdr"]; si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
tot_e = sum(int(r[ei]) for r in b["rows"])
print(b["name"][:90]); print("warp-instr", tot_e, "per warp-layer(32 dofs)", round(tot_e / (ndofs / 32), 1))
op = collections.Counter(); ops = collections.Counter()
for r in b["rows"]:
    m = r[1].strip().split()
    if not m: continue
    o = (m[1] if m[0].startswith("@") else m[0]).split(".")[0]
    op[o] += int(r[ei]); ops[o] += int(r[si])
print(" ".join(f"{o}:{round(c/(ndofs/32),1)}" for o, c in op.most_common(30)))
print("--- top stall sites (samples, executed, sass)")
for r in sorted(b["rows"], key=lambda r: -int(r[si]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 20]:
    print(r[si].rjust(6), r[ei].rjust(9), r[1][:90])
