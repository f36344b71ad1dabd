"""Fine-level kernel classes of the C2b PCG solve (bench.py's byte model):
average launch time and GB/s per class, PCG time.  Dev probe; optional
argument: extra nvcc -D flags build a variant library (as st_probe.py)."""
import os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B
from paper_1605_00492_b200 import build as pb
extra = sys.argv[1:]
if extra:
    lib = os.path.join(HERE, "libhmg_fk_" + "_".join(e.strip("-D").replace("=", "") for e in extra) + ".so")
    subprocess.check_call([pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], *extra, "-shared",
                           *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", lib, "-ldl"])
    B._LIB_PATH = lib
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy, MGParams
cfg = hi.CONFIGS[os.environ.get("CFG", "C2b")]
lam, b = hi.make_inputs(cfg)
h = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
r = cfg.fine_ref
bd = h.to_device(r, b)
x = h.empty(r)
params = MGParams()
for _ in range(3):
    h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = 10
for _ in range(n):
    h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
BPD = {"sweep": 64.0, "sweep_zero": 32.0, "sweep_prolong": 66.0, "apply": 56.0, "apply_pupdate": 72.0,
       "resid_restrict": 58.0}
es = h.edge_store(r)
if es["sweep"]:
    BPD["sweep"] -= 12; BPD["sweep_prolong"] -= 12
if es["apply"]:
    BPD["apply"] -= 12; BPD["apply_pupdate"] -= 12
if es["resid_restrict"]:
    BPD["resid_restrict"] -= 12
h.profile_select(None)
h.profile_begin()
for _ in range(2):
    h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
torch.cuda.synchronize()
h.profile_end()
out = [f"{' '.join(extra) or 'default'} {cfg.name}: PCG {ms:.3f} ms"]
for k in BPD:
    nk, mk = h.profile_query(k, r)
    if nk:
        us = mk / nk * 1e3
        out.append(f"{k} {us:.1f}us {BPD[k] * cfg.ndofs / (us * 1e-6) / 1e9 / 6552:.3f}")
for k in ("restrict", "prolong", "vector", "coarse_tail"):
    nk, mk = h.profile_query(k, -1)
    out.append(f"{k} {mk / 2 * 1e3:.0f}us/solve")
print(" | ".join(out))
