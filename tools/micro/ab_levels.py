"""A/B of the streamed sweep on one box: library built from a git revision (or
the working tree) -> per-level line-smooth time (ref 7, 6, 5 of C2b; back to
back, 20 launches each).  Usage: python tools/micro/ab_levels.py [REV ...]"""
import os, subprocess, sys, tempfile
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B
from paper_1605_00492_b200 import build as pb

def lib_for(rev):
    if rev.endswith(".so"):                                 # a library built elsewhere (e.g. with -D flags)
        return os.path.abspath(rev)
    if rev == "work":
        return os.path.join(ROOT, "paper_1605_00492_b200", "libhmg.so")
    out = os.path.join(HERE, f"libhmg_{rev}.so")
    if not os.path.exists(out):
        d = tempfile.mkdtemp()
        subprocess.check_call(f"git -C {ROOT} archive {rev} paper_1605_00492_b200/csrc include | tar -x -C {d}", shell=True)
        csrc = os.path.join(d, "paper_1605_00492_b200", "csrc")
        srcs = [os.path.join(csrc, s) for s in pb.SOURCES if os.path.exists(os.path.join(csrc, s))]
        subprocess.check_call([pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], "-shared", *srcs,
                               "-o", out, "-ldl"])
    return out

if len(sys.argv) > 1 and sys.argv[1] == "--build":   # build the libraries here, time them on the GPU box
    for r in sys.argv[2:]:
        print(lib_for(r))
    sys.exit(0)
rev = sys.argv[1] if len(sys.argv) > 1 else "work"
zero = len(sys.argv) > 2 and sys.argv[2] == "zero"      # time the zero-guess sweep instead
app = len(sys.argv) > 2 and sys.argv[2] == "apply"     # time the operator apply instead
B._LIB_PATH = lib_for(rev)
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
cfg = hi.CONFIGS["C2b"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(7, 0, 64, cfg.thickness, cfg.w2, lam)
out = []
for r in (7, 6, 5):
    n = hi.ncells(r)
    bd = g.to_device(r, hi.uniform_vector((64, n), 5))
    u = g.to_device(r, hi.uniform_vector((64, n), 3))
    def one():
        if app:
            g.apply_helmholtz(r, u, bd)
        else:
            g.line_smooth(r, bd, u, 1, 0.8, zero)
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    g.profile_begin()
    for _ in range(20):
        one()
    torch.cuda.synchronize()
    g.profile_end()
    k, ms = g.profile_query("apply" if app else "sweep_zero" if zero else "sweep", r)
    out.append(f"ref {r} {ms * 1e3 / k:.1f} us")
print(rev, "apply" if app else "zero" if zero else "", os.environ.get("HMG_ZERO_ST", ""), " | ".join(out))
