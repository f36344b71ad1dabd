"""Is the streamed sweep bound by its consumers' residual work?  Times the
fine-level general sweep (C2b size, edge store) of the normal build and of a
-DHMG_PROBE_NORES build whose consumers skip the residual (wrong results,
same data movement).  Dev probe."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_1605_00492_b200.binding as B
from paper_1605_00492_b200 import build as pb
variant = sys.argv[1] if len(sys.argv) > 1 else "normal"
extra = sys.argv[2:]          # e.g. -DHMG_ST_G=4
if variant != "normal" or extra:
    lib = os.path.join(HERE, f"libhmg_{variant}{len(extra)}.so")
    cmd = [pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], *([f"-DHMG_PROBE_{variant.upper()}"] if variant != "normal" else []), *extra,
           "-shared", *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", lib, "-ldl"]
    subprocess.check_call(cmd)
    B._LIB_PATH = lib
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
cfg = hi.CONFIGS["C2b"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(7, 0, 64, cfg.thickness, cfg.w2, lam)
bd = g.to_device(7, b)
u = g.to_device(7, hi.uniform_vector(b.shape, 3))
for _ in range(3):
    g.line_smooth(7, bd, u, 1, 0.8, False)
torch.cuda.synchronize()
g.profile_begin()
for _ in range(20):
    g.line_smooth(7, bd, u, 1, 0.8, False)
torch.cuda.synchronize()
g.profile_end()
n, ms = g.profile_query("sweep", 7)
us = ms * 1e3 / n
print(f"{variant} {' '.join(extra)}: fine sweep {us:.1f} us = {52 * cfg.ndofs / (us * 1e-6) / 1e9:.0f} GB/s (52 B/dof)")
