"""Per-level (ref 7, 6, 5 of C2b) general-sweep time of probe builds of the
streamed sweep: normal, -DHMG_PROBE_NOCHAIN (no Thomas chain), -DHMG_PROBE_NORES
(no residual work) -- wrong results, same data movement.  Bounds what a shorter
per-layer chain can buy on the latency-bound levels.  Dev probe.
  python tools/micro/st_probe_levels.py --build     (here, no GPU)
  python tools/micro/st_probe_levels.py VARIANT     (GPU box)"""
import os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B
from paper_1605_00492_b200 import build as pb

VARIANTS = ["normal", "nochain", "nores"]


def lib_for(v):
    if v == "work":
        return os.path.join(ROOT, "paper_1605_00492_b200", "libhmg.so")
    out = os.path.join(HERE, f"libhmg_probe_{v}.so")
    if not os.path.exists(out):
        flags = [f"-DHMG_PROBE_{v.upper()}"] if v != "normal" else []
        subprocess.check_call([pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], *flags,
                               "-shared", *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", out, "-ldl"])
    return out


if len(sys.argv) > 1 and sys.argv[1] == "--build":
    for v in VARIANTS:
        print(lib_for(v))
    sys.exit(0)
v = sys.argv[1] if len(sys.argv) > 1 else "work"
B._LIB_PATH = lib_for(v)
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
    for _ in range(3):
        g.line_smooth(r, bd, u, 1, 0.8, False)
    torch.cuda.synchronize()
    g.profile_begin()
    for _ in range(20):
        g.line_smooth(r, bd, u, 1, 0.8, False)
    torch.cuda.synchronize()
    g.profile_end()
    k, ms = g.profile_query("sweep", r)
    out.append(f"ref {r} {ms * 1e3 / k:.1f} us")
print(v, " | ".join(out))
