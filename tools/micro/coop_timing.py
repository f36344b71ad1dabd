"""clock64 stamps of the cooperative coarse kernel (CTA 0, lane 0) from a
-DHMG_TIMING build of the library (dev tool).  Usage: python coop_timing.py [coop_ref]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B  # noqa: E402
from paper_1605_00492_b200 import build as pb  # noqa: E402

lib = os.path.join(HERE, "libhmg_timing.so")
if True:
    cmd = [pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], "-DHMG_TIMING", "-shared",
           *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", lib, "-ldl"]
    subprocess.check_call(cmd)
B._LIB_PATH = lib
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy  # noqa: E402

os.environ["HMG_COOP_REF"] = sys.argv[1] if len(sys.argv) > 1 else "3"
cfg = hi.Config("t", 5, 0, 64, 0.001, 1e-5)
lam, b = hi.make_inputs(cfg)
g = Hierarchy(5, 0, 64, 0.001, 1e-5, lam)
bd = g.to_device(5, b)
z = g.empty(5)
for _ in range(3):
    g.vcycle(bd, z)
torch.cuda.synchronize()
t = (ctypes.c_longlong * 512)()
B.load_library().hmg_debug_coop_timing(t)
v = [x for x in t]
n = next((i for i in range(1, 512) if v[i] == 0 or v[i] < v[i - 1]), 512)
d = [v[i] - v[i - 1] for i in range(1, n)]
print("stamps", n, "total cycles", v[n - 1] - v[0], f"= {(v[n - 1] - v[0]) / 1.965e3:.1f} us at 1965 MHz")
print(" ".join(str(x) for x in d))
lb = (ctypes.c_int * 512)()
B.load_library().hmg_debug_coop_labels(lb)
names = {1: "operand loads (incl. previous stores)", 2: "tile sweeps", 3: "to grid barrier passed", 4: "coarsest sweeps"}
for key, nm in names.items():
    tot = sum(d[i - 1] for i in range(1, n) if lb[i] == key)
    cnt = sum(1 for i in range(1, n) if lb[i] == key)
    print(f"  {nm}: {cnt} x, {tot} cyc = {tot / 1.965e3:.1f} us")
f = B.load_library().hmg_debug_tile_slow
f.restype = ctypes.c_ulonglong
print("exact-division redos over 3 V-cycles (all CTAs):", f())

ph = (ctypes.c_ulonglong * 5)()
B.load_library().hmg_debug_tile_phase(ph)
n = max(ph[3], 1)
print(f"tile_sweep_cta calls (CTA 0) {ph[3]}: residual pass {ph[0] / n:.0f} cyc, forward chain {ph[1] / n:.0f} cyc, "
      f"backward {ph[2] / n:.0f} cyc per call; forward waiting for residual batches {ph[4] / n:.0f}")
