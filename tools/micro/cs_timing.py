import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1605_00492_b200.binding as B
B._LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhmg_timing.so")
import torch, hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
lib = B.load_library()
cfg = hi.Config("s", 2, 0, 64, 0.01, 1e-4); lam, b = hi.make_inputs(cfg)
g = Hierarchy(2, 0, 64, 0.01, 1e-4, lam); bd = g.to_device(2, b); z = g.empty(2)
for _ in range(3): g.vcycle(bd, z)
torch.cuda.synchronize()
t = (ctypes.c_longlong * 64)(); lib.hmg_debug_cs_timing(t); v = list(t)
print("load", v[1] - v[0])
for s in range(6):
    print(f"sweep {s}: forward {v[3+3*s]-v[2+3*s]} back {v[4+3*s]-v[3+3*s]} gap-from-prev {v[2+3*s]-(v[4+3*(s-1)] if s else v[1])}")
