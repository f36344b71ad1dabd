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
t = (ctypes.c_longlong * 64)(); lib.hmg_debug_sm_timing(t); v = list(t)
print("prologue", v[1] - v[0])
for s in range(3):
    print(f"sweep {s}: residual {v[2+4*s]-(v[1] if s==0 else v[5+4*(s-1)])}, z-pass {v[3+4*s]-v[2+4*s]}, back {v[4+4*s]-v[3+4*s]}, sync {v[5+4*s]-v[4+4*s]}")
