import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1605_00492_b200.binding as B
B._LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhmg_timing.so")
import torch, hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
lib = B.load_library()
for ref in (5, 6, 7):
    cfg = hi.Config("s", ref, ref, 64, 0.01, 1e-4); lam, b = hi.make_inputs(cfg)
    g = Hierarchy(ref, ref, 64, 0.01, 1e-4, lam); bd = g.to_device(ref, b); u = g.empty(ref)
    for zero in (True, False):
        for _ in range(3): g.line_smooth(ref, bd, u, 1, 0.8, zero)
        torch.cuda.synchronize()
        t = (ctypes.c_longlong * 16)(); lib.hmg_debug_tc_timing(t)
        v = list(t)[:7]
        print(f"ref {ref} zero {zero}: init {v[1]-v[0]}, first data {v[2]-v[1]}, forward {v[3]-v[2]} (of which full-barrier wait {t[8]}), tmem wait {v[4]-v[3]}, back {v[5]-v[4]}, teardown {v[6]-v[5]} cycles")
