"""ncu target: sweeps on a small level (ref given, nz 64) to study latency-bound behaviour."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
ref = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = hi.Config("small", ref, ref, 64, 0.01, 1e-4)
lam, b = hi.make_inputs(cfg)
g = Hierarchy(ref, ref, 64, 0.01, 1e-4, lam)
bd = g.to_device(ref, b)
u = g.empty(ref)
for _ in range(3):
    g.line_smooth(ref, bd, u, 2, 0.8, True)
torch.cuda.synchronize()
import time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.profile_begin()
for _ in range(5):
    g.line_smooth(ref, bd, u, 2, 0.8, False)
torch.cuda.synchronize()
g.profile_end()
print("sweep us per launch", g.profile_query("sweep", ref)[1] * 1e3 / max(1, g.profile_query("sweep", ref)[0]))
