"""Discrepancy probe: ref-5 sweeps timed several ways (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
cfg = hi.CONFIGS["C1"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(5, 4, 64, cfg.thickness, cfg.w2, lam)
bd = g.to_device(5, b)
u = g.to_device(5, hi.uniform_vector(b.shape, 102))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def prof(label, fn, nlaunch):
    fn(); torch.cuda.synchronize()
    g.profile_begin(); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); g.profile_end()
    n, ms = g.profile_query("sweep", 5)
    print(f"{label}: profiler {ms*1e3/max(n,1):.1f} us x{n}; wall {e0.elapsed_time(e1)*1e3/nlaunch:.1f} us per sweep")
prof("1 call x 100 sweeps", lambda: g.line_smooth(5, bd, u, 100, 0.8, False), 100)
prof("100 calls x 1 sweep", lambda: [g.line_smooth(5, bd, u, 1, 0.8, False) for _ in range(100)], 100)
prof("100 calls x 1 zero sweep", lambda: [g.line_smooth(5, bd, u, 1, 0.8, True) for _ in range(100)], 100)
u2 = g.to_device(5, hi.uniform_vector(b.shape, 103) * 1e-3)
prof("1 call x 100 sweeps, small u", lambda: g.line_smooth(5, bd, u2, 100, 0.8, False), 100)
