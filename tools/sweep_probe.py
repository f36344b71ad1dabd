"""Time one non-zero-iterate sweep at a given level for several (t, w2) (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
for (t, w2, coarse) in [(0.01, 1e-4, 4), (0.001, 1e-5, 4), (0.01, 1e-4, 0), (0.001, 1e-5, 0)]:
    cfg = hi.Config("p", 5, coarse, 64, t, w2)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, coarse, 64, t, w2, lam)
    bd = g.to_device(5, b)
    for useed in (None, 102):
        u = g.to_device(5, hi.uniform_vector(b.shape, useed) if useed else 0 * b)
        for _ in range(3):
            g.line_smooth(5, bd, u, 1, 0.8, False)
        torch.cuda.synchronize()
        g.profile_begin()
        for _ in range(20):
            g.line_smooth(5, bd, u, 1, 0.8, False)
        torch.cuda.synchronize()
        g.profile_end()
        n, ms = g.profile_query("sweep", 5)
        print(f"t={t} w2={w2} coarsest={coarse} u={'rand' if useed else 'zero'}: sweep {ms*1e3/n:.1f} us")
    g.close()
