"""Small, deterministic workload for ncu: C2a hierarchy, a warm-up V-cycle,
then one apply, one general sweep, one zero sweep and one V-cycle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy

cfg = hi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2a"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
r = cfg.fine_ref
bd = g.to_device(r, b)
z = g.empty(r)
g.vcycle(bd, z)
torch.cuda.synchronize()
x = g.to_device(r, hi.uniform_vector(b.shape, 5))
y = g.empty(r)
g.apply_helmholtz(r, x, y)
g.line_smooth(r, bd, x, 1, 0.8, False)
g.line_smooth(r, bd, y, 1, 0.8, True)
g.vcycle(bd, z)
torch.cuda.synchronize()
print("done")
