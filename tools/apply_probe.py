"""Time the fine-level operator apply variants (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
cfg = hi.CONFIGS["C2b"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
r = cfg.fine_ref
bd = g.to_device(r, b)
x = g.empty(r)
for _ in range(3):
    g.pcg_solve(bd, x)
torch.cuda.synchronize()
g.profile_begin()
for _ in range(5):
    g.pcg_solve(bd, x)
torch.cuda.synchronize()
g.profile_end()
out = []
for k in ("apply", "apply_pupdate", "resid_restrict", "vector"):
    n, ms = g.profile_query(k, r)
    out.append(f"{k} {ms * 1e3 / max(n, 1):.1f} us x{n}")
print(os.environ.get("HMG_VCHUNK_LAYERS", "auto"), " | ".join(out))
# parity of the matrix-free apply against the stored-band apply (bitwise)
x2 = g.to_device(r, hi.uniform_vector(b.shape, 5))
y1 = g.apply_helmholtz(r, x2)
print("apply sample", float(y1.view(-1)[12345]))
