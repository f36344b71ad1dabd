"""One mixed-system GMRES solve at C2b (ncu target; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy  # noqa: E402

cfg = hi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2b"]
lam, _ = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
lay = g.mixed_layout()
N = lay["ne"] * cfg.nz + (cfg.nz - 1) * cfg.n + cfg.nz * cfg.n
F = g.mixed_to_device(hi.uniform_vector(N, 67))
X, it, rr, st = g.mixed_gmres(F)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
X, it, rr, st = g.mixed_gmres(F, X)
e1.record()
torch.cuda.synchronize()
print(f"{cfg.name}: {it} iterations, {e0.elapsed_time(e1):.1f} ms, relres {rr:.3e}, {st}")
