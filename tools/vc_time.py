"""Median V-cycle time (CUDA events, inputs larger than L2) of a config, for
comparing library settings passed through the environment (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy  # noqa: E402

cfg = hi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2b"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
bd = g.to_device(cfg.fine_ref, b)
z = g.empty(cfg.fine_ref)
for _ in range(5):
    g.vcycle(bd, z)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.vcycle(bd, z)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{cfg.name} {os.environ.get('HMG_COOP_REF', 'default')}: V-cycle median {np.median(ts) * 1e3:.1f} us, "
      f"min {np.min(ts) * 1e3:.1f} us")
