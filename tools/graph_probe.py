"""Is the V-cycle launch-bound?  Eager hmg_vcycle vs the same calls captured
into a CUDA graph with torch.cuda.graph (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy  # noqa: E402

cfg = hi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2b"]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
r = cfg.fine_ref
bd = g.to_device(r, b)
z = g.empty(r)
x = g.empty(r)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"eager V-cycle {t(lambda: g.vcycle(bd, z)):.1f} us")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    g.vcycle(bd, z)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        g.vcycle(bd, z)
print(f"graph V-cycle {t(lambda: gr.replay()):.1f} us")
print(f"eager PCG {t(lambda: g.pcg_solve(bd, x), 5):.1f} us")
