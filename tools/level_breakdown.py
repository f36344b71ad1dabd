"""Per-level, per-kernel-class time of a V-cycle and of a PCG solve (dev tool).

Uses the library's CUDA-event profiler (hmg_profile_*); the difference between
the summed kernel time and the wall time is launch gaps / host syncs.
Usage: python tools/level_breakdown.py [C2b]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy, MGParams  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2b"
cfg = hi.CONFIGS[name]
lam, b = hi.make_inputs(cfg)
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
r = cfg.fine_ref
bd = g.to_device(r, b)
z = g.empty(r)
x = g.empty(r)
p = MGParams()
classes = list(Hierarchy.KERNEL_CLASSES)


def run(label, fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.profile_begin()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    g.profile_end()
    wall = e0.elapsed_time(e1) / reps * 1e3
    print(f"== {label}: {wall:.1f} us per call")
    tot = 0.0
    for ref in range(r, -1, -1):
        row = []
        lev = 0.0
        for c in classes:
            n, ms = g.profile_query(c, ref)
            if n:
                us = ms * 1e3 / reps
                lev += us
                row.append(f"{c}={us:.1f}({n // reps})")
        tot += lev
        if row:
            print(f"  ref {ref}: {lev:8.1f} us  " + "  ".join(row))
    print(f"  kernels {tot:.1f} us, gaps {wall - tot:.1f} us")


run("V-cycle", lambda: g.vcycle(bd, z, p), 20)
run("PCG solve", lambda: g.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=p), 5)
