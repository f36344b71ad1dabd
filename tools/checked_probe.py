"""Checked-build run (the stand-in for compute-sanitizer, which the GPU pool
refuses): builds tools/micro/libhmg_checked.so with -DHMG_CHECKED -- device-side
bounds checks on every gathered index of the streamed kernels and a sequence
tag on every ring stage (producer writes the stage number, consumers check
it) -- and runs, against the oracle: the sanitize_probe workload (C0, C1,
mixed system, band kernels), the interleaved sweep on ref 6 with partial top
chunks (one and two CTAs per SM), and full-size C2b (apply, sweeps, V-cycle,
PCG count).  A failed check traps the kernel and the run fails."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B  # noqa: E402
from paper_1605_00492_b200 import build as pb  # noqa: E402

lib = os.path.join(HERE, "micro", "libhmg_checked.so")
if len(sys.argv) > 1 and sys.argv[1] == "--build":
    subprocess.check_call([pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], "-DHMG_CHECKED",
                           "-shared", *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", lib, "-ldl"])
    sys.exit(0)
B._LIB_PATH = lib
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
import oracle  # noqa: E402
from paper_1605_00492_b200 import Hierarchy  # noqa: E402

sys.argv = [sys.argv[0], "all"]
exec(open(os.path.join(HERE, "sanitize_probe.py")).read())


def check(cfg, sweeps=True):
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    r = cfg.fine_ref
    x = hi.uniform_vector(b.shape, 29)
    bd = g.to_device(r, b)
    assert np.array_equal(g.to_host(r, g.apply_helmholtz(r, g.to_device(r, x))), o.apply(r, x))
    if sweeps:
        u = g.to_device(r, x)
        g.line_smooth(r, bd, u, 2, 0.8, False)
        assert np.array_equal(g.to_host(r, u), o.sweep(r, b, x, 2, 0.8))
    assert np.array_equal(g.to_host(r, g.vcycle(bd)), o.vcycle(b, 2, 2, 20, 0.8))
    _, it, _, st = g.pcg_solve(bd)
    assert st == "HMG_OK" and it == o.pcg(b)[1], (it, o.pcg(b)[1])
    torch.cuda.synchronize()
    g.close()
    o.close()
    print(cfg.name, "checked ok", it, flush=True)


for nz in (9, 60, 65, 100):
    check(hi.Config(f"ref6_nz{nz}", 6, 4, nz, 0.001, 1e-5))
check(hi.CONFIGS["C2b"], sweeps=False)
print("checked build: all ok")
