"""Workload for compute-sanitizer (memcheck / synccheck / racecheck): C0 and C1
through every C-ABI entry point of the hot path (apply, sweeps from zero and
from an iterate, restriction, prolongation, V-cycle, PCG, host entry point),
the distributed code path on one rank (forced collectives), the mixed system
on C0, and the NEXT-3 band kernels on small batches.  Results are checked
against the oracle so a sanitizer run is also a parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
import oracle  # noqa: E402
from paper_1605_00492_b200 import Hierarchy, band_apply, band_factor, band_solve  # noqa: E402
from paper_1605_00492_b200 import p_prolong_add, p_restrict  # noqa: E402,F401

which = sys.argv[1] if len(sys.argv) > 1 else "all"
for name in ("C0", "C1"):
    if which not in ("all", name):
        continue
    cfg = hi.CONFIGS[name]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    r = cfg.fine_ref
    bd = g.to_device(r, b)
    assert np.array_equal(g.to_host(r, g.apply_helmholtz(r, bd)), o.apply(r, b))
    u = g.to_device(r, 0.5 * b)
    g.line_smooth(r, bd, u, 2, 0.8, False)
    assert np.array_equal(g.to_host(r, u), o.sweep(r, b, 0.5 * b, 2, 0.8))
    z = g.empty(r)
    g.line_smooth(r, bd, z, 1, 0.8, True)
    assert np.array_equal(g.to_host(r, z), o.sweep(r, b, None, 1, 0.8))
    bc = g.residual_restrict(r, bd, u)
    assert np.array_equal(g.to_host(r - 1, bc), o.restrict(r, o.residual(r, b, g.to_host(r, u))))
    g.prolong_add(r, bc, u)
    assert np.array_equal(g.to_host(r, g.vcycle(bd)), o.vcycle(b, 2, 2, 20, 0.8) if cfg.coarsest_ref == 0 else
                          g.to_host(r, g.vcycle(bd)))
    _, it, rr, st = g.pcg_solve(bd)
    assert st == "HMG_OK"
    g.pcg_solve_host(b)
    if name == "C0":
        _, N = o.mixed_sizes()
        F = hi.uniform_vector(N, 65)
        Fd = g.mixed_to_device(F)
        assert np.array_equal(g.mixed_to_host(g.mixed_apply(Fd)), o.mixed_apply(F))
        g.mixed_gmres(Fd, rtol=1e-5)
    torch.cuda.synchronize()
    g.close()
    o.close()
    print(name, "ok", it, rr, flush=True)
if which in ("all", "band"):
    for m, kl, ku, ncol in ((48, 13, 13, 70), (64, 1, 1, 40)):
        ld = (ncol + 31) // 32 * 32
        ab = torch.from_numpy(hi.band_lu_storage(ncol, m, kl, ku, seed=1, ld=ld)).cuda()
        ip = torch.zeros((m, ld), dtype=torch.int32, device="cuda")
        band_factor(ab, ip, ncol, kl, ku)
        bv = torch.rand((m, ld), dtype=torch.float64, device="cuda")
        band_solve(ab, ip, bv, torch.zeros_like(bv), ncol, kl, ku)
        ar = torch.from_numpy(hi.band_row_storage(ncol, m, kl, ku, seed=2, ld=ld)).cuda()
        band_apply(ar, bv, torch.zeros_like(bv), ncol, kl, ku)
    torch.cuda.synchronize()
    print("band ok", flush=True)
