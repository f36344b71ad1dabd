"""Quick CUDA-event timing of the C2a kernels through the C-ABI (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy, MGParams

name = sys.argv[1] if len(sys.argv) > 1 else "C2a"
cfg = hi.CONFIGS[name]
lam, b = hi.make_inputs(cfg)
t0 = time.time()
g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
print(f"setup {time.time()-t0:.2f}s")
r = cfg.fine_ref
bd = g.to_device(r, b)
x = g.to_device(r, hi.uniform_vector(b.shape, 5))
y = g.empty(r)
flush = torch.empty(int(300e6) // 4, dtype=torch.float32, device="cuda")
ndof = cfg.ndofs

def timeit(fn, reps=20, fl=True):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if fl: flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.median(ts)

t = timeit(lambda: g.apply_helmholtz(r, x, y))
print(f"apply   {t*1e3:8.1f} us  {56*ndof/t/1e6:8.1f} GB/s (56 B/dof)")
u = g.empty(r)
t = timeit(lambda: g.line_smooth(r, bd, u, 1, 0.8, True))
print(f"sweep0  {t*1e3:8.1f} us  {32*ndof/t/1e6:8.1f} GB/s (32 B/dof, incl. flag sync)")
u2 = x.clone()
t = timeit(lambda: g.line_smooth(r, bd, u2, 1, 0.8, False))
print(f"sweep   {t*1e3:8.1f} us  {64*ndof/t/1e6:8.1f} GB/s (64 B/dof, incl copy+sync)")
t = timeit(lambda: g.residual_restrict(r, bd, x))
print(f"resres  {t*1e3:8.1f} us  {58*ndof/t/1e6:8.1f} GB/s")
z = g.empty(r)
t = timeit(lambda: g.vcycle(bd, z), reps=10)
print(f"vcycle  {t*1e3:8.1f} us  {ndof/t/1e6:8.3f} Gdof/s")
t0 = time.time()
xx, it, rr, st = g.pcg_solve(bd); torch.cuda.synchronize()
print(f"pcg warm {time.time()-t0:.3f}s it={it} rr={rr:.2e} {st}")
t = timeit(lambda: g.pcg_solve(bd, xx), reps=3)
print(f"pcg     {t:8.2f} ms  it={it}")

# per-class, per-level breakdown of one V-cycle (library CUDA events)
g.profile_begin()
g.vcycle(bd, z)
torch.cuda.synchronize()
g.profile_end()
tot = 0.0
for cls in g.KERNEL_CLASSES:
    for lev in range(cfg.fine_ref, -1, -1):
        n_, ms_ = g.profile_query(cls, lev)
        if n_:
            tot += ms_
            print(f"  {cls:15s} ref {lev}: {n_:3d} launches {ms_*1e3:9.1f} us")
print(f"  sum of kernel time {tot*1e3:.1f} us")
