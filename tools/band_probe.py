"""NEXT-3 probe: N2 (81,920 columns x 384 rows, kl = ku = 13) factor, solve and
apply, for ncu captures of k_gbtrs / k_gbmv (tools/gpu_runs/r02*.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import band_apply, band_factor, band_solve  # noqa: E402

ref, nz = hi.NLO_CONFIGS["N2"]
ncol, m, kl, ku = 20 * 4 ** ref, 6 * nz, 13, 13
ld = (ncol + 31) // 32 * 32
g = torch.Generator(device="cuda")
g.manual_seed(2)
ab = torch.zeros((m, 2 * kl + ku + 1, ld), dtype=torch.float64, device="cuda")
ab[:, kl:, :ncol] = torch.rand((m, kl + ku + 1, ncol), generator=g, dtype=torch.float64, device="cuda") * 2 - 1
ip = torch.zeros((m, ld), dtype=torch.int32, device="cuda")
band_factor(ab, ip, ncol, kl, ku)
b = torch.rand((m, ld), generator=g, dtype=torch.float64, device="cuda")
x = torch.zeros_like(b)
for _ in range(3):
    band_solve(ab, ip, b, x, ncol, kl, ku)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    band_solve(ab, ip, b, x, ncol, kl, ku)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"solve {ms * 1e3:.1f} us  {ncol * 4 * m * (3 * 27 + 4) / ms / 1e6:.1f} GB/s (Eq. 15)")
del ab
ar = torch.rand((m, kl + ku + 1, ld), generator=g, dtype=torch.float64, device="cuda")
for _ in range(3):
    band_apply(ar, b, x, ncol, kl, ku)
e0.record()
for _ in range(10):
    band_apply(ar, b, x, ncol, kl, ku)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"apply {ms * 1e3:.1f} us  {ncol * 8 * m * 29 / ms / 1e6:.1f} GB/s (Eq. 14)")
print("ok")
