"""The multi-GPU path run on ONE GPU: P ranks as threads of one
process, collectives through the in-process transport (HMG_TRANSPORT=local,
csrc/local_transport.cu, a test-only transport).  Partition, halo
pack/send/recv/unpack on every distributed level, all-reduced CG dots and the
coarse all-gather all run on the device.  Compared with the ORACLE on the
global problem: the distributed apply, V(2,2) and V(1,3) cycles and the public
restriction calls must be bitwise the oracle's (halos move exact values, the
replicated tail runs the same arithmetic) and PCG must take the oracle's
number of iterations (dots differ only in summation order).  The ref-7 cases
have >= 81,920 owned cells per rank on the finest level, so the streamed
sweep kernels (no precomputed pivots) run with distributed halos; the last is
BASELINE.json's C3 problem (C2a, ref 7 x 64, 20.97M dofs) strong-scaled over 4
ranks."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [(2, 4, 16, 2, "C2b"), (4, 5, 24, 3, "C2b"), (5, 5, 8, 2, "C2b"), (8, 6, 16, 3, "C2b"), (2, 7, 8, 3, "C2b"),
         (2, 6, 16, 5, "C2a"), pytest.param(4, 7, 64, 3, "C2a", marks=pytest.mark.slow)]


@pytest.mark.parametrize("nranks,fine,nz,gref,aniso", CASES)
def test_distributed_solve_matches_oracle(nranks, fine, nz, gref, aniso):
    env = dict(os.environ, HMG_TRANSPORT="local")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dist_local_worker.py"), str(nranks), str(fine),
                          str(nz), str(gref), aniso], capture_output=True, text=True, env=env, timeout=1200)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["apply_bitwise"] and out["v22_bitwise"] and out["v13_bitwise"], out
    assert all(out["resid_restrict_bitwise"].values()) and all(out["restrict_bitwise"].values()), out
    assert out["oracle_status"] == 0 and all(s == "HMG_OK" for s in out["pcg_status"]), out
    assert out["pcg_iters"] == [out["pcg_iters_oracle"]] * nranks, out
