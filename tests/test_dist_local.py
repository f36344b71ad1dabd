"""The multi-GPU path run on ONE GPU: P ranks as threads of one
process, collectives through the in-process transport (HMG_TRANSPORT=local,
csrc/local_transport.cu).  Partition, halo pack/send/recv/unpack on every
distributed level, all-reduced CG dots and the coarse all-gather all run on the
device; the distributed V-cycle must be bitwise the 1-GPU one (halos move exact
values, the replicated tail runs the same arithmetic) and PCG must take the
same number of iterations (dots differ only in summation order).  The last case
has 163,840 owned cells per rank on the finest level, so the streamed sweep
kernels (no precomputed pivots) run with distributed halos."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nranks,fine,nz,gref", [(2, 4, 16, 2), (4, 5, 24, 3), (5, 5, 8, 2), (8, 6, 16, 3), (2, 7, 8, 3)])
def test_distributed_solve_matches_single_gpu(nranks, fine, nz, gref):
    env = dict(os.environ, HMG_TRANSPORT="local")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dist_local_worker.py"), str(nranks), str(fine),
                          str(nz), str(gref)], capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["apply_bitwise"] and out["v22_bitwise"] and out["v13_bitwise"], out
    assert all(s == "HMG_OK" for s in out["pcg_status"]), out
    assert out["pcg_iters"] == [out["pcg_iters_1gpu"]] * nranks, out
    assert out["x_rel_err"] < 1e-10, out
