"""The multi-GPU path over REAL NCCL (one process per GPU, torch.distributed.run),
compared with the oracle: distributed apply and V-cycles bitwise, PCG the
oracle's iteration count.  Skipped when fewer than 2 GPUs are visible (the
round's GPU boxes have one; the in-process-transport test test_dist_local.py
covers the same library code there).  Also: bench.py --gpus N starts its N
ranks itself and refuses to run with fewer GPUs than asked for."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,fine,nz,gref", [(2, 5, 16, 3), (2, 6, 64, 3), (4, 5, 24, 2), (8, 6, 16, 3)])
def test_nccl_distributed_matches_oracle(nranks, fine, nz, gref):
    if _ngpus() < nranks:
        pytest.skip(f"needs {nranks} GPUs, {_ngpus()} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "nccl_worker.py"),
           str(fine), str(nz), str(gref)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["apply_bitwise"] and out["v22_bitwise"] and out["v13_bitwise"], out
    assert out["resid_restrict_bitwise"], out
    assert all(s == "HMG_OK" for s in out["pcg_status"]), out
    assert out["pcg_iters"] == [out["pcg_iters_oracle"]] * nranks, out


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N (no torchrun) launches N ranks itself; with fewer than N
    visible GPUs it exits non-zero naming the shortfall instead of silently
    running one GPU."""
    n = max(2, _ngpus() + 1)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode != 0
    assert f"--gpus {n}: only" in res.stderr


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 4" in res.stderr
