"""One rank of a real multi-GPU run over NCCL (launched by tests/test_nccl_multi.py
through torch.distributed.run, one process per GPU).

Every rank builds its part of the distributed hierarchy (hmg_build_hierarchy_dist,
the library's own NCCL communicator from a unique id broadcast over the torch
process group), runs the operator apply, V(2,2) and V(1,3) cycles, the public
residual + restriction call and a PCG solve, and rank 0 compares the gathered
parts with the ORACLE on the global problem: bitwise for the V-cycle path, the
oracle's iteration count for PCG.  Rank 0 prints one JSON line.
Usage (under torchrun): nccl_worker.py FINE_REF NZ GATHER_REF
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy, MGParams, nccl_unique_id  # noqa: E402

fine, nz, gref = (int(a) for a in sys.argv[1:4])
rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
cfg = hi.Config("nccl", fine, 0, nz, 0.001, 1e-5)
lam, b = hi.make_inputs(cfg)
x0 = hi.uniform_vector(b.shape, 11)
PARAMS = {"v22": MGParams(), "v13": MGParams(1, 3, 5, 0.9)}

nid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
if rank == 0:
    nid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(nid, 0)
per = cfg.n // ws
sl = slice(rank * per, (rank + 1) * per)
h = Hierarchy(fine, 0, nz, 0.001, 1e-5, np.ascontiguousarray(lam[:, sl]), device=local,
              dist=(rank, ws, bytes(nid.cpu().numpy()), gref))
out = {"apply": h.to_host(fine, h.apply_helmholtz(fine, h.to_device(fine, x0[:, sl])))}
for name, prm in PARAMS.items():
    out[name] = h.to_host(fine, h.vcycle(h.to_device(fine, b[:, sl]), params=prm))
u1 = hi.uniform_vector(b.shape, 21)
out["rr"] = h.to_host(fine - 1, h.residual_restrict(fine, h.to_device(fine, b[:, sl]), h.to_device(fine, u1[:, sl])))
_, it, rr, st = h.pcg_solve(h.to_device(fine, b[:, sl]))
out["it"], out["st"] = it, st
torch.cuda.synchronize()
h.close()
parts = [None] * ws
dist.all_gather_object(parts, out)
if rank == 0:
    import oracle
    o = oracle.Hierarchy(fine, 0, nz, 0.001, 1e-5, lam)
    cat = lambda k: np.concatenate([p[k] for p in parts], axis=1)  # noqa: E731
    ref_rr = o.restrict(fine, o.residual(fine, b, u1))
    rr_ok = (bool(np.array_equal(cat("rr"), ref_rr)) if fine - 1 > gref
             else all(bool(np.array_equal(p["rr"], ref_rr)) for p in parts))
    res = {
        "nranks": ws,
        "apply_bitwise": bool(np.array_equal(cat("apply"), o.apply(fine, x0))),
        "v22_bitwise": bool(np.array_equal(cat("v22"), o.vcycle(b))),
        "v13_bitwise": bool(np.array_equal(cat("v13"), o.vcycle(b, 1, 3, 5, 0.9))),
        "resid_restrict_bitwise": rr_ok,
        "pcg_iters": [p["it"] for p in parts], "pcg_status": [p["st"] for p in parts],
        "pcg_iters_oracle": o.pcg(b, rtol=1e-8)[1],
    }
    o.close()
    print(json.dumps(res))
dist.barrier()
dist.destroy_process_group()
