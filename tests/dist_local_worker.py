"""Multi-rank run of the distributed path on ONE GPU (HMG_TRANSPORT=local).

Spawned by tests/test_dist_local.py in a fresh process (the transport is
chosen when the library first resolves its NCCL table).  Every rank is a host
thread with its own CUDA stream; the library's collectives go through the
in-process transport (csrc/local_transport.cu), which only orders streams with
events -- no kernel waits on another rank.  Prints one JSON line: per-check
booleans comparing the distributed results with the 1-GPU hierarchy.
Usage: python tests/dist_local_worker.py NRANKS FINE_REF NZ GATHER_REF
"""
import json
import os
import sys
import threading

os.environ["HMG_TRANSPORT"] = "local"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hmg_inputs as hi  # noqa: E402
from paper_1605_00492_b200 import Hierarchy, MGParams, nccl_unique_id  # noqa: E402

P, fine, nz, gref = (int(a) for a in sys.argv[1:5])
cfg = hi.Config("dist", fine, 0, nz, 0.001, 1e-5)
lam, b = hi.make_inputs(cfg)
x0 = hi.uniform_vector(b.shape, 11)
n = cfg.n
per = n // P
nid = nccl_unique_id()

# 1-GPU reference (its own stream)
g1 = Hierarchy(fine, 0, nz, 0.001, 1e-5, lam)
ref_apply = g1.to_host(fine, g1.apply_helmholtz(fine, g1.to_device(fine, x0)))
ref_v = {}
for name, prm in (("v22", MGParams()), ("v13", MGParams(1, 3, 5, 0.9))):
    ref_v[name] = g1.to_host(fine, g1.vcycle(g1.to_device(fine, b), params=prm))
xr, it1, rr1, st1 = g1.pcg_solve(g1.to_device(fine, b))
ref_x = g1.to_host(fine, xr)
torch.cuda.synchronize()

results = [None] * P
errors = []


def rank_main(r):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            own = slice(r * per, (r + 1) * per)
            h = Hierarchy(fine, 0, nz, 0.001, 1e-5, np.ascontiguousarray(lam[:, own]), dist=(r, P, nid, gref))
            out = {}
            out["apply"] = h.to_host(fine, h.apply_helmholtz(fine, h.to_device(fine, x0[:, own])))
            for name, prm in (("v22", MGParams()), ("v13", MGParams(1, 3, 5, 0.9))):
                out[name] = h.to_host(fine, h.vcycle(h.to_device(fine, b[:, own]), params=prm))
            x, it, rr, st = h.pcg_solve(h.to_device(fine, b[:, own]))
            out["x"] = h.to_host(fine, x)
            out["it"], out["st"] = it, st
            s.synchronize()
            h.close()
            results[r] = out
    except Exception as e:  # pragma: no cover - reported to the parent test
        errors.append(f"rank {r}: {e!r}")


threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
for t in threads:
    t.start()
for t in threads:
    t.join()
if errors:
    print(json.dumps({"errors": errors}))
    sys.exit(1)


def cat(key):
    return np.concatenate([results[r][key] for r in range(P)], axis=1)


rel = lambda a, c: float(np.max(np.abs(a - c)) / np.max(np.abs(c)))  # noqa: E731
print(json.dumps({
    "apply_bitwise": bool(np.array_equal(cat("apply"), ref_apply)),
    "v22_bitwise": bool(np.array_equal(cat("v22"), ref_v["v22"])),
    "v13_bitwise": bool(np.array_equal(cat("v13"), ref_v["v13"])),
    "pcg_iters": [results[r]["it"] for r in range(P)], "pcg_iters_1gpu": it1,
    "pcg_status": [results[r]["st"] for r in range(P)],
    "x_rel_err": rel(cat("x"), ref_x),
}))
