"""Multi-rank run of the distributed path on ONE GPU (HMG_TRANSPORT=local).

Spawned by tests/test_dist_local.py in a fresh process (the transport is
chosen when the library first resolves its NCCL table).  Every rank is a host
thread with its own CUDA stream; the library's collectives go through the
in-process transport (csrc/local_transport.cu), which only orders streams with
events -- no kernel waits on another rank.  Prints one JSON line: per-check
booleans comparing the distributed results with the ORACLE (oracle/, the
global problem on the host): apply, V(2,2) and V(1,3) cycles and the public
restriction calls bitwise, PCG the oracle's iteration count.
Usage: python tests/dist_local_worker.py NRANKS FINE_REF NZ GATHER_REF [ANISO]
(ANISO: C2a / C2b / C2c thickness and w2; default C2b's 0.001, 1e-5)
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
import oracle  # noqa: E402
from paper_1605_00492_b200 import Hierarchy, MGParams, nccl_unique_id  # noqa: E402

P, fine, nz, gref = (int(a) for a in sys.argv[1:5])
aniso = hi.CONFIGS[sys.argv[5] if len(sys.argv) > 5 else "C2b"]
T, W2 = aniso.thickness, aniso.w2
cfg = hi.Config("dist", fine, 0, nz, T, W2)
lam, b = hi.make_inputs(cfg)
x0 = hi.uniform_vector(b.shape, 11)
nid = nccl_unique_id()
PARAMS = {"v22": MGParams(), "v13": MGParams(1, 3, 5, 0.9)}

# the oracle on the global problem (host; test infrastructure)
o = oracle.Hierarchy(fine, 0, nz, T, W2, lam)
ref_apply = o.apply(fine, x0)
ref_v = {name: o.vcycle(b, p.nu_pre, p.nu_post, p.n_coarse, p.omega) for name, p in PARAMS.items()}
_, it_o, _, _, st_o = o.pcg(b, rtol=1e-8)
# public residual + restriction calls on two levels: the finest (coarser level
# distributed unless gather_ref = fine - 1) and gather_ref + 1 (coarser level
# replicated: the output is the whole coarse vector on every rank)
rr_levels = sorted({fine, gref + 1})
u_lev, b_lev, ref_rr, ref_r = {}, {}, {}, {}
for r in rr_levels:
    n_r = hi.ncells(r)
    u_lev[r] = hi.uniform_vector((nz, n_r), 20 + r)
    b_lev[r] = hi.uniform_vector((nz, n_r), 40 + r)
    ref_rr[r] = o.restrict(r, o.residual(r, b_lev[r], u_lev[r]))
    ref_r[r] = o.restrict(r, b_lev[r])
o.close()

results = [None] * P
errors = []


def own(r, ref):
    per = hi.ncells(ref) // P
    return slice(r * per, (r + 1) * per)


def rank_main(r):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            sl = own(r, fine)
            h = Hierarchy(fine, 0, nz, T, W2, np.ascontiguousarray(lam[:, sl]), dist=(r, P, nid, gref))
            out = {}
            out["apply"] = h.to_host(fine, h.apply_helmholtz(fine, h.to_device(fine, x0[:, sl])))
            for name, prm in PARAMS.items():
                out[name] = h.to_host(fine, h.vcycle(h.to_device(fine, b[:, sl]), params=prm))
            for lv in rr_levels:
                so = own(r, lv)
                ud, bd = h.to_device(lv, u_lev[lv][:, so]), h.to_device(lv, b_lev[lv][:, so])
                out[f"rr{lv}"] = h.to_host(lv - 1, h.residual_restrict(lv, bd, ud))
                out[f"r{lv}"] = h.to_host(lv - 1, h.restrict(lv, bd))
            x, it, rr, st = h.pcg_solve(h.to_device(fine, b[:, sl]))
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


def coarse_ok(key, ref_val, lv):
    """Coarse level lv - 1 distributed: the ranks' parts concatenate to the
    oracle's vector; replicated (lv - 1 <= gather_ref): every rank holds it whole."""
    if lv - 1 > gref:
        return bool(np.array_equal(cat(key), ref_val))
    return all(bool(np.array_equal(results[r][key], ref_val)) for r in range(P))


print(json.dumps({
    "apply_bitwise": bool(np.array_equal(cat("apply"), ref_apply)),
    "v22_bitwise": bool(np.array_equal(cat("v22"), ref_v["v22"])),
    "v13_bitwise": bool(np.array_equal(cat("v13"), ref_v["v13"])),
    "resid_restrict_bitwise": {str(lv): coarse_ok(f"rr{lv}", ref_rr[lv], lv) for lv in rr_levels},
    "restrict_bitwise": {str(lv): coarse_ok(f"r{lv}", ref_r[lv], lv) for lv in rr_levels},
    "pcg_iters": [results[r]["it"] for r in range(P)], "pcg_iters_oracle": it_o, "oracle_status": st_o,
    "pcg_status": [results[r]["st"] for r in range(P)],
}))
