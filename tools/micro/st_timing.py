"""Where a streamed sweep CTA spends its time (CTA 0, consumer thread 0), from a
-DHMG_TIMING build: total cycles, cycles waiting for forward / backward stages."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_1605_00492_b200.binding as B
from paper_1605_00492_b200 import build as pb
extra = sys.argv[1:]          # e.g. -DHMG_PROBE_NOMOVE
REFS = [int(r) for r in os.environ.get("REFS", "7,6,5").split(",")]   # one level per process: clean CTA stamps
lib = os.path.join(HERE, f"libhmg_timing{len(extra)}.so")
cmd = [pb.NVCC, *pb.ARCH, *[f for f in pb.FLAGS if f not in ("-Xptxas", "-v")], "-DHMG_TIMING", *extra, "-shared",
       *[os.path.join(pb.CSRC, s) for s in pb.SOURCES], "-o", lib, "-ldl"]
if not os.path.exists(lib) or os.environ.get("REBUILD"):
    subprocess.check_call(cmd)
B._LIB_PATH = lib
import torch
import hmg_inputs as hi
from paper_1605_00492_b200 import Hierarchy
print(" ".join(extra) or "normal")
for ref in REFS:
    cfg = hi.Config("t", ref, ref - 1 if ref > 5 else 4, 64, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(ref, cfg.coarsest_ref, 64, 0.001, 1e-5, lam)
    bd = g.to_device(ref, b)
    u = g.to_device(ref, hi.uniform_vector(b.shape, 3))
    om = float(os.environ.get("OMEGA", "0.8"))
    for _ in range(3):
        g.line_smooth(ref, bd, u, 1, om, False)
    torch.cuda.synchronize()
    t = (ctypes.c_longlong * 12)()
    B.load_library().hmg_debug_st_timing(t)
    tot, wf, wb, nt, tf, tb, tws = t[0], t[1], t[2], t[3], t[4], t[5], t[6]
    print(f"ref {ref}: tiles/CTA {nt}, total {tot} cyc = {tot/1965:.1f} us, per tile {tot/max(nt,1)/1965:.1f} us; "
          f"waiting fwd {wf/tot:.0%} bwd {wb/tot:.0%}; forward phase {tf/max(nt,1)/64:.0f} cyc/layer "
          f"(of which waiting {wf/max(nt,1)/64:.0f}), back phase incl. redo check {tb/max(nt,1)/64:.0f} cyc/layer, of which slow check + TMEM store wait {tws/max(nt,1)/64:.0f}; producer: {t[8]} cyc, waiting for free slots {t[9]/max(t[8],1):.0%}, forward stages {t[10]} ({(t[8]-t[9])/max(t[10],1):.0f} busy cyc per forward stage incl. backward issue, of which halo gathers {t[11]/max(t[10],1):.0f})")
    ns = (ctypes.c_ulonglong * 2048)()
    sm = (ctypes.c_uint * 1024)()
    B.load_library().hmg_debug_st_cta(ns, sm)
    ncta = next(i for i in range(1024) if ns[2 * i] == 0)
    st = [ns[2 * i] for i in range(ncta)]
    en = [ns[2 * i + 1] for i in range(ncta)]
    t0 = min(st)
    dur = sorted(en[i] - st[i] for i in range(ncta))
    print("  start offsets (us, sorted):", [round((x - t0) / 1e3, 2) for x in sorted(st)][::max(1, ncta // 16)])
    print("  end offsets (us, sorted):", [round((x - t0) / 1e3, 2) for x in sorted(en)][::max(1, ncta // 16)])
    print(f"  CTAs {ncta}: start spread {(max(st) - t0) / 1e3:.1f} us, end spread {(max(en) - min(en)) / 1e3:.1f} us, "
          f"kernel span {(max(en) - t0) / 1e3:.1f} us; CTA durations min {dur[0] / 1e3:.1f} median {dur[ncta // 2] / 1e3:.1f} "
          f"max {dur[-1] / 1e3:.1f} us")
    from collections import Counter
    per_sm = Counter(sm[i] for i in range(ncta))
    lone = [i for i in range(ncta) if per_sm[sm[i]] == 1]
    if lone:
        print(f"  {len(lone)} CTAs alone on their SM: durations {sorted(round((en[i] - st[i]) / 1e3, 1) for i in lone)[:6]} us")
    g.close()
