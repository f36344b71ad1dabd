#!/usr/bin/env python
"""Benchmark of the B200 tensor-product multigrid Helmholtz solver (arXiv:1605.00492 hot path).

One step = one full solve of BASELINE.json config C2 (anisotropy C2b: ref 7 x 64
layers = 20,971,520 fp64 dofs, thickness 0.001, w2 1e-5, hierarchy ref 7 -> 0,
PCG preconditioned by one V(2,2) cycle per iteration, damped line-Jacobi
omega = 0.8, 20 coarse sweeps, relative residual 1e-8).  C2b is the C2
anisotropy that BASELINE.json's weak-scaling config C4 (thickness 0.001) pairs
with.  Every row of SURVEY.md 8(a) runs inside the step:
operator apply, fused sweeps, residual+restriction, prolongation, the coarse
solve, the V-cycle driver and the PCG vector/dot kernels.

Metric (BASELINE.json): fp64 Helmholtz dofs/s per V-cycle = fine dofs x
V-cycles executed in the step / step time (the PCG's own apply and vector
work is included in the time, so this under-states the bare V-cycle rate,
which is reported as `vcycle_only`).  Also reported: PCG solve time, the
dominant kernel's achieved HBM GB/s against MEASURED_PEAKS.json, the oracle on
the host cores, and an end-to-end number through the host-buffer entry point.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Multi-GPU (torchrun, N > 1): ONE distributed solve over NCCL (SURVEY 8(e):
horizontal partition by ref-2 blocks, one-ring halo exchange on every
distributed level, all-reduced CG inner products, coarse gather at ref 3).
Weak scaling at 20,971,520 dofs per GPU, thickness 0.001, w2 1e-5:
N=1 ref 7 x 64 (C2b), N=2 ref 7 x 128, N=4 ref 8 x 64, N=8 ref 8 x 128 (C4);
other N divide C2b (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hmg_inputs as hi  # noqa: E402

METRIC = "fp64 Helmholtz dofs/s per V-cycle"
UNIT = "dof/s"
# Algorithmic bytes per dof of each kernel class
BYTES_PER_DOF = {"sweep": 64.0, "sweep_zero": 32.0, "sweep_prolong": 66.0, "apply": 56.0, "apply_pupdate": 72.0,
                 "resid_restrict": 58.0}
# The streamed kernels (general sweep with or without the fused prolongation,
# apply, streamed residual + restriction; not the apply with the p update) do not read D:
# their consumers re-form D_k from the prism volume and the streamed couplings
# (DESIGN 7.7), 8 B/dof less than the per-cell store's figure above.
D_REFORMED = 8.0


def store_bytes(es: dict) -> dict:
    """Bytes per dof each fine-level kernel class actually reads and writes on a
    level with edge-store flags `es` (hmg_edge_store): the edge-deduplicated
    couplings save 12 B/dof, the re-formed diagonal 8."""
    bpd = dict(BYTES_PER_DOF)
    for k in ("sweep", "sweep_prolong", "apply"):
        bpd[k] -= D_REFORMED
    if es["sweep"]:
        bpd["sweep"] -= 12.0
        bpd["sweep_prolong"] -= 12.0
    if es["apply"]:
        bpd["apply"] -= 12.0
        bpd["apply_pupdate"] -= 12.0
    if es["resid_restrict"]:            # the streamed residual (k_apply_st): edge store and re-formed D
        bpd["resid_restrict"] -= 12.0 + D_REFORMED
    return bpd


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hmg", choices=["hmg", "reference"])
    ap.add_argument("--config", default="C2b", choices=["C2a", "C2b", "C2c", "C0", "C1", "C4"])
    ap.add_argument("--gather-ref", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config: str, edge: bool):
    """Per-launch DRAM bytes of the dominant kernel (the general fine-level sweep,
    with or without the edge store) from the committed ncu capture of the same
    configuration (null when no capture of this config exists)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            kernels = json.load(fh).get(config, {})
    except Exception:
        return None
    for chk in (0, 1):
        name = f"k_sweep_st<0, 0, 0, 2, {chk}, 0, 1>" if edge else f"k_sweep_st<0, 0, 0, 2, {chk}, 0>"
        if name in kernels:
            return kernels[name]
    return None


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id, self.lines, self.proc = gpu_id, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_baseline(cfg, lam, b, cores: int) -> dict:
    """The oracle as it stands on the host cores: the full PCG +
    V(2,2) solve to 1e-8 on all cores (the metric's own unit: fine dofs x
    V-cycles / solve time), and one V(2,2) cycle on ONE thread.  Bounded: about
    10-30 s of CPU work at C2 size."""
    import oracle
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    oracle.set_threads(cores)
    t0 = time.perf_counter()
    _, it, rel, hist, st = h.pcg(b, rtol=1e-8)
    t_pcg = time.perf_counter() - t0
    oracle.set_threads(1)
    t0 = time.perf_counter()
    h.vcycle(b, 2, 2, 20, 0.8)
    t_one = time.perf_counter() - t0
    oracle.set_threads(cores)
    h.close()
    nv = it                      # V-cycles in the solve: 1 before the loop + 1 per non-final iteration
    return {"value": cfg.ndofs * nv / t_pcg, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"one oracle PCG + V(2,2) solve of {cfg.name} to 1e-8 ({it} iterations, {nv} V-cycles, "
                      f"{cfg.ndofs} dofs) on {cores} threads: {t_pcg:.2f} s",
            "pcg_solve_s": t_pcg, "pcg_iterations": it, "residual_history": [float(v) for v in hist],
            "single_thread": {"value": cfg.ndofs / t_one, "unit": UNIT, "cores": 1,
                              "sample": f"one oracle V(2,2) cycle over {cfg.ndofs} dofs on 1 thread: {t_one:.2f} s"}}


def run_reference(args, ws, rank):
    """--impl reference: the oracle (the paper-defined CPU program of this
    repo, oracle/) timed as it stands on the host cores; rank 0 only.  One step
    = one oracle V(2,2) cycle over the whole workload (~1.5 s on 16 cores for
    C2b), so the default 100 timed steps end within a few minutes."""
    if rank != 0:
        return
    cfg = hi.CONFIGS[args.config]
    lam, b = hi.make_inputs(cfg)
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    import oracle
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    for _ in range(args.warmup):
        h.vcycle(b, 2, 2, 20, 0.8)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        h.vcycle(b, 2, 2, 20, 0.8)
        times.append(time.perf_counter() - t0)
    h.close()
    t = float(np.mean(times))
    value = cfg.ndofs / t
    sample = f"one oracle V(2,2) cycle over all {cfg.ndofs} dofs of {cfg.name} per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: ref {cfg.fine_ref}->0 x {cfg.nz} layers, {cfg.ndofs} dofs, "
                               f"t={cfg.thickness}, w2={cfg.w2}", "params": "V(2,2) omega 0.8, 20 coarse sweeps"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


WEAK = {1: (7, 64), 2: (7, 128), 4: (8, 64), 8: (8, 128)}   # (fine ref, layers): 20,971,520 dofs per GPU


def workload(args, ws):
    base = hi.CONFIGS[args.config]
    if ws == 1:
        return base, "weak"
    if ws in WEAK and args.config == "C2b":
        ref, nz = WEAK[ws]
        return hi.Config(f"C2b-weak-x{ws}" if ws != 8 else "C4", ref, 0, nz, 0.001, 1e-5), "weak"
    return base, "strong"


def run_hmg(args, ws, rank, local):
    import torch
    import torch.distributed as dist
    from paper_1605_00492_b200 import Hierarchy, MGParams, nccl_unique_id

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (no CPU fallback exists)")
    torch.cuda.set_device(local)
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg, scaling = workload(args, ws)
    lam, b = hi.make_inputs(cfg)                 # the global problem (seeded); each rank keeps its part
    t0 = time.perf_counter()
    if ws == 1:
        h = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, device=local)
    else:
        nid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            nid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(nid, 0)
        # the finest level is always distributed (gather_ref < fine_ref), so each
        # rank passes its owned part of lam and b (include/hmg.h)
        gref = max(2, min(args.gather_ref, cfg.fine_ref - 1))
        if cfg.fine_ref <= 2:
            raise SystemExit(f"{cfg.name}: fine ref {cfg.fine_ref} has no level to distribute (needs ref > 2)")
        per = cfg.n // ws
        own = slice(rank * per, (rank + 1) * per)
        lam, b = np.ascontiguousarray(lam[:, own]), np.ascontiguousarray(b[:, own])
        h = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, device=local,
                      dist=(rank, ws, bytes(nid.cpu().numpy()), gref))
    setup_s = time.perf_counter() - t0
    r = cfg.fine_ref
    bd = h.to_device(r, b)
    x = h.empty(r)
    params = MGParams()
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up ------------------------------------------------------------
    iters = None
    for _ in range(max(args.warmup, 3)):
        _, iters, relres, st = h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
    assert st == "HMG_OK", st
    nv = iters  # V-cycles per solve: 1 before the loop + 1 per non-final iteration

    # ---- timed region: K full solves, CUDA events on the launching stream ----
    props = torch.cuda.get_device_properties(local)
    gpu_id = f"GPU-{props.uuid}" if hasattr(props, "uuid") else str(local)
    launches0 = h.launches
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_id) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            _, it, relres, st = h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
            assert it == iters and st == "HMG_OK"
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = h.launches - launches0
    value = cfg.ndofs * nv / (ms * 1e-3)        # cfg is the global problem

    # ---- the same K steps again, with CUDA events around every launch of the
    # dominant kernel (an event pair between two kernels serialises them and
    # costs the sweep its programmatic-launch overlap, so the pass that gives
    # `value` above runs without them) ----
    h.profile_select("sweep", cfg.fine_ref)
    h.profile_begin()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
    e1.record(stream)
    barrier()
    h.profile_end()
    ms_events = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # ---- dominant kernel: the fused line-Jacobi sweep on the finest level ----
    # algorithmic bytes of the store the kernels actually read: with the
    # edge-deduplicated coupling store 1.5 couplings per dof instead of 3 (12 B
    # less), and D re-formed in the streamed kernels (8 B less)
    es = h.edge_store(r)
    bpd = store_bytes(es)
    n_sw, ms_sw = h.profile_query("sweep", r)
    avg_sw = ms_sw / max(n_sw, 1)
    dofs_local = cfg.ndofs // ws
    bytes_sw = bpd["sweep"] * dofs_local
    peak, peak_note = measured_peak()
    achieved = bytes_sw / (avg_sw * 1e-3) / 1e9
    # per-class breakdown: two further solves with every launch recorded (untimed)
    h.profile_select(None)
    h.profile_begin()
    prof_steps = 2
    for _ in range(prof_steps):
        h.pcg_solve(bd, x, rtol=1e-8, maxit=200, params=params)
    barrier()
    h.profile_end()
    shares = {}
    for k in ("sweep", "sweep_zero", "sweep_prolong", "apply", "apply_pupdate", "resid_restrict", "restrict", "prolong",
              "vector", "coarse_tail"):
        n_k, ms_k = h.profile_query(k, -1)
        shares[k] = round(ms_k / (ms * prof_steps), 4)
    fine = {}
    for k in ("sweep", "sweep_zero", "sweep_prolong", "apply", "apply_pupdate", "resid_restrict"):
        n_k, ms_k = h.profile_query(k, r)
        if n_k:
            avg = ms_k / n_k
            fine[k] = {"us": round(avg * 1e3, 2), "bytes_per_dof": bpd[k],
                       "GB/s": round(bpd[k] * dofs_local / (avg * 1e-3) / 1e9, 1)}

    hist = [float(v) for v in h.pcg_history()]
    levels = level_table(h, cfg, ws, bpd, r) if ws == 1 else None

    # ---- V-cycle alone -------------------------------------------------------
    z = h.empty(r)
    for _ in range(3):
        h.vcycle(bd, z, params)
    barrier()
    e0.record(stream)
    nvc = 20
    for _ in range(nvc):
        h.vcycle(bd, z, params)
    e1.record(stream)
    barrier()
    ms_vc = max_over_ranks(e0.elapsed_time(e1) / nvc)
    n = cfg.n // ws

    # ---- NEXT-1: the paper's single-level preconditioner (2 damped line sweeps,
    # P:815-817) in the same PCG, against the multigrid V-cycle ----
    sl = None
    if ws == 1:
        xs = h.empty(r)
        h.pcg_solve_single_level(bd, xs, nsweeps=2, omega=0.8, rtol=1e-8, maxit=2000)
        barrier()
        e0.record(stream)
        _, it_sl, rr_sl, st_sl = h.pcg_solve_single_level(bd, xs, nsweeps=2, omega=0.8, rtol=1e-8, maxit=2000)
        e1.record(stream)
        barrier()
        sl = {"preconditioner": "2 damped line-Jacobi sweeps (single level)", "pcg_iterations": it_sl,
              "status": st_sl, "solve_ms": e0.elapsed_time(e1), "final_relres": rr_sl,
              "multigrid_pcg_iterations": iters, "multigrid_solve_ms": ms}

    # ---- NEXT-4: the paper's outer solve -- the mixed velocity-pressure system
    # (Eq. 5, omega_N = 0) by right-preconditioned GMRES(30) to 1e-5 with the
    # Schur-complement preconditioner (Eq. 6, lumped mass + one V-cycle) ----
    mixed = None
    lay = h.mixed_layout() if ws == 1 else None
    # GMRES(30) keeps 31 basis vectors + 3 work vectors of the mixed system
    # (C2: 20 GB; C4 whole on one GPU would need 160 GB next to the hierarchy)
    need = 34 * 8 * lay["ntot"] if lay else 0
    if lay and need > 0.9 * torch.cuda.mem_get_info(local)[0]:
        mixed = {"skipped": f"GMRES(30) workspace {need / 1e9:.0f} GB does not fit next to the hierarchy"}
    elif lay:
        unknowns = lay["ne"] * cfg.nz + (cfg.nz - 1) * cfg.n + cfg.nz * cfg.n
        Fm = hi.uniform_vector(unknowns, 67)      # seeded U(-1, 1) over every unknown (reading R15)
        Fd = h.mixed_to_device(Fm)
        del Fm
        Xd = h.mixed_empty()
        h.mixed_gmres(Fd, Xd, rtol=1e-5, restart=30, maxit=300, params=params)
        barrier()
        h.profile_select(None)
        h.profile_begin()
        e0.record(stream)
        _, it_m, rr_m, st_m = h.mixed_gmres(Fd, Xd, rtol=1e-5, restart=30, maxit=300, params=params)
        e1.record(stream)
        barrier()
        h.profile_end()
        ms_m = e0.elapsed_time(e1)
        share = {k: round(h.profile_query(k, -1)[1] / ms_m, 4) for k in ("sweep", "sweep_zero", "sweep_prolong",
                                                                          "resid_restrict", "coarse_tail", "mixed")}
        # the same solve with ONE Gram-Schmidt pass (CGS, PETSc's default; reading R20)
        _, it_c, rr_c, st_c = h.mixed_gmres(Fd, Xd, rtol=1e-5, restart=30, maxit=300, params=params, gs_passes=1)
        mixed = {"solver": "right-preconditioned GMRES(30), CGS2, to ||r|| <= 1e-5 ||F||",
                 "single_pass_cgs": {"gmres_iterations": it_c, "status": st_c, "final_relres": rr_c},
                 "preconditioner": "Schur complement (Eq. 6) with two-point lumped velocity mass + one V(2,2)",
                 "unknowns": unknowns, "gmres_iterations": it_m, "status": st_m, "final_relres": rr_m,
                 "solve_ms": ms_m, "ms_per_iteration": ms_m / max(it_m, 1),
                 "unknowns_per_s_per_iteration": unknowns * it_m / (ms_m * 1e-3), "time_share": share}
        # with buoyancy (reading R24): omega_N = 1, i.e. the vertical velocity mass
        # doubled and the pressure operator's vertical couplings halved
        hb = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, device=local, omega_n=1.0)
        hb.mixed_gmres(Fd, Xd, rtol=1e-5, restart=30, maxit=300, params=params)
        barrier()
        e0.record(stream)
        _, it_b, rr_b, st_b = hb.mixed_gmres(Fd, Xd, rtol=1e-5, restart=30, maxit=300, params=params)
        e1.record(stream)
        barrier()
        mixed["with_buoyancy"] = {"omega_N": 1.0, "gmres_iterations": it_b, "status": st_b, "final_relres": rr_b,
                                  "solve_ms": e0.elapsed_time(e1)}
        hb.close()
        del hb
        del Fd, Xd
        if rank == 0 and not args.no_cpu_baseline:
            # the oracle beside it: one preconditioner application + mixed apply on the
            # host cores (the part of a GMRES iteration outside Gram-Schmidt), bounded sample
            import oracle
            cores = len(os.sched_getaffinity(0))
            os.environ["OMP_NUM_THREADS"] = str(cores)
            o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
            Fm = hi.uniform_vector(unknowns, 67)
            t0 = time.perf_counter()
            o.mixed_apply(o.mixed_precond(Fm))
            dt = time.perf_counter() - t0
            o.close()
            del Fm
            mixed["cpu_baseline"] = {"value": unknowns / dt, "unit": "unknowns/s per (preconditioner + apply)",
                                     "cores": cores, "kind": "oracle",
                                     "sample": f"one oracle Schur preconditioner application (incl. one V(2,2)) + "
                                               f"one mixed apply over all {unknowns} unknowns: {dt:.2f} s"}

    # ---- NEXT-3 core: the NLO column operator's banded LU solve (P:736-741,
    # m = 384, n_BW = 27) on the B200-sized NLO problem N2 ----
    nlo = nlo_section(args, stream, local) if ws == 1 else None

    # ---- end to end: host buffers through hmg_pcg_solve_host ----------------
    hb = torch.from_numpy(b).pin_memory()
    hx = torch.empty_like(hb).pin_memory()
    bnp, xnp = hb.numpy(), hx.numpy()
    h.pcg_solve_host(bnp, xnp)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        _, it_e, _, st_e = h.pcg_solve_host(bnp, xnp)
    e1.record(stream)
    barrier()
    ms_e2e_serial = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # pipelined: the K steps as one stream of right-hand sides through
    # hmg_pcg_solve_host_batch -- every step still copies its b in and its x out
    # (pinned host ring of two buffers each), overlapped with the neighbouring
    # steps' solves on separate copy streams
    hbs = [hb.numpy(), torch.from_numpy(b.copy()).pin_memory().numpy()]
    hxs = [xnp, torch.empty_like(hx).pin_memory().numpy()]
    h.pcg_solve_host_batch(hbs, hxs)
    barrier()
    e0.record(stream)
    its_b, _, st_b = h.pcg_solve_host_batch([hbs[i % 2] for i in range(args.steps)],
                                            [hxs[i % 2] for i in range(args.steps)])
    e1.record(stream)
    barrier()
    assert st_b == "HMG_OK" and all(i == iters for i in its_b), (st_b, its_b)
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    e2e_value = cfg.ndofs * nv / (ms_e2e * 1e-3)

    # ---- oracle on the host cores (rank 0, N = 1 only) -----------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(cfg, lam, b, len(os.sched_getaffinity(0)))

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: PCG + V(2,2) solve to 1e-8, ref {cfg.fine_ref}->0 x {cfg.nz} layers",
                       "dofs": cfg.ndofs, "dofs_per_gpu": cfg.ndofs // ws, "thickness": cfg.thickness, "w2": cfg.w2,
                       "pcg_iterations": iters, "vcycles_per_step": nv, "final_relres": relres,
                       "parallelism": (f"domain decomposition x{ws} (NCCL halos, all-reduce, coarse gather at ref "
                                       f"{max(2, min(args.gather_ref, cfg.fine_ref - 1))})") if ws > 1 else "single GPU",
                       "cache": f"inputs larger than L2 (fine-level operator {(3.5 if es['sweep'] else 5) * 8 * cfg.ndofs // ws / 1e6:.0f}"
                                f" MB + vectors per level)"},
            "pcg_solve_ms": ms,
            "vcycle_only": {"value": cfg.ndofs / (ms_vc * 1e-3), "unit": UNIT, "ms": ms_vc},
            "setup_s": setup_s,
            "roofline": {"kernel": "k_sweep_st (fused residual + Thomas line sweep, finest level)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic(cfg.name, es["sweep"]),
                         "store": ("edge-deduplicated couplings, D re-formed: u, b, U, 1.5 H in, u' out = 44 B/dof"
                                   if es["sweep"] else "per-cell couplings, D re-formed: u, b, U, 3 H in, u' out = 56 B/dof"),
                         # the same launch counted with the canonical per-cell store's 64 B/dof (SURVEY
                         # 8(d)), for comparison only: these bytes are not all moved
                         "per_cell_store_equivalent": {
                             "bytes_per_dof": BYTES_PER_DOF["sweep"],
                             "GB/s": BYTES_PER_DOF["sweep"] * dofs_local / (avg_sw * 1e-3) / 1e9,
                             "frac": BYTES_PER_DOF["sweep"] * dofs_local / (avg_sw * 1e-3) / 1e9 / peak},
                         "algorithmic_bytes_per_launch": bytes_sw, "avg_launch_us": avg_sw * 1e3,
                         "launches_timed": n_sw, "peak_source": peak_note,
                         "timing": ("CUDA events around each fine-level sweep launch during a second pass of the "
                                    f"{args.steps} timed steps ({ms_events:.3f} ms per step with the events; the "
                                    "pass that gives value runs without them)")},
            "fine_level_kernels": fine,
            "pcg_residual_history": hist,
            "multigrid_breakdown": levels,
            "time_share": shares,
            "cpu_baseline": cpu,
            "single_level_comparison": sl,
            "next4_mixed_outer_solve": mixed,
            "next3_banded_column_solve": nlo,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(8 * cfg.nz * n * ws),
                    "d2h_bytes_per_step": int(8 * cfg.nz * n * ws), "ms_per_step": ms_e2e,
                    "api": "hmg_pcg_solve_host_batch (copies of neighbouring steps overlap the solve)",
                    "unpipelined": {"value": cfg.ndofs * nv / (ms_e2e_serial * 1e-3), "ms_per_step": ms_e2e_serial,
                                    "api": "hmg_pcg_solve_host, one call per step"}},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(out))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def level_table(h, cfg, ws, bpd_fine, fine_ref) -> dict:
    """The paper's per-level breakdown (Tab. "MultigridBreakdown", P:1011-1038,
    and "usefulBandwidth") for this build: per level, the time of
    one operator application H^ (H^_h + H^_z fused), of one H^_z^-1 (the
    zero-guess sweep, omega T^-1 b: the Thomas solve alone), of one fused sweep
    (residual + H^_z^-1 + update), each launched alone, with useful GB/s from
    the byte model of the store the kernel reads; and the time each level takes
    inside one V(2,2) cycle (all kernels recorded with that level; the levels
    of the cooperative coarse kernel are reported together)."""
    import torch
    from paper_1605_00492_b200 import MGParams
    peak, _ = measured_peak()
    rows = []
    reps = 20
    for ref in range(fine_ref, cfg.coarsest_ref - 1, -1):
        n_r, _ = h.level_info(ref)
        dofs = n_r * cfg.nz
        x = h.empty(ref)
        x[:, :n_r] = torch.rand((cfg.nz, n_r), dtype=torch.float64, device=x.device) * 2 - 1
        y, u = h.empty(ref), h.empty(ref)
        for _ in range(2):
            h.apply_helmholtz(ref, x, y)
            h.line_smooth(ref, x, u, 1, 0.8, True)
        torch.cuda.synchronize()
        h.profile_select(None)
        h.profile_begin()
        for _ in range(reps):
            h.apply_helmholtz(ref, x, y)
        for _ in range(reps):
            h.line_smooth(ref, x, u, 1, 0.8, True)
        for _ in range(reps):
            h.line_smooth(ref, x, u, 1, 0.8, False)
        torch.cuda.synchronize()
        h.profile_end()
        row = {"ref": ref, "cells": n_r, "dofs": dofs}
        es = h.edge_store(ref)
        sb = store_bytes(es)
        for key, cls, bpd in (("H", "apply", sb["apply"]),
                              ("Hz_inv", "sweep_zero", 32.0),
                              ("sweep", "sweep", sb["sweep"])):
            nk, ms = h.profile_query(cls, ref)
            if nk:
                us = ms * 1e3 / nk
                gbs = bpd * dofs / (us * 1e-6) / 1e9
                row[key] = {"us": round(us, 2), "bytes_per_dof": bpd, "GB/s": round(gbs, 1),
                            "frac": round(gbs / peak, 3)}
        rows.append(row)
    # time per level inside one V-cycle
    bd = h.empty(fine_ref)
    bd[:, :cfg.n // ws] = torch.rand((cfg.nz, cfg.n // ws), dtype=torch.float64, device=bd.device) * 2 - 1
    z = h.empty(fine_ref)
    h.vcycle(bd, z, MGParams())
    torch.cuda.synchronize()
    h.profile_select(None)
    h.profile_begin()
    nvc = 5
    for _ in range(nvc):
        h.vcycle(bd, z, MGParams())
    torch.cuda.synchronize()
    h.profile_end()
    in_cycle = {}
    for ref in range(fine_ref, cfg.coarsest_ref - 1, -1):
        tot = 0.0
        for cls in ("sweep", "sweep_zero", "sweep_prolong", "apply", "resid_restrict", "restrict", "prolong",
                    "coarse_tail"):
            tot += h.profile_query(cls, ref)[1]
        if tot > 0:
            in_cycle[str(ref)] = round(tot * 1e3 / nvc, 2)
    return {"per_level_single_launch": rows, "vcycle_us_per_level": in_cycle,
            "note": "H = fused H^_h + H^_z apply; Hz_inv = zero-guess sweep (Thomas solve only); sweep = fused "
                    "residual + Thomas + update; vcycle_us_per_level: the cooperative coarse kernel's levels are "
                    "listed under its top level"}


def nlo_section(args, stream, local):
    """NEXT-3 core at the N2 size (81,920 columns x m = 384 rows, kl = ku = 13):
    the batched LU factorisation (setup, timed once), the dgbtrs solve and the
    paper's banded product (timed per launch with CUDA events on the launching
    stream; inputs of 10.1 / 6.8 GB, far beyond L2), the DG1 <-> DG0 transfers,
    with the paper's useful-byte models: Eq. 15, 4 m (3 n_BW + 4) B per column
    for the solve; Eq. 14, 8 m (n_BW + 2) for the product.  Matrices: seeded
    U(-1, 1) inside the band (reading R21: the BDFM1 operator is not built)."""
    import torch
    from paper_1605_00492_b200 import band_apply, band_factor, band_solve, p_prolong_add, p_restrict

    ref, nz = hi.NLO_CONFIGS["N2"]
    ncol, m, kl, ku = 20 * 4 ** ref, 6 * nz, 13, 13
    nbw = kl + ku + 1
    ld = (ncol + 31) // 32 * 32
    dev = f"cuda:{local}"
    g = torch.Generator(device=dev)
    g.manual_seed(2)
    ldab = 2 * kl + ku + 1
    ab = torch.zeros((m, ldab, ld), dtype=torch.float64, device=dev)
    ab[:, kl:, :ncol] = torch.rand((m, kl + ku + 1, ncol), generator=g, dtype=torch.float64, device=dev) * 2 - 1
    jj = torch.arange(m, device=dev)[:, None]
    rr = torch.arange(kl, ldab, device=dev)[None, :]
    ab[:, kl:, :][(jj + rr - (kl + ku) < 0) | (jj + rr - (kl + ku) >= m)] = 0.0
    ipiv = torch.zeros((m, ld), dtype=torch.int32, device=dev)
    b = torch.rand((m, ld), generator=g, dtype=torch.float64, device=dev) * 2 - 1
    x = torch.zeros_like(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    band_factor(ab, ipiv, ncol, kl, ku)
    e1.record(stream)
    torch.cuda.synchronize()
    factor_ms = e0.elapsed_time(e1)
    peak, peak_note = measured_peak()

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a0, a1 in evs:
            a0.record(stream)
            fn()
            a1.record(stream)
        torch.cuda.synchronize()
        return float(np.mean([a0.elapsed_time(a1) for a0, a1 in evs]))

    reps = max(10, min(args.steps, 30))
    solve_ms = timed(lambda: band_solve(ab, ipiv, b, x, ncol, kl, ku), reps)
    solve_bytes = ncol * 4 * m * (3 * nbw + 4)
    del ab, ipiv
    ar = torch.rand((m, nbw, ld), generator=g, dtype=torch.float64, device=dev) * 2 - 1
    y = torch.zeros_like(b)
    apply_ms = timed(lambda: band_apply(ar, b, y, ncol, kl, ku), reps)
    apply_bytes = ncol * 8 * m * (nbw + 2)
    del ar
    b0 = torch.zeros((nz, ld), dtype=torch.float64, device=dev)
    restr_ms = timed(lambda: p_restrict(b, b0, ncol), reps)
    prol_ms = timed(lambda: p_prolong_add(b0, y, ncol), reps)
    gbs = solve_bytes / (solve_ms * 1e-3) / 1e9
    out = {"workload": f"N2: {ncol} columns x m = {m} rows (ref {ref}, {nz} layers x 6 DG1 dofs), kl = ku = {kl}, "
                       f"n_BW = {nbw}; seeded U(-1, 1) band matrices",
           "factor_ms": factor_ms,
           "solve": {"us": solve_ms * 1e3, "bytes_per_column": 4 * m * (3 * nbw + 4), "GB/s": gbs,
                     "dofs_per_s": ncol * m / (solve_ms * 1e-3)},
           "apply": {"us": apply_ms * 1e3, "bytes_per_column": 8 * m * (nbw + 2),
                     "GB/s": apply_bytes / (apply_ms * 1e-3) / 1e9},
           "p_restrict_us": restr_ms * 1e3, "p_prolong_us": prol_ms * 1e3,
           "roofline": {"kernel": "k_gbtrs<13, 13> (dgbtrs per column, Eq. 15 bytes)", "bound": "hbm",
                        "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "peak_source": peak_note},
           "paper_context": "ARCHER NLO finest level: H^_z^-1 12.36 GB/s, H^_z 45.92 GB/s (P:1166)"}
    del b, x, y, b0
    torch.cuda.empty_cache()
    if not args.no_cpu_baseline:
        # the oracle beside it: dgbtrs on a bounded sample of columns, one thread
        import oracle
        rng = np.random.default_rng(0)
        nsample = 400
        t_cpu = 0.0
        for c in range(nsample):
            abc = hi.band_lu_storage(1, m, kl, ku, seed=1000 + c)[:, :, 0].T.copy()
            lu, ip, _ = oracle.gbtrf(abc, kl, ku)
            bc = rng.uniform(-1, 1, m)
            t0 = time.perf_counter()
            oracle.gbtrs(lu, kl, ku, ip, bc)
            t_cpu += time.perf_counter() - t0
        out["cpu_baseline"] = {"value": nsample * m / t_cpu, "unit": "dofs/s (solve)", "cores": 1, "kind": "oracle",
                               "sample": f"oracle dgbtrs of {nsample} columns (m = {m}, kl = ku = {kl}), one thread, "
                                         f"{t_cpu:.3f} s incl. ctypes call overhead"}
    return out


def run_c1(args):
    """BASELINE.json config C1: kernel microbench at ref 5 x 64 layers (1,310,720
    dofs): 100 launches each of the operator apply, one fused line-Jacobi sweep
    with a non-zero iterate, restriction 5 -> 4 and prolongation 4 -> 5, each
    launch preceded by a 256 MB read that evicts the 126 MB L2 (the C1 working
    set, ~84 MB, would otherwise stay resident).  Kernel durations are the
    library's CUDA events around each launch, on the launching stream."""
    import torch
    from paper_1605_00492_b200 import Hierarchy

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (no CPU fallback exists)")
    cfg = hi.CONFIGS["C1"]
    lam, b = hi.make_inputs(cfg)
    r = cfg.fine_ref
    x = hi.uniform_vector(b.shape, 101)
    u = hi.uniform_vector(b.shape, 102)
    h = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    xd, bd, ud, yd = h.to_device(r, x), h.to_device(r, b), h.to_device(r, u), h.empty(r)
    cd = h.empty(r - 1)
    # L2 eviction by READING 256 MB (a write would leave ~126 MB of dirty lines whose
    # write-back then competes with the timed kernel)
    flush_buf = torch.ones(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    flush_out = torch.empty((), dtype=torch.float32, device="cuda")

    class _Flush:
        @staticmethod
        def zero_():
            torch.sum(flush_buf, dim=0, out=flush_out)

    flush = _Flush()
    ops = {
        "apply": (lambda: h.apply_helmholtz(r, xd, yd), "apply", r, 56.0 - D_REFORMED),
        "sweep": (lambda: h.line_smooth(r, bd, ud, 1, 0.8, False), "sweep", r, 64.0 - D_REFORMED),
        "restrict": (lambda: h.restrict(r, xd, cd), "restrict", r, 10.0),
        "prolong": (lambda: h.prolong_add(r, cd, yd), "prolong", r, 18.0),
    }
    peak, peak_note = measured_peak()
    reps = max(args.steps, 100)
    # warm: 100 launches back to back (the sweep as one 100-sweep line_smooth call)
    warm_ops = {
        "apply": lambda: [h.apply_helmholtz(r, xd, yd) for _ in range(reps)],
        "sweep": lambda: h.line_smooth(r, bd, ud, reps, 0.8, False),
        "restrict": lambda: [h.restrict(r, xd, cd) for _ in range(reps)],
        "prolong": lambda: [h.prolong_add(r, cd, yd) for _ in range(reps)],
    }
    out = {}
    for name, (fn, cls, ref, bpd) in ops.items():
        for _ in range(max(args.warmup, 3)):
            fn()
        torch.cuda.synchronize()
        h.profile_begin()
        for _ in range(reps):
            flush.zero_()
            fn()
        torch.cuda.synchronize()
        h.profile_end()
        n, ms = h.profile_query(cls, ref)
        us = ms * 1e3 / max(n, 1)
        h.profile_begin()
        warm_ops[name]()
        torch.cuda.synchronize()
        h.profile_end()
        nw, msw = h.profile_query(cls, ref)
        usw = msw * 1e3 / max(nw, 1)
        gbs = bpd * cfg.ndofs / (us * 1e-6) / 1e9
        gbw = bpd * cfg.ndofs / (usw * 1e-6) / 1e9
        out[name] = {"us": round(us, 2), "launches": n, "bytes_per_dof": bpd, "GB/s": round(gbs, 1),
                     "frac": round(gbs / peak, 3),
                     "warm": {"us": round(usw, 2), "launches": nw, "GB/s": round(gbw, 1), "frac": round(gbw / peak, 3)}}
    a = out["apply"]
    print(json.dumps({
        "metric": "C1 operator apply dofs/s (kernel microbench)", "value": cfg.ndofs / (a["us"] * 1e-6),
        "unit": "dof/s", "n_gpus": 1, "steps": reps, "warmup": args.warmup, "higher_is_better": True,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C1: ref 5 x 64 layers, 1,310,720 dofs; t 0.01, w2 1e-4",
                   "cache": "L2 evicted (256 MB read) before every launch; 'warm': 100 launches back to back, "
                            "working set (84 MB) L2-resident"},
        "roofline": {"kernel": "k_apply_st (operator apply, ref 5)", "bound": "hbm", "achieved": a["GB/s"],
                     "peak": peak, "unit": "GB/s", "frac": a["frac"], "peak_source": peak_note},
        "kernels": out}))


def launch_ranks(args) -> int:
    """`bench.py --gpus N` started without torchrun: start the N ranks here
    (one process per GPU, torch.distributed.run on 127.0.0.1) and return their
    exit code.  Fails loudly when fewer than N GPUs are visible."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible", file=sys.stderr)
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and not (args.impl == "reference" or args.config == "C1"):
        sys.exit(launch_ranks(args))
    if ws > 1 and ws != args.gpus:
        raise SystemExit(f"WORLD_SIZE={ws} but --gpus {args.gpus}: launch one rank per GPU")
    if ws > 1:
        # NCCL's communicator lines (rank / nranks / device per rank) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif args.config == "C1":
        if rank == 0:
            run_c1(args)
    else:
        run_hmg(args, ws, rank, local)


if __name__ == "__main__":
    main()
