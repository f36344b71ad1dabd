"""GPU path == oracle, through the C-ABI (libhmg.so), on seeded inputs.

Parity contract: the V-cycle path (assembly, apply,
sweeps, transfers, V-cycle) reproduces the oracle's operation order with no
FMA contraction, so it must be BITWISE equal; the tests assert the
BASELINE.json tolerances (relative 1e-12 on applies/sweeps/transfers, 1e-10
on the V-cycle, max-norm relative) and additionally bitwise equality.  PCG
differs only in the order of its dot-product sums and must reach the same
iteration count for relative residual 1e-8.
"""
import numpy as np
import pytest

import hmg_inputs as hi
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1605_00492_b200 import Hierarchy, HmgError, MGParams  # noqa: E402


def rel(a, b):
    d = np.max(np.abs(a - b))
    s = np.max(np.abs(b))
    return d / s if s > 0 else d


CASES = {
    "C0": hi.CONFIGS["C0"],
    "C1": hi.CONFIGS["C1"],
    "C2a_r4": hi.Config("C2a_r4", 4, 0, 64, 0.01, 1e-4),
    "C2b_r4": hi.Config("C2b_r4", 4, 0, 64, 0.001, 1e-5),
    "C2c_r4": hi.Config("C2c_r4", 4, 0, 64, 1e-4, 1e-6),
    "C4_r3": hi.Config("C4_r3", 3, 0, 128, 0.001, 1e-5),
    "nz1": hi.Config("nz1", 3, 0, 1, 0.01, 1e-4),
    "nz3_r1": hi.Config("nz3_r1", 1, 0, 3, 0.01, 1e-4),
    "w2zero": hi.Config("w2zero", 2, 0, 8, 0.01, 0.0),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    cfg = CASES[request.param]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    yield cfg, g, o, lam, b
    g.close()
    o.close()


def levels(cfg):
    return range(cfg.coarsest_ref, cfg.fine_ref + 1)


def test_hierarchy_bitwise(pair):
    """P7: the two independent builders produce identical neighbour tables and
    bitwise-identical geometry, coefficients and bands on every level."""
    cfg, g, o, lam, b = pair
    for r in levels(cfg):
        G, O = g.export_level(r), o.level(r)
        assert np.array_equal(G["nbr"], O["nbr"]), f"ref {r} neighbours"
        for k in ("area", "len", "cd", "lam", "D", "U", "H"):
            assert np.array_equal(G[k], O[k]), f"ref {r} {k}"


def test_apply(pair):
    cfg, g, o, lam, b = pair
    for r in levels(cfg):
        x = hi.uniform_vector(o.shape(r), 100 + r)
        y = g.to_host(r, g.apply_helmholtz(r, g.to_device(r, x)))
        ref = o.apply(r, x)
        assert rel(y, ref) <= 1e-12
        assert np.array_equal(y, ref), f"ref {r}: not bitwise ({rel(y, ref):.2e})"


def test_sweeps(pair):
    cfg, g, o, lam, b = pair
    for r in levels(cfg):
        bb = hi.uniform_vector(o.shape(r), 200 + r)
        u0 = hi.uniform_vector(o.shape(r), 300 + r)
        for ns, zero in ((1, True), (1, False), (3, False), (2, True)):
            u = g.to_device(r, u0)
            g.line_smooth(r, g.to_device(r, bb), u, ns, 0.8, zero)
            got = g.to_host(r, u)
            ref = o.sweep(r, bb, None if zero else u0, ns, 0.8)
            assert rel(got, ref) <= 1e-12
            assert np.array_equal(got, ref), f"ref {r} ns {ns} zero {zero}"


def test_transfers(pair):
    cfg, g, o, lam, b = pair
    for r in levels(cfg):
        if r == cfg.coarsest_ref:
            continue
        rf = hi.uniform_vector(o.shape(r), 400 + r)
        uc = hi.uniform_vector(o.shape(r - 1), 500 + r)
        uf = hi.uniform_vector(o.shape(r), 600 + r)
        got = g.to_host(r - 1, g.restrict(r, g.to_device(r, rf)))
        assert np.array_equal(got, o.restrict(r, rf))
        ud = g.to_device(r, uf)
        g.prolong_add(r, g.to_device(r - 1, uc), ud)
        assert np.array_equal(g.to_host(r, ud), o.prolong_add(r, uc, uf))
        # fused residual + restriction
        got = g.to_host(r - 1, g.residual_restrict(r, g.to_device(r, rf), g.to_device(r, uf)))
        ref = o.restrict(r, o.residual(r, rf, uf))
        assert rel(got, ref) <= 1e-12
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("params", [MGParams(), MGParams(1, 1, 2, 0.8), MGParams(0, 2, 5, 0.8),
                                    MGParams(2, 0, 3, 0.8), MGParams(3, 1, 20, 1.0)])
def test_vcycle(pair, params):
    cfg, g, o, lam, b = pair
    z = g.to_host(cfg.fine_ref, g.vcycle(g.to_device(cfg.fine_ref, b), params=params))
    ref = o.vcycle(b, params.nu_pre, params.nu_post, params.n_coarse, params.omega)
    assert rel(z, ref) <= 1e-10
    assert np.array_equal(z, ref), f"V-cycle not bitwise ({rel(z, ref):.2e})"


def test_pcg_iterations(pair):
    cfg, g, o, lam, b = pair
    x, it, rr, st = g.pcg_solve(g.to_device(cfg.fine_ref, b), rtol=1e-8, maxit=200)
    xo, it_o, rr_o, hist, st_o = o.pcg(b, rtol=1e-8, maxit=200)
    assert st == "HMG_OK" and st_o == 0
    assert it == it_o, f"iterations {it} vs oracle {it_o} (oracle history tail {hist[-3:]})"
    assert rr <= 1e-8
    assert rel(g.to_host(cfg.fine_ref, x), xo) <= 1e-6
    # residual history (P:913-919 reports convergence histories): the same
    # recursively updated ||r_k|| / ||b|| up to the dots' summation order
    h = g.pcg_history()
    assert len(h) == it + 1 and h[0] == 1.0 and h[-1] == rr
    assert np.allclose(h, hist, rtol=1e-5, atol=1e-14)


def test_single_level_pcg(pair):
    """NEXT-1: the paper's single-level preconditioner (2 line sweeps) in the same PCG."""
    cfg, g, o, lam, b = pair
    x, it, rr, st = g.pcg_solve_single_level(g.to_device(cfg.fine_ref, b), nsweeps=2, rtol=1e-8, maxit=500)
    _, it_o, _, _, st_o = o.pcg(b, precond="single", nu_pre=2, rtol=1e-8, maxit=500)
    assert st == "HMG_OK" and st_o == 0 and it == it_o


def test_pcg_maxit_zero_and_zero_rhs(pair):
    """maxit = 0: x = x0 = 0, relres 1, 0 iterations, HMG_ERR_NOT_CONVERGED
    (outputs filled, include/hmg.h); b = 0: x = 0 in 0 iterations, HMG_OK; the
    residual history reports only the start."""
    cfg, g, o, lam, b = pair
    r = cfg.fine_ref
    x = g.to_device(r, np.full(o.shape(r), 7.0))
    _, it, rr, st = g.pcg_solve(g.to_device(r, b), x, maxit=0)
    assert st == "HMG_ERR_NOT_CONVERGED" and it == 0 and rr == 1.0
    assert np.all(g.to_host(r, x) == 0.0)
    assert list(g.pcg_history()) == [1.0]
    x = g.to_device(r, np.full(o.shape(r), 7.0))
    _, it, rr, st = g.pcg_solve(g.empty(r), x)
    assert st == "HMG_OK" and it == 0 and rr == 0.0 and np.all(g.to_host(r, x) == 0.0)
    assert list(g.pcg_history()) == [0.0]


def test_host_entry_point(pair):
    cfg, g, o, lam, b = pair
    x, it, rr, st = g.pcg_solve_host(b)
    xd, itd, rrd, std = g.pcg_solve(g.to_device(cfg.fine_ref, b))
    assert st == std == "HMG_OK" and it == itd
    assert np.array_equal(x, g.to_host(cfg.fine_ref, xd))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_batch_entry_point(pair, pinned):
    """Pipelined batch (copies on their own streams, two staging pairs): every
    solve bitwise equal to the one-at-a-time solve, for 5 different right-hand
    sides (odd count: both staging buffers reused), pinned and pageable."""
    cfg, g, o, lam, b = pair
    bs = [np.ascontiguousarray(b * (1.0 + 0.25 * i) + hi.uniform_vector(b.shape, 100 + i) * (i % 2))
          for i in range(5)]
    if pinned:
        bs = [torch.from_numpy(v).pin_memory().numpy() for v in bs]
        xs = [torch.empty(b.shape, dtype=torch.float64).pin_memory().numpy() for _ in bs]
    else:
        xs = [np.empty_like(v) for v in bs]
    its, rrs, st = g.pcg_solve_host_batch(bs, xs)
    assert st == "HMG_OK"
    for v, x, it, rr in zip(bs, xs, its, rrs):
        x1, it1, rr1, st1 = g.pcg_solve_host(v)
        assert st1 == "HMG_OK" and it == it1 and rr == rr1
        assert np.array_equal(x, x1)
    assert g.pcg_solve_host_batch([], []) == ([], [], "HMG_OK")


def test_padding_untouched_and_ignored():
    """ref 0 (20 cells, ld 32) and ref 1 (80 cells, ld 96): padding entries are
    never read (NaN there changes nothing) and never written."""
    cfg = hi.Config("pad", 1, 0, 4, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(1, 0, 4, 0.01, 1e-3, lam)
    o = oracle.Hierarchy(1, 0, 4, 0.01, 1e-3, lam)
    for r in (0, 1):
        n, ld = g.level_info(r)
        assert ld % 32 == 0 and ld >= n
        x = g.to_device(r, hi.uniform_vector((4, n), 7))
        x[:, n:] = float("nan")
        y = g.empty(r)
        y[:, n:] = 12345.0
        g.apply_helmholtz(r, x, y)
        assert np.array_equal(g.to_host(r, y), o.apply(r, x[:, :n].cpu().numpy()))
        assert torch.all(y[:, n:] == 12345.0)
    bd = g.to_device(1, b)
    bd[:, 80:] = float("nan")
    z = g.empty(1)
    z[:, 80:] = 7.0
    g.vcycle(bd, z)
    assert np.array_equal(g.to_host(1, z), o.vcycle(b))
    assert torch.all(z[:, 80:] == 7.0)
    x, it, rr, st = g.pcg_solve(bd)
    assert st == "HMG_OK" and it == o.pcg(b)[1]


def test_errors_name_arguments():
    cfg = hi.CONFIGS["C0"]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(2, 0, 8, 0.01, 1e-4, lam)
    x = g.empty(2)
    with pytest.raises(HmgError, match="ref"):
        g.apply_helmholtz(3, x, g.empty(2))
    with pytest.raises(HmgError, match="alias"):
        g.apply_helmholtz(2, x, x)
    with pytest.raises(HmgError, match="n_coarse"):
        g.vcycle(x, params=MGParams(2, 2, 0, 0.8))
    with pytest.raises(HmgError, match="coarser"):
        g.restrict(0, g.empty(0), g.empty(0))
    x, it, rr, st = g.pcg_solve(g.to_device(2, b), rtol=1e-30, maxit=2)
    assert st == "HMG_ERR_NOT_CONVERGED" and it == 2
    x, it, rr, st = g.pcg_solve(g.empty(2))
    assert st == "HMG_OK" and it == 0 and float(x.abs().max()) == 0.0


def test_singular_column_reported_at_build():
    """An overflowing vertical coupling (two adjacent coefficients of 1.7e308)
    makes column 5's Thomas pivot non-finite: hmg_build_hierarchy fails with
    HMG_ERR_SINGULAR_COLUMN naming the level and the column."""
    lam, _ = hi.make_inputs(hi.CONFIGS["C0"])
    lam = lam.copy()
    lam[3, 5] = lam[4, 5] = 1.7e308
    with pytest.raises(HmgError, match="singular column: ref 2 column 5"):
        Hierarchy(2, 0, 8, 0.01, 1e-4, lam)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2a", "C2b", "C2c"])
def test_full_size_c2(name):
    """BASELINE.json config C2 at full size (ref 7 x 64 = 20.97M dofs), in the
    launch configuration bench.py times: V-cycle bitwise equal to the oracle,
    apply bitwise, and the same PCG iteration count."""
    cfg = hi.CONFIGS[name]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    r = cfg.fine_ref
    bd = g.to_device(r, b)
    assert np.array_equal(g.to_host(r, g.apply_helmholtz(r, bd)), o.apply(r, b))
    z = g.to_host(r, g.vcycle(bd))
    zo = o.vcycle(b)
    assert rel(z, zo) <= 1e-10 and np.array_equal(z, zo)
    _, it, rr, st = g.pcg_solve(bd)
    _, it_o, _, _, st_o = o.pcg(b)
    assert st == "HMG_OK" and st_o == 0 and it == it_o
    g.close()
    o.close()


@pytest.mark.slow
def test_full_size_c4():
    """BASELINE.json config C4 whole on one GPU (ref 8 x 128 = 167.8M dofs, the
    8-GPU weak-scaling problem; 128 layers: one sweep CTA per SM, no cooperative
    tail): the operator apply and the V-cycle bitwise equal to the oracle, and
    the PCG solve to 1e-8 in the oracle's iteration count (north_star: "the same
    CG iteration count ... on all five configs")."""
    cfg = hi.CONFIGS["C4"]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    r = cfg.fine_ref
    bd = g.to_device(r, b)
    assert np.array_equal(g.to_host(r, g.apply_helmholtz(r, bd)), o.apply(r, b))
    z = g.to_host(r, g.vcycle(bd))
    zo = o.vcycle(b)
    assert rel(z, zo) <= 1e-10 and np.array_equal(z, zo)
    del z, zo
    x, it, rr, st = g.pcg_solve(bd)
    xo, it_o, rr_o, _, st_o = o.pcg(b)
    assert st == "HMG_OK" and st_o == 0 and it == it_o, (it, it_o, rr, rr_o)
    # the two solutions differ only through the dot products' summation order
    assert rel(g.to_host(r, x), xo) <= 1e-10
    g.close()
    o.close()


def test_shared_reciprocal_division_is_bitwise_ieee():
    """The sweep's shared-reciprocal division equals the compiler's a / b bit
    for bit: 2^24 random pairs over a wide exponent range plus special values."""
    from paper_1605_00492_b200.binding import selftest_div
    rng = np.random.default_rng(5)
    n = 1 << 24
    a = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-300, 300, n)
    b = rng.uniform(0, 1, n) * 10.0 ** rng.uniform(-300, 300, n)
    special = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, 1e-310, 3.0, 7.0])
    sa, sb = np.meshgrid(special, special)
    a = np.concatenate([a, sa.ravel(), rng.uniform(1e-8, 1e4, 1 << 20)])
    b = np.concatenate([b, sb.ravel(), rng.uniform(1e-8, 1e4, 1 << 20)])
    fast, ref = selftest_div(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    f, r = fast.cpu().numpy(), ref.cpu().numpy()
    both_nan = np.isnan(f) & np.isnan(r)
    assert np.array_equal(f.view(np.int64)[~both_nan], r.view(np.int64)[~both_nan])
    assert np.array_equal(np.isnan(f), np.isnan(r))
    ok = ~np.isnan(r) & (b != 0) & np.isfinite(a) & np.isfinite(b)
    # and the compiler's division is the IEEE quotient numpy computes
    assert np.array_equal(r[ok].view(np.int64), (a[ok] / b[ok]).view(np.int64))


@pytest.mark.parametrize("coop", ["-1", "0", "1", "3", "4"])
@pytest.mark.parametrize("params", [MGParams(), MGParams(0, 1, 3, 0.8), MGParams(1, 0, 2, 0.9)])
def test_coarse_split_pcg(monkeypatch, coop, params):
    """Levels <= HMG_COOP_REF in the cooperative launch, the rest as per-level
    kernels: V-cycle bitwise the oracle's and the same PCG behaviour for any
    split point."""
    monkeypatch.setenv("HMG_COOP_REF", coop)
    cfg = hi.Config("tail", 4, 0, 16, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(4, 0, 16, 0.01, 1e-3, lam)
    o = oracle.Hierarchy(4, 0, 16, 0.01, 1e-3, lam)
    z = g.to_host(4, g.vcycle(g.to_device(4, b), params=params))
    assert np.array_equal(z, o.vcycle(b, params.nu_pre, params.nu_post, params.n_coarse, params.omega))
    # (V(0,1) / V(1,0) are not symmetric preconditioners: CG need not converge,
    # but both sides must behave identically)
    _, it, _, st = g.pcg_solve(g.to_device(4, b), params=params, maxit=60)
    _, it_o, _, _, st_o = o.pcg(b, nu_pre=params.nu_pre, nu_post=params.nu_post, n_coarse=params.n_coarse,
                                omega=params.omega, maxit=60)
    assert it == it_o and (st == "HMG_OK") == (st_o == 0)


@pytest.mark.parametrize("coop", ["-1", "0", "1", "2", "3", "4"])
@pytest.mark.parametrize("params", [MGParams(), MGParams(0, 1, 3, 0.8), MGParams(1, 0, 2, 0.9),
                                    MGParams(3, 3, 4, 1.0)])
def test_cooperative_coarse_levels(monkeypatch, coop, params):
    """Levels <= HMG_COOP_REF in one cooperative launch (32-column tiles in
    shared memory, grid barriers between the dependent steps; ref 4 has more
    tiles than SMs, so CTAs take several): the same bits as the oracle."""
    monkeypatch.setenv("HMG_COOP_REF", coop)
    cfg = hi.Config("coop", 5, 0, 24, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 0, 24, 0.01, 1e-3, lam)
    o = oracle.Hierarchy(5, 0, 24, 0.01, 1e-3, lam)
    z = g.to_host(5, g.vcycle(g.to_device(5, b), params=params))
    assert np.array_equal(z, o.vcycle(b, params.nu_pre, params.nu_post, params.n_coarse, params.omega))
    g.close()
    o.close()


@pytest.mark.parametrize("fine,coarsest,nz", [(4, 2, 64), (5, 1, 128), (3, 0, 1), (2, 2, 13)])
def test_coarse_tail_shapes(fine, coarsest, nz):
    """Coarse tails with a coarsest level wider than one tile (grid barriers
    between its sweeps), 128 layers (16-column tiles), a one-layer mesh, and a
    layer count that is not a multiple of 8: bitwise equal to the oracle."""
    cfg = hi.Config("coop", fine, coarsest, nz, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(fine, coarsest, nz, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(fine, coarsest, nz, 0.001, 1e-5, lam)
    z = g.to_host(fine, g.vcycle(g.to_device(fine, b)))
    assert np.array_equal(z, o.vcycle(b, 2, 2, 20, 0.8))
    g.close()
    o.close()


@pytest.mark.parametrize("ref,fine", [(2, 2), (4, 4), (3, 5)])
def test_sweep_exact_division_fallback(ref, fine):
    """Zero numerators leave the shared-reciprocal division's fast range: the
    sweep must then recompute the column with '/' and still match the oracle
    bit for bit (zero right-hand-side columns and isolated zero entries)."""
    cfg = hi.Config("zeros", fine, 0, 16, 0.01, 1e-4)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(fine, 0, 16, 0.01, 1e-4, lam)
    o = oracle.Hierarchy(fine, 0, 16, 0.01, 1e-4, lam)
    bb = hi.uniform_vector(o.shape(ref), 77)
    bb[:, ::7] = 0.0
    bb[3, 1::5] = 0.0
    for zero in (True, False):
        u0 = np.zeros(o.shape(ref)) if zero else hi.uniform_vector(o.shape(ref), 78)
        u = g.to_device(ref, u0)
        g.line_smooth(ref, g.to_device(ref, bb), u, 2, 0.8, zero)
        assert np.array_equal(g.to_host(ref, u), o.sweep(ref, bb, None if zero else u0, 2, 0.8))


@pytest.mark.parametrize("fine,nz,edge", [(5, 16, False), (6, 64, False), (5, 64, True)])
def test_streamed_sweep_zero_residual_columns(monkeypatch, fine, nz, edge):
    """Streamed sweep (ref >= 5) on columns whose residual is exactly zero
    (b = H^ u0 computed by the oracle in the kernel's own operation order): the
    z recurrence meets +0 / -0 numerators, which leave the shared-reciprocal
    division's checked fast path, so the warp redoes its columns with '/' and
    must match the oracle bit for bit; also with the fused prolongation inside a
    V-cycle, the fused <r, z> of PCG and the edge-deduplicated coupling store."""
    if edge:
        monkeypatch.setenv("HMG_EDGE_MIN_DOFS", "1000000")
    cfg = hi.Config("cert", fine, 0, nz, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(fine, 0, nz, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(fine, 0, nz, 0.001, 1e-5, lam)
    u0 = hi.uniform_vector(o.shape(fine), 81)
    bb = hi.uniform_vector(o.shape(fine), 82)
    hu = o.apply(fine, u0)
    bb[:, 3::41] = hu[:, 3::41]                        # exactly zero residual in these columns
    bb[:, 200] = hu[:, 200]
    u = g.to_device(fine, u0)
    g.line_smooth(fine, g.to_device(fine, bb), u, 1, 0.8, False)
    assert np.array_equal(g.to_host(fine, u), o.sweep(fine, bb, u0, 1, 0.8))
    # inside the V-cycle (fused prolongation) and PCG (fused <r, z>)
    z = g.to_host(fine, g.vcycle(g.to_device(fine, bb)))
    assert np.array_equal(z, o.vcycle(bb))
    _, it, _, st = g.pcg_solve(g.to_device(fine, bb))
    assert st == "HMG_OK" and it == o.pcg(bb)[1]
    g.close()
    o.close()


@pytest.mark.parametrize("gather_ref", [2, 3, 5])
@pytest.mark.parametrize("force", ["0", "1"])
def test_distributed_path_one_rank(monkeypatch, gather_ref, force):
    """The multi-GPU code path with a one-rank NCCL communicator: distributed
    levels above gather_ref (unfused prolongation, halo exchange plan, coarse
    gather) give the oracle's V-cycle bit for bit and the same CG count;
    HMG_FORCE_COLLECTIVES=1 runs the NCCL all-reduce / all-gather and their
    pack kernels anyway."""
    from paper_1605_00492_b200 import nccl_unique_id
    monkeypatch.setenv("HMG_FORCE_COLLECTIVES", force)
    cfg = hi.Config("dist1", 5, 0, 16, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 0, 16, 0.01, 1e-3, lam, dist=(0, 1, nccl_unique_id(), gather_ref))
    o = oracle.Hierarchy(5, 0, 16, 0.01, 1e-3, lam)
    bd = g.to_device(5, b)
    assert np.array_equal(g.to_host(5, g.apply_helmholtz(5, bd)), o.apply(5, b))
    for params in (MGParams(), MGParams(0, 2, 5, 0.8), MGParams(2, 0, 3, 0.8)):
        z = g.to_host(5, g.vcycle(bd, params=params))
        assert np.array_equal(z, o.vcycle(b, params.nu_pre, params.nu_post, params.n_coarse, params.omega))
    _, it, rr, st = g.pcg_solve(bd)
    assert st == "HMG_OK" and it == o.pcg(b)[1]
    g.close()
    o.close()


def test_pcg_fused_finalize_deterministic_and_equal_to_unfused(monkeypatch):
    """The fused finalize (the last CTA of each partial-sum kernel applies the
    CG scalar update, DESIGN 7 k_update_xr row): two solves on one hierarchy give
    bitwise the same x and residual history (fixed reduction order, the CTA
    counter reset after every launch); a one-rank hierarchy through the
    unfused path (k_finalize + the NCCL all-reduce, HMG_FORCE_COLLECTIVES=1)
    reaches the same iterate up to the partial sums' order, with the oracle's
    iteration count on both."""
    from paper_1605_00492_b200 import nccl_unique_id
    cfg = hi.Config("fin", 5, 0, 16, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    o = oracle.Hierarchy(5, 0, 16, 0.01, 1e-3, lam)
    it_o = o.pcg(b)[1]
    g = Hierarchy(5, 0, 16, 0.01, 1e-3, lam)
    bd = g.to_device(5, b)
    runs = []
    for _ in range(2):
        x, it, rr, st = g.pcg_solve(bd)
        assert st == "HMG_OK" and it == it_o
        runs.append((g.to_host(5, x), g.pcg_history()))
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
    monkeypatch.setenv("HMG_FORCE_COLLECTIVES", "1")
    gd = Hierarchy(5, 0, 16, 0.01, 1e-3, lam, dist=(0, 1, nccl_unique_id(), 3))
    xd, itd, rrd, std = gd.pcg_solve(gd.to_device(5, b))
    assert std == "HMG_OK" and itd == it_o
    assert rel(gd.to_host(5, xd), runs[0][0]) <= 1e-12
    assert np.allclose(gd.pcg_history(), runs[0][1], rtol=1e-10, atol=0)
    g.close()
    gd.close()
    o.close()


@pytest.mark.parametrize("w2", [1e-4, 1e-290])
def test_matrix_free_operator(monkeypatch, w2):
    """NEXT-2 matrix-free store (HMG_OPERATOR=free): couplings recomputed from
    lam and the column geometry in k_assemble's order, so applies, sweeps (zero
    guess, general, with the fused prolongation) and the V-cycle are bitwise the
    oracle's.  w2 = 1e-290 makes the couplings subnormal: the build-time range
    proof fails, the checked division runs and its exact redo path is taken."""
    monkeypatch.setenv("HMG_OPERATOR", "free")
    cfg = hi.Config("mf", 5, 0, 16, 0.01, w2)       # ref 5 (20,480 cells): streamed kernels, no precomputed pivots
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 0, 16, 0.01, w2, lam)
    o = oracle.Hierarchy(5, 0, 16, 0.01, w2, lam)
    x = hi.uniform_vector(b.shape, 7)
    assert np.array_equal(g.to_host(5, g.apply_helmholtz(5, g.to_device(5, x))), o.apply(5, x))
    for zero in (True, False):
        u = g.to_device(5, np.zeros_like(x) if zero else x)
        g.line_smooth(5, g.to_device(5, b), u, 2, 0.8, zero)
        assert np.array_equal(g.to_host(5, u), o.sweep(5, b, None if zero else x, 2, 0.8))
    z = g.to_host(5, g.vcycle(g.to_device(5, b)))
    assert np.array_equal(z, o.vcycle(b, 2, 2, 20, 0.8))
    g.close()
    o.close()


@pytest.mark.parametrize("nz", [1, 2, 3, 7, 9, 65, 128, 130])
def test_streamed_kernels_layer_counts(nz):
    """The streamed persistent kernels (k_sweep_st, k_apply_st, k_sweep_tc zero
    guess) on a level without precomputed pivots (ref 5: 20,480 cells) for layer
    counts that leave partial stages and a partial top back-substitution chunk,
    the 128-layer TMEM limit and the fallback beyond it: apply, sweeps, V-cycle
    and the fused <r, z> PCG bitwise / iteration-count equal to the oracle."""
    cfg = hi.Config("nz", 5, 3, nz, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 3, nz, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(5, 3, nz, 0.001, 1e-5, lam)
    x = hi.uniform_vector(b.shape, 21)
    assert np.array_equal(g.to_host(5, g.apply_helmholtz(5, g.to_device(5, x))), o.apply(5, x))
    for zero in (True, False):
        u = g.to_device(5, np.zeros_like(x) if zero else x)
        g.line_smooth(5, g.to_device(5, b), u, 3, 0.8, zero)
        assert np.array_equal(g.to_host(5, u), o.sweep(5, b, None if zero else x, 3, 0.8))
    z = g.to_host(5, g.vcycle(g.to_device(5, b)))
    assert np.array_equal(z, o.vcycle(b, 2, 2, 20, 0.8))
    _, it, _, st = g.pcg_solve(g.to_device(5, b))
    assert st == "HMG_OK" and it == o.pcg(b)[1]
    g.close()
    o.close()


@pytest.mark.parametrize("nz", [9, 60, 65, 100])
def test_interleaved_sweep_multi_tile_layer_counts(nz):
    """The interleaved schedule of the streamed sweep (k_sweep_st):
    on ref 6 (640 tiles, three per CTA) every CTA runs forward passes with the
    mirrored TMEM slots (odd passes) and back substitutions of a previous tile
    between them; layer counts with a partial top chunk (9, 60, 65, 100), one and
    two CTAs per SM.  Sweeps, the V-cycle (fused prolongation) and PCG (fused
    <r, z>) against the oracle."""
    cfg = hi.Config("il", 6, 4, nz, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(6, 4, nz, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(6, 4, nz, 0.001, 1e-5, lam)
    x = hi.uniform_vector(b.shape, 23)
    u = g.to_device(6, x)
    g.line_smooth(6, g.to_device(6, b), u, 3, 0.8, False)
    assert np.array_equal(g.to_host(6, u), o.sweep(6, b, x, 3, 0.8))
    assert np.array_equal(g.to_host(6, g.vcycle(g.to_device(6, b))), o.vcycle(b, 2, 2, 20, 0.8))
    _, it, _, st = g.pcg_solve(g.to_device(6, b))
    assert st == "HMG_OK" and it == o.pcg(b)[1]
    g.close()
    o.close()


@pytest.mark.parametrize("nz", [64, 128])
def test_edge_store_forced_on_small_levels(monkeypatch, nz):
    """The edge-deduplicated coupling store is built only on
    levels of >= 16M dofs by default; forced onto ref 5 (HMG_EDGE_MIN_DOFS), the
    streamed apply, sweeps (with and without the fused prolongation), the
    streamed residual + restriction and the V-cycle stay bitwise equal to the
    oracle, and PCG takes its iteration count."""
    monkeypatch.setenv("HMG_EDGE_MIN_DOFS", "1000000")
    cfg = hi.Config("edge", 5, 0, nz, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 0, nz, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(5, 0, nz, 0.001, 1e-5, lam)
    es = g.edge_store(5)
    assert es["apply"] and es["sweep"] == (nz <= 64) and es["resid_restrict"] == (nz <= 64)
    x = hi.uniform_vector(b.shape, 71)
    bd, xd = g.to_device(5, b), g.to_device(5, x)
    assert np.array_equal(g.to_host(5, g.apply_helmholtz(5, xd)), o.apply(5, x))
    u = g.to_device(5, x)
    g.line_smooth(5, bd, u, 2, 0.8, False)
    assert np.array_equal(g.to_host(5, u), o.sweep(5, b, x, 2, 0.8))
    assert np.array_equal(g.to_host(4, g.residual_restrict(5, bd, xd)), o.restrict(5, o.residual(5, b, x)))
    assert np.array_equal(g.to_host(5, g.vcycle(bd)), o.vcycle(b))
    _, it, _, st = g.pcg_solve(bd)
    _, it_o, _, _, st_o = o.pcg(b)
    assert st == "HMG_OK" and st_o == 0 and it == it_o
    g.close()
    o.close()


@pytest.mark.parametrize("env", [{}, {"HMG_DEFER_X": "0"}, {"HMG_X_BLOCKS": "0"}, {"HMG_X_BLOCKS": "7"}])
def test_deferred_x_update_paths(monkeypatch, env):
    """The CG update x = x + alpha p runs deferred on a side stream (default), on
    the solve stream (HMG_DEFER_X=0), at full width (HMG_X_BLOCKS=0) or trickled
    by a few CTAs: every variant gives the same x bit for bit, also when PCG
    stops at maxit (NOT_CONVERGED, the last update still lands)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = hi.Config("defx", 5, 0, 64, 0.001, 1e-5)
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(5, 0, 64, 0.001, 1e-5, lam)
    o = oracle.Hierarchy(5, 0, 64, 0.001, 1e-5, lam)
    bd = g.to_device(5, b)
    x, it, rr, st = g.pcg_solve(bd, rtol=1e-8)
    xo, it_o, _, _, st_o = o.pcg(b, rtol=1e-8)
    assert st == "HMG_OK" and it == it_o
    x = g.to_host(5, x)
    assert rel(x, xo) <= 1e-9                      # x differs from the oracle's only by dot rounding
    x2, it2, _, st2 = g.pcg_solve(bd, rtol=1e-30, maxit=2)
    xo2, _, _, _, st_o2 = o.pcg(b, rtol=1e-30, maxit=2)
    assert st2 == "HMG_ERR_NOT_CONVERGED" and st_o2 == oracle.NOT_CONVERGED and it2 == 2
    assert rel(g.to_host(5, x2), xo2) <= 1e-9
    # reference for the bitwise comparison across variants: the solve-stream update
    monkeypatch.setenv("HMG_DEFER_X", "0")
    g0 = Hierarchy(5, 0, 64, 0.001, 1e-5, lam)
    x0, _, _, _ = g0.pcg_solve(g0.to_device(5, b), rtol=1e-8)
    assert np.array_equal(x, g0.to_host(5, x0))
    g.close()
    g0.close()
    o.close()
