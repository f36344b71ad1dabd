"""NEXT-4 on the GPU == oracle: the mixed velocity-pressure system (readings
R15-R20), through the C-ABI (hmg_mixed_*).

The mixed apply and the Schur-complement preconditioner reproduce the
oracle's operation order (and the preconditioner's V-cycle is the bitwise
V-cycle path), so both must be BITWISE equal to the oracle; GMRES differs
from the oracle only in the summation order of its dot products and must
take the same number of iterations to reach ||r|| <= 1e-5 ||F|| (the
paper's outer tolerance), with solutions equal to a tolerance
derived from that residual.
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

CASES = {
    "C0": hi.CONFIGS["C0"],
    "C2b_r4": hi.Config("C2b_r4", 4, 0, 64, 0.001, 1e-5),
    "C2a_r3": hi.Config("C2a_r3", 3, 0, 64, 0.01, 1e-4),
    "C4_r3": hi.Config("C4_r3", 3, 0, 128, 0.001, 1e-5),
    "nz1": hi.Config("nz1", 2, 0, 1, 0.01, 1e-4),
    "nz2_r0": hi.Config("nz2_r0", 0, 0, 2, 0.01, 1e-4),
    "nz5_r1": hi.Config("nz5_r1", 1, 0, 5, 0.01, 1e-4),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    cfg = CASES[request.param]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    yield cfg, g, o
    g.close()
    o.close()


def test_layout_and_edges(pair):
    cfg, g, o = pair
    lay = g.mixed_layout()
    ne, N = o.mixed_sizes()
    n, ld = g.level_info(cfg.fine_ref)
    assert lay["ne"] == ne and lay["ldh"] % 32 == 0 and lay["ldh"] >= ne
    assert lay["off_z"] == cfg.nz * lay["ldh"] and lay["off_p"] == lay["off_z"] + (cfg.nz - 1) * ld
    assert lay["ntot"] == lay["off_p"] + cfg.nz * ld
    ec, ce = g.mixed_edges()
    eco, _, ceo = o.mixed_edges()
    assert np.array_equal(ec, eco) and np.array_equal(ce, ceo)


def test_apply_bitwise(pair):
    cfg, g, o = pair
    _, N = o.mixed_sizes()
    for seed in (61, 62):
        x = hi.uniform_vector(N, seed)
        y = g.mixed_to_host(g.mixed_apply(g.mixed_to_device(x)))
        yo = o.mixed_apply(x)
        assert np.array_equal(y, yo)


def test_padding_stays_zero(pair):
    cfg, g, o = pair
    _, N = o.mixed_sizes()
    x = g.mixed_to_device(hi.uniform_vector(N, 63))
    y = g.mixed_apply(x)
    z = g.mixed_precond(x)
    mask = g.mixed_to_device(np.ones(N)) == 0
    assert torch.all(y[mask] == 0) and torch.all(z[mask] == 0)


@pytest.mark.parametrize("params", [MGParams(), MGParams(1, 1, 2, 0.8)], ids=["V22", "V11"])
def test_precond_bitwise(pair, params):
    cfg, g, o = pair
    _, N = o.mixed_sizes()
    f = hi.uniform_vector(N, 64)
    x = g.mixed_to_host(g.mixed_precond(g.mixed_to_device(f), params=params))
    xo = o.mixed_precond(f, nu_pre=params.nu_pre, nu_post=params.nu_post, n_coarse=params.n_coarse,
                         omega=params.omega)
    assert np.array_equal(x, xo)
    assert np.array_equal(g.mixed_to_host(g.mixed_precond(g.mixed_to_device(f), params=None)), f)


@pytest.mark.parametrize("gs_passes", [2, 1], ids=["CGS2", "CGS"])
def test_gmres_iterations_match_oracle(pair, gs_passes):
    """Both Gram-Schmidt variants (R20: CGS2 the default, CGS = PETSc's default
    and most likely the paper's) take the oracle's iteration count."""
    cfg, g, o = pair
    _, N = o.mixed_sizes()
    F = hi.uniform_vector(N, 65)
    X, it, rr, st = g.mixed_gmres(g.mixed_to_device(F), rtol=1e-5, gs_passes=gs_passes)
    Xo, it_o, rr_o, _, st_o = o.mixed_gmres(F, rtol=1e-5, gs_passes=gs_passes)
    assert st == "HMG_OK" and st_o == 0
    assert it == it_o, (it, it_o, rr, rr_o)
    assert rr <= 1e-5 and rr == pytest.approx(rr_o, rel=1e-2)
    # both solutions meet the 1e-5 tolerance, so they differ by at most 2e-5 in
    # the residual norm; in practice by dot-product rounding only
    x = g.mixed_to_host(X)
    assert np.linalg.norm(o.mixed_apply(x - Xo)) <= 2e-5 * np.linalg.norm(F)
    assert np.max(np.abs(x - Xo)) <= 1e-6 * np.max(np.abs(Xo))
    # the reported residual is the true one
    r = g.mixed_to_device(F) - g.mixed_apply(X)
    assert float(torch.linalg.norm(r) / np.linalg.norm(F)) == pytest.approx(rr, rel=1e-9)


def test_gmres_restart_and_unpreconditioned():
    """Short restarts and no preconditioner against the oracle (same count)."""
    cfg = hi.Config("r2", 2, 0, 8, 0.01, 1e-4)
    lam, _ = hi.make_inputs(cfg)
    g = Hierarchy(2, 0, 8, 0.01, 1e-4, lam)
    o = oracle.Hierarchy(2, 0, 8, 0.01, 1e-4, lam)
    _, N = o.mixed_sizes()
    F = hi.uniform_vector(N, 66)
    _, it, rr, st = g.mixed_gmres(g.mixed_to_device(F), rtol=1e-5, restart=4)
    _, it_o, rr_o, _, st_o = o.mixed_gmres(F, rtol=1e-5, restart=4)
    assert st == "HMG_OK" and st_o == 0 and it == it_o
    _, it, rr, st = g.mixed_gmres(g.mixed_to_device(F), rtol=1e-5, maxit=40, params=None)
    _, it_o, rr_o, _, st_o = o.mixed_gmres(F, rtol=1e-5, maxit=40, precond="none")
    assert st == "HMG_ERR_NOT_CONVERGED" and st_o == oracle.NOT_CONVERGED and it == it_o == 40
    assert rr == pytest.approx(rr_o, rel=1e-2)
    g.close()
    o.close()


@pytest.mark.parametrize("name", ["C0", "C2b_r4"])
def test_gmres_paper_cycle(name):
    """The paper's own cycle, V(1,1) with 2 coarse sweeps, as the
    Schur complement's pressure solve: same GMRES iteration count as the oracle."""
    cfg = CASES[name]
    lam, _ = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    _, N = o.mixed_sizes()
    F = hi.uniform_vector(N, 68)
    _, it, rr, st = g.mixed_gmres(g.mixed_to_device(F), rtol=1e-5, params=MGParams(1, 1, 2, 0.8))
    _, it_o, rr_o, _, st_o = o.mixed_gmres(F, rtol=1e-5, nu_pre=1, nu_post=1, n_coarse=2, omega=0.8)
    assert st == "HMG_OK" and st_o == 0 and it == it_o, (it, it_o)
    g.close()
    o.close()


def test_mixed_errors():
    cfg = hi.CONFIGS["C0"]
    lam, _ = hi.make_inputs(cfg)
    g = Hierarchy(2, 0, 8, 0.01, 1e-4, lam)
    x = g.mixed_empty()
    with pytest.raises(HmgError, match="y: must not alias x"):
        g.mixed_apply(x, x)
    with pytest.raises(HmgError, match="restart"):
        g.mixed_gmres(x, restart=0)
    with pytest.raises(HmgError, match="gs_passes"):
        g.mixed_gmres(x, gs_passes=3)
    X, it, rr, st = g.mixed_gmres(x)          # zero right-hand side: zero iterations, X = 0
    assert it == 0 and st == "HMG_OK" and torch.all(X == 0)
    g.close()


@pytest.mark.slow
def test_full_size_c2b_mixed():
    """C2b at full size (ref 7 x 64: 73.4M mixed unknowns), the launch
    configuration bench.py times: apply and preconditioner bitwise equal to the
    oracle, and GMRES to 1e-5 in the oracle's iteration count."""
    cfg = hi.CONFIGS["C2b"]
    lam, _ = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    _, N = o.mixed_sizes()
    F = hi.uniform_vector(N, 67)
    Fd = g.mixed_to_device(F)
    assert np.array_equal(g.mixed_to_host(g.mixed_apply(Fd)), o.mixed_apply(F))
    assert np.array_equal(g.mixed_to_host(g.mixed_precond(Fd)), o.mixed_precond(F))
    _, it, rr, st = g.mixed_gmres(Fd, rtol=1e-5)
    _, it_o, rr_o, _, st_o = o.mixed_gmres(F, rtol=1e-5)
    assert st == "HMG_OK" and st_o == 0 and it == it_o, (it, it_o, rr, rr_o)
    g.close()
    o.close()


@pytest.mark.parametrize("name", ["C0", "C2b_r4", "C4_r3"])
@pytest.mark.parametrize("omega_n", [0.5, 2.0])
def test_buoyancy_bitwise(name, omega_n):
    """Buoyancy (reading R24; hmg_build_hierarchy_ex): the hierarchy's bands on
    every level, the V-cycle, the mixed apply and the Schur preconditioner are
    bitwise the oracle's; PCG and GMRES (both Gram-Schmidt variants) take the
    oracle's iteration counts."""
    cfg = CASES[name]
    lam, b = hi.make_inputs(cfg)
    g = Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, omega_n=omega_n)
    o = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, omega_n=omega_n)
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        G, O = g.export_level(ref), o.level(ref)
        assert np.array_equal(G["D"], O["D"]) and np.array_equal(G["U"], O["U"]) and np.array_equal(G["H"], O["H"])
    r = cfg.fine_ref
    bd = g.to_device(r, b)
    assert np.array_equal(g.to_host(r, g.vcycle(bd)), o.vcycle(b))
    _, it, _, st = g.pcg_solve(bd)
    assert st == "HMG_OK" and it == o.pcg(b)[1]
    _, N = o.mixed_sizes()
    F = hi.uniform_vector(N, 69)
    Fd = g.mixed_to_device(F)
    assert np.array_equal(g.mixed_to_host(g.mixed_apply(Fd)), o.mixed_apply(F))
    assert np.array_equal(g.mixed_to_host(g.mixed_precond(Fd)), o.mixed_precond(F))
    for gs in (2, 1):
        _, itm, rrm, stm = g.mixed_gmres(Fd, rtol=1e-5, gs_passes=gs)
        _, itm_o, _, _, stm_o = o.mixed_gmres(F, rtol=1e-5, gs_passes=gs)
        assert stm == "HMG_OK" and stm_o == 0 and itm == itm_o, (gs, itm, itm_o)
    g.close()
    o.close()


def test_buoyancy_argument_errors(monkeypatch):
    lam, _ = hi.make_inputs(CASES["C0"])
    with pytest.raises(HmgError, match="omega_n"):
        Hierarchy(2, 0, 8, 0.01, 1e-4, lam, omega_n=-1.0)
    monkeypatch.setenv("HMG_OPERATOR", "free")
    with pytest.raises(HmgError, match="omega_n"):
        Hierarchy(2, 0, 8, 0.01, 1e-4, lam, omega_n=1.0)
