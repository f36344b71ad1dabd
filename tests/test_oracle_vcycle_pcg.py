"""Pins P8 (V-cycle, reading R9; Alg. 1 at P:201-219) and P9/P10 (PCG,
readings R10/R12) of the oracle."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import hmg_inputs as hi
import oracle
from dense import helmholtz_sparse, vcycle_matrix

EPS = np.finfo(np.float64).eps


def _levels(h, cfg):
    return [h.level(r) for r in range(cfg.coarsest_ref, cfg.fine_ref + 1)]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_vcycle_matches_matrix_form(seed):
    """The oracle's recursive V(2,2) equals Alg. 1 written as a matrix product
    (tests/dense.py), 3 levels (C0), seeds 0-2."""
    cfg = hi.CONFIGS["C0"]
    lam, b = hi.make_inputs(cfg, seed=seed)
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    B = vcycle_matrix(_levels(h, cfg), cfg.nz, 2, 2, 20, 0.8)
    z = h.vcycle(b)
    ref = (B @ b.reshape(-1)).reshape(b.shape)
    assert np.max(np.abs(z - ref)) <= 1e-12 * np.max(np.abs(ref))
    # V(1,1) with 2 coarse sweeps: the paper's own setting
    B11 = vcycle_matrix(_levels(h, cfg), cfg.nz, 1, 1, 2, 0.8)
    assert np.allclose(h.vcycle(b, 1, 1, 2), (B11 @ b.reshape(-1)).reshape(b.shape), rtol=0,
                       atol=1e-12 * np.max(np.abs(ref)))
    h.close()


def test_two_grid_with_exact_coarse_solve():
    """2-level cycle with many coarse sweeps approaches the two-grid cycle
    with the exact coarse inverse (M3 of Alg. 1)."""
    cfg = hi.Config("tg", 1, 0, 8, 0.01, 1e-4)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(1, 0, 8, 0.01, 1e-4, lam)
    B = vcycle_matrix(_levels(h, cfg), 8, 2, 2, 0, 0.8, exact_coarse=True)
    z = h.vcycle(b, 2, 2, 400)
    ref = (B @ b.reshape(-1)).reshape(b.shape)
    assert np.max(np.abs(z - ref)) <= 1e-10 * np.max(np.abs(ref))
    h.close()


def test_single_level_is_coarse_sweeps():
    """A 1-level hierarchy's V-cycle is n_coarse sweeps from zero."""
    cfg = hi.Config("one", 2, 2, 8, 0.01, 1e-4)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(2, 2, 8, 0.01, 1e-4, lam)
    assert np.array_equal(h.vcycle(b, 2, 2, 20), h.sweep(2, b, None, 20, 0.8))
    h.close()


def test_vcycle_linear_symmetric_positive(c0_oracle):
    """V is linear, symmetric and positive definite (nu_pre = nu_post,
    R = P^T, symmetric T, convergent smoother): <Vx,y> = <x,Vy>, <Vx,x> > 0."""
    cfg, h, lam, b = c0_oracle
    x = hi.uniform_vector(h.shape(cfg.fine_ref), 71)
    y = hi.uniform_vector(h.shape(cfg.fine_ref), 72)
    Vx, Vy = h.vcycle(x), h.vcycle(y)
    assert abs(np.sum(Vx * y) - np.sum(x * Vy)) <= 1e-12 * np.sum(np.abs(Vx * y))
    assert np.sum(Vx * x) > 0 and np.sum(Vy * y) > 0
    Vxy = h.vcycle(2.5 * x + y)
    assert np.max(np.abs(Vxy - (2.5 * Vx + Vy))) <= 1e-12 * np.max(np.abs(Vxy))
    assert np.array_equal(h.vcycle(np.zeros_like(x)), np.zeros_like(x))
    assert np.array_equal(h.vcycle(x), Vx)          # stationary, deterministic


def test_w2_zero_vcycle_closed_form():
    """w2 = 0: every level is diag(vol) and the V-cycle is a per-cell scalar
    recursion, computed here in closed form from the level volumes."""
    nz = 4
    cfg = hi.Config("w0", 2, 0, nz, 0.01, 0.0)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(2, 0, nz, 0.01, 0.0, lam)
    w = 0.8
    vols = {r: h.level(r)["area"] * (0.01 / nz) for r in range(3)}

    def V(r, bb):
        if r == 0:
            return (1 - (1 - w) ** 20) * bb / vols[0][None, :]
        u = (1 - (1 - w) ** 2) * bb / vols[r][None, :]
        res = bb - vols[r][None, :] * u
        bc = res.reshape(nz, -1, 4).sum(axis=2)
        u = u + np.repeat(V(r - 1, bc), 4, axis=1)
        for _ in range(2):
            u = u + w * (bb - vols[r][None, :] * u) / vols[r][None, :]
        return u

    assert np.allclose(h.vcycle(b), V(2, b), rtol=1e-13, atol=0)
    h.close()


def _scipy_cg_iters(A, b, M=None):
    count = [0]

    def cb(xk):
        count[0] += 1

    x, info = spla.cg(A, b, rtol=1e-8, atol=0.0, M=M, maxiter=500, callback=cb)
    return x, info, count[0]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pcg_iterations_match_scipy(seed):
    """P9: scipy.sparse.linalg.cg with M = the oracle V-cycle takes the same
    number of iterations; V = I matches plain CG; x close to the dense solve."""
    cfg = hi.CONFIGS["C0"]
    lam, b = hi.make_inputs(cfg, seed=seed)
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    A = helmholtz_sparse(h.level(cfg.fine_ref), cfg.nz)
    shp = b.shape
    M = spla.LinearOperator(A.shape, matvec=lambda v: h.vcycle(v.reshape(shp)).reshape(-1))
    _, info, it_ref = _scipy_cg_iters(A, b.reshape(-1), M)
    x, it, rel, hist, st = h.pcg(b)
    assert st == 0 and info == 0 and it == it_ref
    assert rel <= 1e-8 and np.all(np.diff(hist) < 0)
    xs = np.linalg.solve(A.toarray(), b.reshape(-1))
    kappa = np.linalg.cond(A.toarray())
    assert np.max(np.abs(x.reshape(-1) - xs)) <= kappa * 1e-8 * np.max(np.abs(xs)) * 10
    _, info0, it0 = _scipy_cg_iters(A, b.reshape(-1))
    _, itp, _, _, st0 = h.pcg(b, precond="none", maxit=500)
    assert st0 == 0 and itp == it0
    h.close()


def test_pcg_aniso_iterations_match_scipy():
    """Same check on a strongly anisotropic small problem (C2c-like ratios)."""
    cfg = hi.Config("an", 2, 0, 16, 1e-4, 1e-6)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(2, 0, 16, 1e-4, 1e-6, lam)
    A = helmholtz_sparse(h.level(2), 16)
    shp = b.shape
    M = spla.LinearOperator(A.shape, matvec=lambda v: h.vcycle(v.reshape(shp)).reshape(-1))
    _, info, it_ref = _scipy_cg_iters(A, b.reshape(-1), M)
    _, it, rel, _, st = h.pcg(b)
    assert st == 0 and it == it_ref
    h.close()


def test_single_level_preconditioner():
    """Single-level preconditioner (two block-Jacobi line sweeps from zero,
    P:815-817) in the same PCG: scipy agrees on the count, and with strong
    horizontal coupling the multigrid V-cycle needs fewer iterations
    (the paper's MG vs single-level comparison)."""
    cfg = hi.Config("sl", 3, 0, 16, 0.01, 1e-2)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(3, 0, 16, 0.01, 1e-2, lam)
    A = helmholtz_sparse(h.level(3), 16)
    shp = b.shape
    Ms = spla.LinearOperator(A.shape, matvec=lambda v: h.sweep(3, v.reshape(shp), None, 2, 0.8).reshape(-1))
    _, info_s, it_s_ref = _scipy_cg_iters(A, b.reshape(-1), Ms)
    _, it_s, _, _, st_s = h.pcg(b, precond="single", nu_pre=2)
    _, it_mg, _, _, st = h.pcg(b)
    assert st_s == 0 and st == 0 and it_s == it_s_ref and it_s > 2 * it_mg
    h.close()


def test_pcg_zero_rhs_and_not_converged(c0_oracle):
    cfg, h, lam, b = c0_oracle
    x, it, rel, hist, st = h.pcg(np.zeros_like(b))
    assert it == 0 and st == 0 and np.all(x == 0)
    x, it, rel, hist, st = h.pcg(b, maxit=1, rtol=1e-30)
    assert st == oracle.NOT_CONVERGED and it == 1


def _factor(h, b, k=6):
    _, it, rel, hist, st = h.pcg(b, rtol=1e-10)
    return hist[min(k, len(hist) - 1)] ** (1.0 / min(k, len(hist) - 1))


@pytest.mark.slow
def test_convergence_factor_mesh_and_anisotropy_independent():
    """P10 (parity unpinned in absolute value: the paper prints no factor for
    PCG on H^): at fixed horizontal Courant-like ratio (w2 ~ h^2) the PCG
    contraction factor is independent of the mesh size, and across the
    three C2 anisotropies at ref 4 the spread is <= 0.1 (BASELINE.json)."""
    nz = 32
    facs = []
    for ref in (2, 3, 4):
        w2 = 1e-4 * 4.0 ** (3 - ref)
        cfg = hi.Config("m", ref, 0, nz, 0.01, w2)
        lam, b = hi.make_inputs(cfg)
        h = oracle.Hierarchy(ref, 0, nz, 0.01, w2, lam)
        facs.append(_factor(h, b))
        h.close()
    assert max(facs) - min(facs) <= 0.1 and max(facs) < 0.5
    facs = []
    for t, w2 in ((0.01, 1e-4), (0.001, 1e-5), (1e-4, 1e-6)):
        cfg = hi.Config("a", 4, 0, nz, t, w2)
        lam, b = hi.make_inputs(cfg)
        h = oracle.Hierarchy(4, 0, nz, t, w2, lam)
        facs.append(_factor(h, b))
        h.close()
    assert max(facs) - min(facs) <= 0.1 and max(facs) < 0.5
