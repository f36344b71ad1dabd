"""Pins P6 (sweep, reading R7; Eq. 10/13 at P:619) and P7 (transfers,
reading R8) of the oracle."""
import numpy as np
import scipy.sparse.linalg as spla

import hmg_inputs as hi
import oracle
from dense import column_block_sparse, helmholtz_sparse, prolongation, smoother_matrices

EPS = np.finfo(np.float64).eps


def test_sweep_fixed_point(c0_oracle):
    """The exact solution u* = H^{-1} b is a fixed point of the sweep."""
    cfg, h, lam, b = c0_oracle
    L = h.level(cfg.fine_ref)
    A = helmholtz_sparse(L, cfg.nz).toarray()
    ustar = np.linalg.solve(A, b.reshape(-1)).reshape(b.shape)
    kappa = np.linalg.cond(A)
    u1 = h.sweep(cfg.fine_ref, b, ustar, 1, 0.8)
    assert np.max(np.abs(u1 - ustar)) <= kappa * EPS * np.max(np.abs(ustar))


def test_sweep_matches_matrix_form(c0_oracle):
    """Sweeps equal the affine map u <- (I - w T^-1 H^) u + w T^-1 b."""
    cfg, h, lam, b = c0_oracle
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        L = h.level(ref)
        S, W = smoother_matrices(helmholtz_sparse(L, cfg.nz), column_block_sparse(L, cfg.nz), 0.8)
        bb = hi.uniform_vector(h.shape(ref), 20 + ref)
        u0 = hi.uniform_vector(h.shape(ref), 30 + ref)
        u = u0.reshape(-1)
        for _ in range(3):
            u = S @ u + W @ bb.reshape(-1)
        got = h.sweep(ref, bb, u0, 3, 0.8)
        assert np.max(np.abs(got.reshape(-1) - u)) <= 1e-12 * np.max(np.abs(u))
        # zero-guess form == general form with u_old = 0, bitwise
        assert np.array_equal(h.sweep(ref, bb, None, 2, 0.8), h.sweep(ref, bb, np.zeros_like(bb), 2, 0.8))


def test_sweep_w2_zero_closed_form():
    """w2 = 0: H^ = T = diag(vol), so s sweeps from zero give
    u_s = (1 - (1 - w)^s) b / vol per cell."""
    cfg = hi.Config("w0", 2, 0, 8, 0.01, 0.0)
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(2, 0, 8, 0.01, 0.0, lam)
    vol = h.level(2)["area"] * (0.01 / 8)
    for s in (1, 2, 3):
        u = h.sweep(2, b, None, s, 0.8)
        assert np.allclose(u, (1 - 0.2 ** s) * b / vol[None, :], rtol=8 * EPS, atol=0)
    h.close()


def test_one_undamped_sweep_exact_without_horizontal(c0_oracle):
    """With the horizontal bands removed, H^ = T and one sweep with w = 1
    from zero is the exact solve."""
    cfg = hi.CONFIGS["C0"]
    lam, b = hi.make_inputs(cfg)
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    L = h.level(cfg.fine_ref)
    h.set_bands(cfg.fine_ref, H=np.zeros_like(L["H"]))
    L = h.level(cfg.fine_ref)
    T = column_block_sparse(L, cfg.nz).tocsc()
    exact = spla.spsolve(T, b.reshape(-1)).reshape(b.shape)
    u = h.sweep(cfg.fine_ref, b, None, 1, 1.0)
    assert np.max(np.abs(u - exact)) <= 1e-12 * np.max(np.abs(exact))
    h.close()


def test_transfer_adjoint_and_identities(c0_oracle):
    """<R r, x> = <r, P x>; R P = 4 I (to 2 ulp); P const = const exactly."""
    cfg, h, lam, b = c0_oracle
    for fr in range(cfg.coarsest_ref + 1, cfg.fine_ref + 1):
        r = hi.uniform_vector(h.shape(fr), 40 + fr)
        x = hi.uniform_vector(h.shape(fr - 1), 50 + fr)
        Rr = h.restrict(fr, r)
        Px = h.prolong_add(fr, x, np.zeros(h.shape(fr)))
        lhs, rhs = np.sum(Rr * x), np.sum(r * Px)
        assert abs(lhs - rhs) <= 1e-15 * np.sum(np.abs(r * Px)) * 4
        RP = h.restrict(fr, Px)
        assert np.all(np.abs(RP - 4 * x) <= 2 * np.spacing(4 * np.abs(x)))
        const = np.full(h.shape(fr - 1), 0.3)
        assert np.array_equal(h.prolong_add(fr, const, np.zeros(h.shape(fr))), np.full(h.shape(fr), 0.3))
        # matrix form of the transfers (DG0 children 4p..4p+3)
        P = prolongation(h.n(fr), cfg.nz)
        assert np.allclose(Rr.reshape(-1), P.T @ r.reshape(-1), rtol=0, atol=4 * EPS * 4)
        u0 = hi.uniform_vector(h.shape(fr), 60 + fr)
        assert np.array_equal(h.prolong_add(fr, x, u0), (u0.reshape(-1) + P @ x.reshape(-1)).reshape(u0.shape))
