"""Pin P5 of the oracle's Thomas solve (reading R6, the textbook
tridiagonal algorithm of the cited Press et al. section 2.4)."""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle

EPS = np.finfo(np.float64).eps


def _dense(D, U):
    return np.diag(D) + np.diag(U[:-1], 1) + np.diag(U[:-1], -1)


def test_spec_examples():
    """tridiag(-1,2,-1) (1,1,1) = (1,0,1), so its solve maps (1,0,1) -> (1,1,1)."""
    x = oracle.thomas([2, 2, 2], [-1, -1, 0], [1, 0, 1])
    assert np.allclose(x, [1, 1, 1], rtol=0, atol=4 * EPS)
    assert np.array_equal(oracle.thomas([1.0] * 5, [0.0] * 5, [1, 2, 3, 4, 5]), [1, 2, 3, 4, 5])
    assert np.array_equal(oracle.thomas([4.0], [0.0], [2.0]), [0.5])


def test_matches_dense_on_every_c0_column(c0_oracle):
    cfg, h, lam, b = c0_oracle
    L = h.level(cfg.fine_ref)
    D, U = L["D"], L["U"]
    for c in range(D.shape[1]):
        T = _dense(D[:, c], U[:, c])
        x = oracle.thomas(D[:, c], U[:, c], b[:, c])
        ref = np.linalg.solve(T, b[:, c])
        kappa = np.linalg.cond(T)
        assert np.max(np.abs(x - ref)) <= 10 * kappa * EPS * np.max(np.abs(ref))


@pytest.mark.parametrize("aniso", [64.0, 4096.0, 409600.0])
def test_random_columns_vs_solve_banded(aniso):
    """Random thin-shell-like columns (V/vol = aniso) vs LAPACK solve_banded."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        nz = 64
        vol = 1.0
        Vc = aniso * rng.uniform(0.9, 1.1, nz - 1)
        hsum = rng.uniform(0.0, 20.0, nz)
        D = vol + hsum
        D[:-1] += Vc
        D[1:] += Vc
        U = np.zeros(nz)
        U[:-1] = -Vc
        r = rng.uniform(-1, 1, nz)
        x = oracle.thomas(D, U, r)
        ab = np.zeros((3, nz))
        ab[0, 1:] = U[:-1]
        ab[1] = D
        ab[2, :-1] = U[:-1]
        ref = scipy.linalg.solve_banded((1, 1), ab, r)
        kappa = np.linalg.cond(_dense(D, U))
        assert np.max(np.abs(x - ref)) <= 10 * kappa * EPS * np.max(np.abs(ref))


def test_exact_rational_solve():
    """Against an exact Fraction Gaussian elimination on a 64-row column."""
    rng = np.random.default_rng(11)
    nz = 64
    Vc = 4096.0 * rng.uniform(0.9, 1.1, nz - 1)
    D = 1.0 + rng.uniform(0, 2, nz)
    D[:-1] += Vc
    D[1:] += Vc
    U = np.zeros(nz)
    U[:-1] = -Vc
    r = rng.uniform(-1, 1, nz)
    # exact solve of the tridiagonal system in rationals
    d = [Fraction(v) for v in D]
    u = [Fraction(v) for v in U]
    rr = [Fraction(v) for v in r]
    cp, dp = [Fraction(0)] * nz, [Fraction(0)] * nz
    cp[0] = u[0] / d[0]
    dp[0] = rr[0] / d[0]
    for k in range(1, nz):
        den = d[k] - u[k - 1] * cp[k - 1]
        cp[k] = u[k] / den if k < nz - 1 else Fraction(0)
        dp[k] = (rr[k] - u[k - 1] * dp[k - 1]) / den
    xe = [Fraction(0)] * nz
    xe[-1] = dp[-1]
    for k in range(nz - 2, -1, -1):
        xe[k] = dp[k] - cp[k] * xe[k + 1]
    exact = np.array([float(v) for v in xe])
    x = oracle.thomas(D, U, r)
    kappa = np.linalg.cond(_dense(D, U))
    assert np.max(np.abs(x - exact)) <= 4 * kappa * EPS * np.max(np.abs(exact))


def test_singular_column_reported():
    with pytest.raises(oracle.OracleError) as e:
        oracle.thomas([1.0, 1.0], [-1.0, 0.0], [1.0, 1.0])
    assert e.value.code == oracle.SINGULAR
