"""Pins of the NEXT-3 core oracle (oracle/band_oracle.c): the per-column banded
LU of the next-to-lowest-order column operator (dgbtrf / dgbtrs, P:736-741;
m = 384 rows, bandwidth n_BW = 27), the paper's banded
matrix-vector kernel and the DG1 <-> DG0 p-coarsening by the
natural embedding (reading R21).

What fixes each part independently of the oracle's own code:
  * LAPACK itself (scipy.linalg.lapack.dgbtrf / dgbtrs): the same pivot rows
    (an integer decision) and factors / solutions equal to rounding (LAPACK's
    BLAS may fuse multiply-adds, so not bitwise);
  * the factorisation reproduces A: P L U = A assembled densely;
  * the solve inverts A: numpy.linalg.solve and the residual, within kappa eps;
  * LAPACK's exact-zero-pivot report (info = j + 1) on a singular column;
  * without pivots (a diagonally dominant tridiagonal column) the banded LU is
    the Thomas solve of the LO oracle;
  * the band product equals the dense product;
  * R P = 6 I, R = P^T (adjoint), P maps a constant to the constant.
"""
import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import oracle

EPS = np.finfo(np.float64).eps


def band_matrix(m, kl, ku, seed, dominant=False):
    rng = np.random.default_rng(seed)
    A = np.zeros((m, m))
    for i in range(m):
        lo, hi = max(0, i - kl), min(m, i + ku + 1)
        A[i, lo:hi] = rng.uniform(-1, 1, hi - lo)
        if dominant:
            A[i, i] = np.sum(np.abs(A[i, lo:hi])) + 1.0
    return A


def to_lapack(A, kl, ku):
    """Dense -> LAPACK band storage for dgbtrf, [2 kl + ku + 1][m]."""
    m = A.shape[0]
    ab = np.zeros((2 * kl + ku + 1, m))
    for j in range(m):
        for i in range(max(0, j - ku), min(m, j + kl + 1)):
            ab[kl + ku + i - j, j] = A[i, j]
    return ab


def to_rows(A, kl, ku):
    """Dense -> the paper's row-wise generalised band storage [m][kl + ku + 1]."""
    m = A.shape[0]
    r = np.zeros((m, kl + ku + 1))
    for i in range(m):
        for j in range(max(0, i - kl), min(m, i + ku + 1)):
            r[i, j - (i - kl)] = A[i, j]
    return r


SHAPES = [(384, 13, 13), (48, 13, 13), (40, 3, 5), (30, 5, 2), (17, 0, 0), (25, 1, 1), (13, 13, 13), (1, 13, 13)]


@pytest.mark.parametrize("m,kl,ku", SHAPES)
@pytest.mark.parametrize("seed", [0, 1])
def test_gbtrf_gbtrs_match_lapack(m, kl, ku, seed):
    A = band_matrix(m, kl, ku, seed)
    ab = to_lapack(A, kl, ku)
    lu, ipiv, info = oracle.gbtrf(ab, kl, ku)
    lu_l, ipiv_l, info_l = lapack.dgbtrf(ab, kl, ku)
    assert info == info_l == 0
    assert np.array_equal(ipiv, ipiv_l)                   # the same pivot rows, exactly
    scale = max(np.max(np.abs(lu_l)), 1.0)
    assert np.max(np.abs(lu - lu_l)) <= 64 * m * EPS * scale
    b = np.random.default_rng(seed + 10).uniform(-1, 1, m)
    x = oracle.gbtrs(lu, kl, ku, ipiv, b)
    x_l, info_s = lapack.dgbtrs(lu_l, kl, ku, b, ipiv_l)
    assert info_s == 0
    kappa = np.linalg.cond(A)
    assert np.max(np.abs(x - x_l)) <= 16 * m * kappa * EPS * max(np.max(np.abs(x_l)), 1.0)
    assert np.max(np.abs(x - np.linalg.solve(A, b))) <= 16 * m * kappa * EPS * max(np.max(np.abs(x_l)), 1.0)


@pytest.mark.parametrize("m,kl,ku", [(384, 13, 13), (40, 3, 5), (30, 5, 2)])
def test_gbtrf_reproduces_a(m, kl, ku):
    """P L U = A: L unit lower with the stored multipliers, U the upper band
    (kl + ku super-diagonals with the fill-in), P the recorded interchanges."""
    A = band_matrix(m, kl, ku, 3)
    lu, ipiv, info = oracle.gbtrf(to_lapack(A, kl, ku), kl, ku)
    assert info == 0
    kv = kl + ku
    U = np.zeros((m, m))
    for j in range(m):
        for i in range(max(0, j - kv), j + 1):
            U[i, j] = lu[kv + i - j, j]
    # apply L^-1 P to A column by column the way dgbtrf does: P_j then the Gauss transform
    B = A.copy()
    for j in range(m):
        B[[j, ipiv[j]]] = B[[ipiv[j], j]]
        for i in range(1, min(kl, m - 1 - j) + 1):
            B[j + i] -= lu[kv + i, j] * B[j]
    assert np.max(np.abs(B - U)) <= 64 * m * EPS * np.max(np.abs(A))


def test_gbtrf_singular_column_reported_like_lapack():
    m, kl, ku = 30, 4, 3
    A = band_matrix(m, kl, ku, 4)
    A[:, 11] = 0.0                                        # column 11 identically zero
    ab = to_lapack(A, kl, ku)
    _, _, info = oracle.gbtrf(ab, kl, ku)
    _, _, info_l = lapack.dgbtrf(ab, kl, ku)
    assert info == info_l == 12


def test_no_pivoting_reduces_to_thomas():
    """Tridiagonal, strictly diagonally dominant, symmetric: partial pivoting
    never swaps, and the banded LU solve is the LO Thomas solve (O6) to rounding."""
    m = 64
    rng = np.random.default_rng(5)
    U = -rng.uniform(0.5, 1.0, m)
    U[-1] = 0.0
    D = 2.5 + rng.uniform(0, 1, m)
    A = np.diag(D) + np.diag(U[:-1], 1) + np.diag(U[:-1], -1)
    lu, ipiv, info = oracle.gbtrf(to_lapack(A, 1, 1), 1, 1)
    assert info == 0 and np.array_equal(ipiv, np.arange(m))
    b = rng.uniform(-1, 1, m)
    x = oracle.gbtrs(lu, 1, 1, ipiv, b)
    assert np.max(np.abs(x - oracle.thomas(D, U, b))) <= 64 * EPS * np.max(np.abs(x))


@pytest.mark.parametrize("m,kl,ku", [(384, 13, 13), (40, 3, 5), (7, 13, 13), (20, 0, 0)])
def test_gbmv_is_the_dense_product(m, kl, ku):
    A = band_matrix(m, kl, ku, 6)
    x = np.random.default_rng(7).uniform(-1, 1, m)
    y = oracle.gbmv(to_rows(A, kl, ku), kl, ku, x)
    # in-order row sums (the kernel's order) are exact to the last bit of each product sum;
    # against BLAS's blocked product: rounding only
    assert np.max(np.abs(y - A @ x)) <= (kl + ku + 1) * EPS * np.max(np.abs(A) @ np.abs(x))
    ref = np.array([sum((A[i, j] * x[j] for j in range(max(0, i - kl), min(m, i + ku + 1))), 0.0) for i in range(m)])
    assert np.array_equal(y, ref)


def test_p_transfers_natural_embedding():
    rng = np.random.default_rng(8)
    ncol, nz = 37, 9
    u0 = rng.uniform(-1, 1, (ncol, nz))
    r1 = rng.uniform(-1, 1, (ncol, 6 * nz))
    Pu0 = oracle.p_prolong_add(u0, np.zeros((ncol, 6 * nz)))
    # P u0: every nodal value of cell k equals u0[k] (the constant in DG1)
    assert np.array_equal(Pu0.reshape(ncol, nz, 6), np.repeat(u0[:, :, None], 6, axis=2))
    # R P = 6 I exactly (a sum of six equal values ... up to rounding of the sum)
    RP = oracle.p_restrict(Pu0)
    assert np.max(np.abs(RP - 6 * u0)) <= 4 * EPS * np.max(np.abs(6 * u0))
    # R = P^T
    lhs = np.sum(oracle.p_restrict(r1) * u0)
    rhs = np.sum(r1 * Pu0)
    assert lhs == pytest.approx(rhs, rel=1e-13)
    # restriction = column sums of the 6 nodal values of each cell
    assert np.max(np.abs(oracle.p_restrict(r1) - r1.reshape(ncol, nz, 6).sum(axis=2))) <= 8 * EPS * 6
    # prolong-add adds
    base = rng.uniform(-1, 1, (ncol, 6 * nz))
    assert np.array_equal(oracle.p_prolong_add(u0, base), base + Pu0)
