"""Matrix-form helpers for the oracle pins (tests only).

These rebuild, from exported bands and the neighbour table, the operators of
the paper as explicit (dense or scipy.sparse) matrices, so the oracle's
loop-form kernels can be checked against a different formulation: library
matvecs, dense LU, eigensolvers and the V-cycle written as a product of
matrices (Alg. 1).  Global dof index = k * n + c (layer-major).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def helmholtz_sparse(level: dict, nz: int, horizontal: bool = True, vertical: bool = True):
    """H^ (Eq. 8) as a scipy CSR matrix from the exported bands."""
    D, U, H, nbr = level["D"], level["U"], level["H"], level["nbr"]
    n = D.shape[1]
    N = nz * n
    rows, cols, vals = [np.arange(N)], [np.arange(N)], [D.reshape(-1)]
    if vertical and nz > 1:
        i = np.arange((nz - 1) * n)
        rows += [i, i + n]
        cols += [i + n, i]
        vals += [U[:-1].reshape(-1), U[:-1].reshape(-1)]
    if horizontal:
        k = np.repeat(np.arange(nz), n)
        c = np.tile(np.arange(n), nz)
        for j in range(3):
            rows.append(k * n + c)
            cols.append(k * n + nbr[c, j])
            vals.append(H[j].reshape(-1))
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))


def column_block_sparse(level: dict, nz: int):
    """T = H^_z: the column-block (tridiagonal) part of H^ (Eq. 9)."""
    return helmholtz_sparse(level, nz, horizontal=False)


def prolongation(n_fine: int, nz: int):
    """DG0 natural embedding P: fine cell c takes coarse c // 4."""
    n_c = n_fine // 4
    k = np.repeat(np.arange(nz), n_fine)
    c = np.tile(np.arange(n_fine), nz)
    return sp.csr_matrix((np.ones(nz * n_fine), (k * n_fine + c, k * n_c + c // 4)),
                         shape=(nz * n_fine, nz * n_c))


def smoother_matrices(A, T, omega):
    """One damped line-Jacobi sweep u <- u + omega T^{-1}(b - A u) as the
    affine map u <- S u + W b with S = I - omega T^{-1} A, W = omega T^{-1}."""
    Ad, Td = A.toarray(), T.toarray()
    W = omega * np.linalg.inv(Td)
    S = np.eye(A.shape[0]) - W @ Ad
    return S, W


def vcycle_matrix(levels: list, nz: int, nu_pre: int, nu_post: int, n_coarse: int, omega: float,
                  exact_coarse: bool = False):
    """The V-cycle of Alg. 1 as a matrix B with z = B b.

    ``levels`` = exported level dicts ordered coarsest -> finest.
    Zero initial guess on every level; coarse level: n_coarse sweeps from zero
    (or the exact inverse if ``exact_coarse``).
    """
    A0 = helmholtz_sparse(levels[0], nz)
    if exact_coarse:
        B = np.linalg.inv(A0.toarray())
    else:
        S, W = smoother_matrices(A0, column_block_sparse(levels[0], nz), omega)
        B = np.zeros_like(S)
        for _ in range(n_coarse):
            B = S @ B + W
    for lev in levels[1:]:
        A = helmholtz_sparse(lev, nz)
        Ad = A.toarray()
        S, W = smoother_matrices(A, column_block_sparse(lev, nz), omega)
        P = prolongation(lev["D"].shape[1], nz).toarray()
        R = P.T
        N = Ad.shape[0]
        M = np.zeros((N, N))           # u after presmoothing, as a function of b
        for _ in range(nu_pre):
            M = S @ M + W
        M = M + P @ B @ R @ (np.eye(N) - Ad @ M)   # restrict residual, coarse solve, prolong
        for _ in range(nu_post):
            M = S @ M + W
        B = M
    return B
