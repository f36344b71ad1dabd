/*
 * band_oracle.c -- CPU oracle for NEXT-3's pinnable core (TEST INFRASTRUCTURE:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may load it).
 *
 * The next-to-lowest-order (NLO) discretisation of arXiv:1605.00492 stores the
 * column operator H^_z of each vertical column as a banded matrix with m = 384
 * rows (6 DG1 unknowns per cell x 64 layers) and bandwidth n_BW = 27
 * (P:1099-1106), and inverts it with the LAPACK routines dgbtrf (LU with
 * partial pivoting, precomputed once) and dgbtrs.  This file
 * writes out exactly those two algorithms for ONE column, step by step in
 * LAPACK's order (dgbtrf with kl < 32 runs its unblocked code dgbtf2), plus
 * the banded matrix-vector product of the paper's listing and the
 * p-coarsening transfers DG1 <-> DG0 by the natural embedding.
 * Plain C, fp64, no FMA contraction (-ffp-contract=off).
 *
 * Storage (LAPACK band format, 0-based): an m x m matrix with kl
 * sub- and ku super-diagonals is ab[j * ldab + r], j = matrix column, and
 * A(i, j) = ab[j * ldab + kv + i - j] with kv = kl + ku for the factorisation
 * (ldab >= 2 kl + ku + 1: the first kl rows receive U's fill-in).  The
 * paper's product kernel instead stores its operand row-wise (ora_gbmv).
 * ipiv[j] is the 0-based row interchanged with row j.
 */
#include <math.h>
#include <stdint.h>

/* dgbtf2 (LAPACK 3.x): LU factorisation with partial pivoting of a banded
 * matrix, in place.  Returns info: 0, or j + 1 when U(j, j) is exactly zero
 * (the factorisation is completed; U is singular), as LAPACK. */
int ora_gbtrf(int m, int kl, int ku, double* ab, int ldab, int32_t* ipiv) {
    const int kv = ku + kl;
    int info = 0;
#define AB(r, c) ab[(int64_t)(c) * ldab + (r)]
    /* zero the fill-in rows of columns ku+1 .. kv-1 (0-based) */
    for (int j = ku + 1; j < kv && j < m; j++)
        for (int i = kv - j; i < kl; i++) AB(i, j) = 0.0;
    int ju = 0;       /* last column touched by U so far (0-based) */
    for (int j = 0; j < m; j++) {
        if (j + kv < m)   /* fill-in rows of column j + kv */
            for (int i = 0; i < kl; i++) AB(i, j + kv) = 0.0;
        const int km = kl < m - 1 - j ? kl : m - 1 - j;
        /* idamax: first index of the largest |value| among km + 1 entries */
        int jp = 0;
        double vmax = fabs(AB(kv, j));
        for (int i = 1; i <= km; i++)
            if (fabs(AB(kv + i, j)) > vmax) { vmax = fabs(AB(kv + i, j)); jp = i; }
        ipiv[j] = j + jp;
        if (AB(kv + jp, j) != 0.0) {
            const int jlast = j + ku + jp < m - 1 ? j + ku + jp : m - 1;
            if (jlast > ju) ju = jlast;
            if (jp != 0)   /* dswap along matrix rows j and j + jp, columns j .. ju */
                for (int c = j; c <= ju; c++) {
                    const double t = AB(kv + jp - (c - j), c);
                    AB(kv + jp - (c - j), c) = AB(kv - (c - j), c);
                    AB(kv - (c - j), c) = t;
                }
            if (km > 0) {
                const double rp = 1.0 / AB(kv, j);       /* dscal by ONE / pivot */
                for (int i = 1; i <= km; i++) AB(kv + i, j) = AB(kv + i, j) * rp;
                /* dger, alpha = -1: A(j+i, c) += L(j+i) * (-U(j, c)), columns j+1 .. ju,
                   skipped where U(j, c) == 0 (as the reference BLAS) */
                for (int c = j + 1; c <= ju; c++) {
                    const double ujc = AB(kv - (c - j), c);
                    if (ujc == 0.0) continue;
                    const double temp = -ujc;
                    for (int i = 1; i <= km; i++)
                        AB(kv + i - (c - j), c) = AB(kv + i - (c - j), c) + AB(kv + i, j) * temp;
                }
            }
        } else if (info == 0) {
            info = j + 1;
        }
    }
#undef AB
    return info;
}

/* dgbtrs, TRANS = 'N', one right-hand side: x = A^-1 b from dgbtrf's factors.
 * L: row interchanges and dger updates (b(j+i) += L(j+i) * (-b(j)));
 * U: dtbsv('U', 'N', 'N') with kd = kl + ku super-diagonals, column-oriented
 * (x(j) = x(j) / U(j, j), then x(i) -= x(j) * U(i, j) above it; columns with
 * x(j) == 0 skipped, as the reference BLAS). */
void ora_gbtrs(int m, int kl, int ku, const double* ab, int ldab, const int32_t* ipiv, const double* b,
               double* x) {
    const int kv = ku + kl;
#define AB(r, c) ab[(int64_t)(c) * ldab + (r)]
    for (int i = 0; i < m; i++) x[i] = b[i];
    if (kl > 0)
        for (int j = 0; j < m - 1; j++) {
            const int lm = kl < m - 1 - j ? kl : m - 1 - j;
            const int l = ipiv[j];
            if (l != j) {
                const double t = x[l];
                x[l] = x[j];
                x[j] = t;
            }
            if (x[j] != 0.0) {
                const double temp = -x[j];
                for (int i = 1; i <= lm; i++) x[j + i] = x[j + i] + AB(kv + i, j) * temp;
            }
        }
    for (int j = m - 1; j >= 0; j--) {
        if (x[j] != 0.0) {
            x[j] = x[j] / AB(kv, j);
            const double temp = x[j];
            const int i0 = j - kv > 0 ? j - kv : 0;
            for (int i = j - 1; i >= i0; i--) x[i] = x[i] - temp * AB(kv + i - j, j);
        }
    }
#undef AB
}

/* y = A x, the paper's banded matrix-vector kernel (listing "ax")
 * with alpha = beta = 1 (W_x and W_y of the same layout): ROW-wise
 * generalised band storage, row i holding its bw = kl + ku + 1 entries
 * A(i, j), j = i - kl .. i + ku, at ab[i * bw + (j - (i - kl))] (entries with
 * j outside [0, m) unused); y(i) = 0, then y(i) += A(i, j) x(j) over
 * j = max(0, i - kl) .. min(m - 1, i + ku) in increasing j. */
void ora_gbmv(int m, int kl, int ku, const double* ab, const double* x, double* y) {
    const int bw = kl + ku + 1;
    for (int i = 0; i < m; i++) {
        const int j0 = i - kl > 0 ? i - kl : 0;
        const int j1 = i + ku < m - 1 ? i + ku : m - 1;
        double s = 0.0;
        for (int j = j0; j <= j1; j++) s = s + ab[(int64_t)i * bw + (j - (i - kl))] * x[j];
        y[i] = s;
    }
}

/* p-coarsening DG1 -> DG0 by the natural embedding (DESIGN.md
 * reading R21): DG1 unknowns of a column ordered cell-major (row 6 k + d for
 * the d-th nodal basis function of cell k); the embedding P maps a cell
 * constant u0 to the DG1 field with every nodal value equal to it, and the
 * restriction is its transpose, the sum of the 6 nodal residuals.
 * r1, u1: [ncol][6 nz] (column-contiguous, the paper's order); b0, u0: [ncol][nz]. */
void ora_p_restrict(int64_t ncol, int nz, const double* r1, double* b0) {
    for (int64_t c = 0; c < ncol; c++)
        for (int k = 0; k < nz; k++) {
            const double* r = r1 + c * 6 * nz + 6 * k;
            b0[c * nz + k] = ((((r[0] + r[1]) + r[2]) + r[3]) + r[4]) + r[5];
        }
}

void ora_p_prolong_add(int64_t ncol, int nz, const double* u0, double* u1) {
    for (int64_t c = 0; c < ncol; c++)
        for (int k = 0; k < nz; k++)
            for (int d = 0; d < 6; d++) u1[c * 6 * nz + 6 * k + d] = u1[c * 6 * nz + 6 * k + d] + u0[c * nz + k];
}
