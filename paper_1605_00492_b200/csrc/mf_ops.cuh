// Matrix-free couplings (the paper's matrix-free operator
// store): the entries of H^ recomputed from the coefficient lam
// and the column geometry instead of read from the band store.
//
// Every coupling is formed with k_assemble's operations in k_assemble's order
// (reading R4, kernels.cu), so it is bitwise the stored band:
//   vertical   V = ((w2 area) (0.5 (lam_a + lam_b))) / dz
//   horizontal Hc_j = (((w2 len_j) dz) (0.5 (lam_c + lam_nj))) / cd_j
//   D = ((((vol + V_dn) + V_up) + Hc_0) + Hc_1) + Hc_2,  U_k = -V_up,  H_j = -Hc_j.
// The quotients by dz and by cd_j (constant down a column) use one
// reciprocal per column and the shared-reciprocal fast path (div_fast,
// bitwise '/'); EXACT = true uses '/' for the rare redo.
#pragma once
#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {

// Per-column constants: vol = area dz, w2 area, (w2 len_j) dz, cd_j and 1/cd_j.
struct ColumnGeom {
    double vol, w2a, hl[3], cd[3], ycd[3];
};

// geom: [7][ld] = area, len_0..2, cd_0..2 (DevLevel::geom)
__device__ __forceinline__ ColumnGeom column_geom(const double* __restrict__ geom, int64_t ld, int64_t c, double w2,
                                                  double dz) {
    ColumnGeom G;
    const double area = geom[c];
    G.vol = area * dz;
    G.w2a = w2 * area;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        G.hl[j] = (w2 * geom[(1 + j) * ld + c]) * dz;
        G.cd[j] = geom[(4 + j) * ld + c];
        G.ycd[j] = div_recip(G.cd[j]);
    }
    return G;
}

// CHECK = false: the level's operands were proven at build time to keep every
// numerator, divisor and quotient in [2^-900, 2^900] (or w2 = 0, where every
// numerator is +0 and the fast path returns +0 = +0 / b); there the fast path
// is exact without its per-quotient test (build_impl, DevLevel::mf_safe).
template <bool EXACT, bool CHECK = true>
__device__ __forceinline__ double mf_div(double a, double b, double y, bool& slow) {
    if (EXACT) return a / b;
    if (!CHECK) return div_fast_unchecked(a, b, y);
    return div_fast(a, b, y, slow);
}

// vertical coupling between layers with coefficients la (lower) and lb (upper)
template <bool EXACT, bool CHECK = true>
__device__ __forceinline__ double mf_vcoup(const ColumnGeom& G, double la, double lb, double dz, double ydz,
                                           bool& slow) {
    return mf_div<EXACT, CHECK>(G.w2a * (0.5 * (la + lb)), dz, ydz, slow);
}

// horizontal coupling through face j: own coefficient lk, neighbour's ln
template <bool EXACT, bool CHECK = true>
__device__ __forceinline__ double mf_hcoup(const ColumnGeom& G, int j, double lk, double ln, bool& slow) {
    return mf_div<EXACT, CHECK>(G.hl[j] * (0.5 * (lk + ln)), G.cd[j], G.ycd[j], slow);
}

// Diagonal from the couplings, k_assemble's order (absent vertical terms skipped).
__device__ __forceinline__ double mf_diag(const ColumnGeom& G, int k, int nz, double vdn, double vup, double h0,
                                          double h1, double h2) {
    double d = G.vol;
    if (k > 0) d = d + vdn;
    if (k < nz - 1) d = d + vup;
    d = d + h0;
    d = d + h1;
    d = d + h2;
    return d;
}

}  // namespace hmg
