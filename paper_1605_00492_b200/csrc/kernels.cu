// sm_100a kernels of the tensor-product multigrid Helmholtz path.
//
// All kernels are fp64 and HBM-bound (no tensor cores: nothing here is a
// dense contraction).  Layout: layer-major [nz][ld], cells contiguous, so a
// warp walking 32 adjacent columns reads and writes 256-byte coalesced rows
// at every layer.  Arithmetic follows the canonical operation order of
// DESIGN.md (readings R4-R10) with no FMA contraction (-fmad=false), so the
// V-cycle path is bitwise equal to the oracle.
#include <cfloat>
#include <cstdlib>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"
#include "mf_ops.cuh"

namespace hmg {
namespace {

constexpr int kApplyBlock = 128;
constexpr int kVecBlock = 256;
constexpr int kVecPerThread = 4;                  // consecutive cells per thread in vector kernels
constexpr int kVecCells = kVecBlock * kVecPerThread;
constexpr int kFinThreads = 1024;

__device__ __forceinline__ bool pivot_ok(double den) { return den > 0.0 && den <= DBL_MAX; }

// Deterministic block sum: fixed shuffle tree per warp, then warp partials
// summed in warp order by thread 0.
__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int off = 16; off > 0; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        for (int w = 0; w < nw; ++w) s = s + red[w];
    }
    return s;
}

// ---------------------------------------------------------------------------
// Setup: coefficient coarsening (reading R3) and band assembly (reading R4,
// Eq. 8 with lumped two-point couplings; u.n = 0 at top and bottom).
// ---------------------------------------------------------------------------
__global__ void k_coarsen_lam(const double* __restrict__ lf, int64_t ldf, double* __restrict__ lc,
                              int64_t ldc, int64_t nc) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (p >= nc) return;
    const double* l = lf + k * ldf + 4 * p;
    lc[k * ldc + p] = 0.25 * (((l[0] + l[1]) + l[2]) + l[3]);
}

__global__ void k_assemble(int64_t n, int64_t ld, int nz, const int32_t* __restrict__ nbr,
                           const double* __restrict__ geom, const double* __restrict__ lam,
                           double w2, double dz, double sn, double* __restrict__ bands) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c >= n) return;
    const int64_t s = (int64_t)nz * ld, i = k * ld + c;
    const double area = geom[c];
    const double vol = area * dz;
    const double lk = lam[i];
    double vdn = 0.0, vup = 0.0;
    // vertical couplings divided by 1 + omega_N^2 (Eq. 8; reading R24; exact for sn = 1)
    if (k > 0) vdn = (((w2 * area) * (0.5 * (lam[i - ld] + lk))) / dz) / sn;
    if (k < nz - 1) vup = (((w2 * area) * (0.5 * (lk + lam[i + ld]))) / dz) / sn;
    double hc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int32_t o = nbr[j * ld + c];
        const double lamf = 0.5 * (lk + lam[k * ld + o]);
        hc[j] = (((w2 * geom[(1 + j) * ld + c]) * dz) * lamf) / geom[(4 + j) * ld + c];
    }
    double d = vol;
    if (k > 0) d = d + vdn;
    if (k < nz - 1) d = d + vup;
    d = d + hc[0];
    d = d + hc[1];
    d = d + hc[2];
    bands[i] = d;
    bands[s + i] = (k < nz - 1) ? -vup : 0.0;
    bands[2 * s + i] = -hc[0];
    bands[3 * s + i] = -hc[1];
    bands[4 * s + i] = -hc[2];
}

// ---------------------------------------------------------------------------
// Operator apply y = H^ x (reading R5).  One thread per column walks
// the layers with a sliding window (x[k-1], x[k], x[k+1], U[k-1] in
// registers); the three face neighbours are gathered from the same layer row.
// DOT additionally accumulates x.y for the CG step (fused <p, H^ p>).
// ---------------------------------------------------------------------------
template <bool DOT, bool PUPD>
__global__ void __launch_bounds__(kApplyBlock) k_apply_t(LevelView L, const double* __restrict__ xin,
                                                         double* __restrict__ y, double* __restrict__ partial,
                                                         const double* __restrict__ zv, double* __restrict__ pnew,
                                                         const PcgScalars* __restrict__ sc) {
    __shared__ double red[kApplyBlock / 32];
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // vertical chunk of this thread (gridDim.y chunks; 1 on fine levels)
    const int nz = L.nz;
    const int kc = (nz + gridDim.y - 1) / gridDim.y;
    const int k0 = blockIdx.y * kc, k1 = min(nz, k0 + kc);
    double dot = 0.0;
    // PUPD (CG): the operand is p = z + beta p_old, formed on the fly for the
    // cell and its neighbours (same arithmetic as a separate update) and
    // written back for the cell -- the p update fused into the operator apply.
    double beta = 0.0;
    if (PUPD) beta = sc->beta;
    auto X = [&](int64_t i) -> double {
        if (PUPD) return zv[i] + beta * xin[i];
        return xin[i];
    };
    if (c < L.n && k0 < k1) {
        const int64_t ld = L.ld;
        const int32_t n0 = L.nbr[c], n1 = L.nbr[ld + c], n2 = L.nbr[2 * ld + c];
        double xm = k0 > 0 ? X((int64_t)(k0 - 1) * ld + c) : 0.0;
        double Um = k0 > 0 ? L.U[(int64_t)(k0 - 1) * ld + c] : 0.0;
        double xk = X((int64_t)k0 * ld + c);
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
            const int64_t row = k * ld, i = row + c;
            const double xp = (k + 1 < nz) ? X(i + ld) : 0.0;
            const double Uk = L.U[i];
            double acc = L.D[i] * xk;
            if (k > 0) acc = acc + Um * xm;
            if (k < nz - 1) acc = acc + Uk * xp;
            acc = acc + L.H0[i] * X(row + n0);
            acc = acc + L.H1[i] * X(row + n1);
            acc = acc + L.H2[i] * X(row + n2);
            y[i] = acc;
            if (PUPD) pnew[i] = xk;
            if (DOT) dot = dot + xk * acc;
            xm = xk;
            xk = xp;
            Um = Uk;
        }
    }
    if (DOT) {
        const double s = block_sum(dot, red);
        if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// Matrix-free operator apply (the paper's matrix-free
// store): the couplings of reading R4 are recomputed from the
// coefficient lam and the column geometry instead of streamed from the band
// store -- lam, x in and y out (24 B/dof instead of 56).  Every coupling is
// formed with k_assemble's operations in k_assemble's order, so it is
// bitwise the stored band; the quotients by dz and by the centroid distances
// use one reciprocal per column (div_fast, bitwise '/', exact redo otherwise).
// ---------------------------------------------------------------------------
// One column's layers [k0, k1) of y = H^ x with the couplings recomputed.
// Returns the column's contribution to x.y (DOT).
template <bool DOT, bool PUPD, bool EXACT>
__device__ __forceinline__ double apply_mf_column(const LevelView& L, const ColumnGeom& G, const double* __restrict__ lam,
                                                  double dz, double ydz, int64_t c, int k0, int k1,
                                                  const double* __restrict__ xin, double* __restrict__ y,
                                                  const double* __restrict__ zv, double* __restrict__ pnew, double beta,
                                                  bool& slow) {
    const int nz = L.nz;
    const int64_t ld = L.ld;
    const int32_t n0 = L.nbr[c], n1 = L.nbr[ld + c], n2 = L.nbr[2 * ld + c];
    auto X = [&](int64_t i) -> double {
        if (PUPD) return zv[i] + beta * xin[i];
        return xin[i];
    };
    // vertical coupling between layers k and k + 1 (k_assemble's vup / vdn)
    auto vcoup = [&](double la, double lb) { return mf_vcoup<EXACT>(G, la, lb, dz, ydz, slow); };
    double dot = 0.0;
    double lk = lam[(int64_t)k0 * ld + c];
    double vdn = 0.0, xm = 0.0;
    if (k0 > 0) {
        vdn = vcoup(lam[(int64_t)(k0 - 1) * ld + c], lk);
        xm = X((int64_t)(k0 - 1) * ld + c);
    }
    double xk = X((int64_t)k0 * ld + c);
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
        const int64_t row = k * ld, i = row + c;
        double xp = 0.0, lp = 0.0, vup = 0.0;
        if (k + 1 < nz) {
            xp = X(i + ld);
            lp = lam[i + ld];
            vup = vcoup(lk, lp);
        }
        const double hc0 = mf_hcoup<EXACT>(G, 0, lk, lam[row + n0], slow);
        const double hc1 = mf_hcoup<EXACT>(G, 1, lk, lam[row + n1], slow);
        const double hc2 = mf_hcoup<EXACT>(G, 2, lk, lam[row + n2], slow);
        const double d = mf_diag(G, k, nz, vdn, vup, hc0, hc1, hc2);
        double acc = d * xk;
        if (k > 0) acc = acc + (-vdn) * xm;
        if (k < nz - 1) acc = acc + (-vup) * xp;
        acc = acc + (-hc0) * X(row + n0);
        acc = acc + (-hc1) * X(row + n1);
        acc = acc + (-hc2) * X(row + n2);
        y[i] = acc;
        if (PUPD) pnew[i] = xk;
        if (DOT) dot = dot + xk * acc;
        xm = xk;
        xk = xp;
        vdn = vup;
        lk = lp;
    }
    return dot;
}

template <bool DOT, bool PUPD>
__global__ void __launch_bounds__(kApplyBlock) k_apply_mf(LevelView L, const double* __restrict__ geom,
                                                          const double* __restrict__ lam, double w2, double dz,
                                                          const double* __restrict__ xin, double* __restrict__ y,
                                                          double* __restrict__ partial, const double* __restrict__ zv,
                                                          double* __restrict__ pnew, const PcgScalars* __restrict__ sc) {
    __shared__ double red[kApplyBlock / 32];
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int nz = L.nz;
    const int kc = (nz + gridDim.y - 1) / gridDim.y;
    const int k0 = blockIdx.y * kc, k1 = min(nz, k0 + kc);
    double dot = 0.0;
    const double beta = PUPD ? sc->beta : 0.0;
    if (c < L.n && k0 < k1) {
        const ColumnGeom G = column_geom(geom, L.ld, c, w2, dz);
        const double ydz = div_recip(dz);
        bool slow = false;
        dot = apply_mf_column<DOT, PUPD, false>(L, G, lam, dz, ydz, c, k0, k1, xin, y, zv, pnew, beta, slow);
        if (slow)   // rare: a quotient left the fast path's exact range; redo the column with '/'
            dot = apply_mf_column<DOT, PUPD, true>(L, G, lam, dz, ydz, c, k0, k1, xin, y, zv, pnew, beta, slow);
    }
    if (DOT) {
        const double s = block_sum(dot, red);
        if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// Fused damped line-Jacobi sweep (Eq. 10 read with Eq. 13; readings R6/R7):
//   r = b - H^ u;  delta = T^{-1} r (Thomas);  u' = u + omega delta
// One thread per column.  Forward pass computes the residual row and the
// Thomas elimination; the (z_k, g_k) state of the column sits in shared
// memory, then back substitution writes u'.  ZERO: u = 0 (u' = omega T^-1 b,
// P:992-995 "before the pre-smoother application the solution is zero").
// PROLONG: the incoming u is u + P u_c (the prolongation M4 of Alg. 1 fused
// into the first post-smoothing sweep; identical arithmetic).
// ---------------------------------------------------------------------------
template <bool ZERO, bool PROLONG>
__global__ void k_sweep(LevelView L, const double* __restrict__ b, const double* __restrict__ uin,
                        const double* __restrict__ uc, int64_t ldc, double* __restrict__ uout,
                        double omega, int ref, unsigned long long* __restrict__ bad) {
    extern __shared__ double sm[];
    const int T = blockDim.x, t = threadIdx.x;
    double* zs = sm;
    double* gs = sm + L.nz * T;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + t;
    if (c >= L.n) return;
    const int64_t ld = L.ld;
    const int nz = L.nz;
    int32_t n0 = 0, n1 = 0, n2 = 0;
    if (!ZERO) { n0 = L.nbr[c]; n1 = L.nbr[ld + c]; n2 = L.nbr[2 * ld + c]; }
    auto U_IN = [&](int k, int64_t cell) -> double {
        if (PROLONG) return uin[k * ld + cell] + uc[k * ldc + (cell >> 2)];
        return uin[k * ld + cell];
    };
    double um = 0.0, uk = 0.0, Um = 0.0, den = 0.0, zprev = 0.0;
    if (!ZERO) uk = U_IN(0, c);
    bool ok = true;
    for (int k = 0; k < nz; ++k) {
        const int64_t i = k * ld + c;
        const double Dk = L.D[i];
        const double Uk = L.U[i];
        double r;
        double up = 0.0;
        if (ZERO) {
            r = b[i];
        } else {
            if (k < nz - 1) up = U_IN(k + 1, c);
            double acc = Dk * uk;
            if (k > 0) acc = acc + Um * um;
            if (k < nz - 1) acc = acc + Uk * up;
            acc = acc + L.H0[i] * U_IN(k, n0);
            acc = acc + L.H1[i] * U_IN(k, n1);
            acc = acc + L.H2[i] * U_IN(k, n2);
            r = b[i] - acc;
        }
        double z;
        if (k == 0) {
            den = Dk;
            z = r / den;
        } else {
            const double g = Um / den;
            gs[(k - 1) * T + t] = g;
            den = Dk - Um * g;
            z = (r - Um * zprev) / den;
        }
        ok = ok && pivot_ok(den);
        zs[k * T + t] = z;
        zprev = z;
        um = uk;
        uk = up;
        Um = Uk;
    }
    if (!ok) atomicMin(bad, ((unsigned long long)ref << 40) | (unsigned long long)c);
    double dl = zs[(nz - 1) * T + t];
    {
        const int64_t i = (int64_t)(nz - 1) * ld + c;
        uout[i] = ZERO ? omega * dl : U_IN(nz - 1, c) + omega * dl;
    }
    for (int k = nz - 2; k >= 0; --k) {
        dl = zs[k * T + t] - gs[k * T + t] * dl;
        const int64_t i = k * ld + c;
        uout[i] = ZERO ? omega * dl : U_IN(k, c) + omega * dl;
    }
}

// ---------------------------------------------------------------------------
// Transfers (reading R8): restriction b_c = ((r0 + r1) + r2) + r3 over the
// children 4p..4p+3 (R = P^T); prolongation u_f = u_f + u_c[c >> 2].
// ---------------------------------------------------------------------------
__global__ void k_restrict(const double* __restrict__ r, int64_t ldf, double* __restrict__ bc,
                           int64_t ldc, int64_t nc, int64_t coff) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (p >= nc) return;
    const double2* q = reinterpret_cast<const double2*>(r + k * ldf + 4 * p);
    const double2 a = q[0], b = q[1];
    bc[k * ldc + coff + p] = ((a.x + a.y) + b.x) + b.y;
}

// Residual of the current iterate restricted to the coarse level: each lane
// computes r = b - H^ u for its column; groups of 4 lanes (the 4 children of
// one parent) combine in child order through shuffles.
__global__ void __launch_bounds__(kApplyBlock) k_resid_restrict(LevelView L, const double* __restrict__ b,
                                                                const double* __restrict__ u,
                                                                double* __restrict__ bc, int64_t ldc, int64_t coff) {
    const int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = cc < L.n;          // n is a multiple of 4: groups are all-valid or all-invalid
    const int64_t c = valid ? cc : L.n - 1;
    const int64_t ld = L.ld;
    const int nz = L.nz;
    const int kc = (nz + gridDim.y - 1) / gridDim.y;
    const int k0 = blockIdx.y * kc, k1 = min(nz, k0 + kc);
    const int32_t n0 = L.nbr[c], n1 = L.nbr[ld + c], n2 = L.nbr[2 * ld + c];
    const int lane = threadIdx.x & 31;
    if (k0 >= k1) return;                 // uniform across the block
    double um = k0 > 0 ? u[(int64_t)(k0 - 1) * ld + c] : 0.0;
    double Um = k0 > 0 ? L.U[(int64_t)(k0 - 1) * ld + c] : 0.0;
    double uk = u[(int64_t)k0 * ld + c];
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const int64_t row = k * ld, i = row + c;
        const double up = (k + 1 < nz) ? u[i + ld] : 0.0;
        const double Uk = L.U[i];
        double acc = L.D[i] * uk;
        if (k > 0) acc = acc + Um * um;
        if (k < nz - 1) acc = acc + Uk * up;
        acc = acc + L.H0[i] * u[row + n0];
        acc = acc + L.H1[i] * u[row + n1];
        acc = acc + L.H2[i] * u[row + n2];
        const double r = b[i] - acc;
        const double r1 = __shfl_down_sync(0xffffffffu, r, 1);
        const double r2 = __shfl_down_sync(0xffffffffu, r, 2);
        const double r3 = __shfl_down_sync(0xffffffffu, r, 3);
        if (valid && (lane & 3) == 0) bc[k * ldc + coff + (cc >> 2)] = ((r + r1) + r2) + r3;
        um = uk;
        uk = up;
        Um = Uk;
    }
}

__global__ void k_prolong_add(const double* __restrict__ uin, const double* __restrict__ uc,
                              double* __restrict__ uout, int64_t ld, int64_t ldc, int64_t n, int64_t coff) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c >= n) return;
    uout[k * ld + c] = uin[k * ld + c] + uc[k * ldc + coff + (c >> 2)];
}

// ---------------------------------------------------------------------------
// Multi-GPU staging.  Halo send buffer: [send_total][nz] (cell
// major, so each peer's segment is contiguous); receive buffer: [n_halo][nz],
// each peer's run of halo slots contiguous.  Coarse gather: owned segment of
// every layer packed [nz][cnt]; the all-gather result is [nranks][nz][cnt].
// ---------------------------------------------------------------------------
__global__ void k_halo_pack(const double* __restrict__ v, int64_t ld, int nz, const int32_t* __restrict__ idx,
                            int64_t total, double* __restrict__ buf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= total * nz) return;
    const int64_t i = t / nz;
    const int k = (int)(t - i * nz);
    buf[t] = v[k * ld + idx[i]];
}

__global__ void k_halo_unpack(const double* __restrict__ buf, int64_t n_halo, int nz, double* __restrict__ v,
                              int64_t ld, int64_t n_own) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_halo * nz) return;
    const int64_t h = t / nz;
    const int k = (int)(t - h * nz);
    v[k * ld + n_own + h] = buf[t];
}

__global__ void k_gather_pack(const double* __restrict__ v, int64_t ld, int64_t off, int64_t cnt,
                              double* __restrict__ buf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (i < cnt) buf[k * cnt + i] = v[k * ld + off + i];
}

__global__ void k_gather_unpack(const double* __restrict__ buf, int64_t cnt, int nz, double* __restrict__ v,
                                int64_t ld) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y, q = blockIdx.z;
    if (i < cnt) v[k * ld + q * cnt + i] = buf[((int64_t)q * nz + k) * cnt + i];
}

// Multi-GPU: the halo slots [n_own, n_own + n_halo) of p_new = z + beta p_old,
// from the (exchanged) halo slots of z and p_old -- the addition the fused
// apply forms for the owned cells.
__global__ void k_halo_pupdate(const double* __restrict__ z, const double* __restrict__ pold, double* __restrict__ pnew,
                               int64_t n_own, int64_t n_halo, int64_t ld, int nz, const PcgScalars* __restrict__ sc) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_halo * nz) return;
    const int k = (int)(t / n_halo);
    const int64_t i = k * ld + n_own + (t - (int64_t)k * n_halo);
    pnew[i] = z[i] + sc->beta * pold[i];
}

__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ z, int64_t n, int64_t ld,
                           const PcgScalars* __restrict__ sc) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c >= n) return;
    const int64_t i = k * ld + c;
    p[i] = z[i] + sc->beta * p[i];
}

// ---------------------------------------------------------------------------
// CG vector kernels (reading R10).  Block (bx, by) owns kVecCells consecutive
// cells (2 per 16-byte access, 4 per thread) of the layers [by*kc, by*kc+kc);
// per-block partial sums are reduced by k_finalize in a fixed order, so dots
// are deterministic (not equal in rounding to the oracle's sequential sum;
// see DESIGN.md parity contract).
// ---------------------------------------------------------------------------
struct VecRange {
    int64_t c0;   // first cell of this thread's first pair
    int k0, k1;   // layers
};
__device__ __forceinline__ VecRange vec_range(int nz) {
    const int kc = (nz + gridDim.y - 1) / gridDim.y;
    VecRange v;
    v.c0 = blockIdx.x * (int64_t)kVecCells + 2 * threadIdx.x;
    v.k0 = blockIdx.y * kc;
    v.k1 = min(nz, v.k0 + kc);
    return v;
}

__global__ void __launch_bounds__(kVecBlock) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                   int64_t n, int64_t ld, int nz, double* __restrict__ partial,
                                                   FinArgs fin) {
    __shared__ double red[kVecBlock / 32];
    const VecRange v = vec_range(nz);
    double s = 0.0;
    for (int k = v.k0; k < v.k1; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = v.c0 + h * 2 * kVecBlock;
            if (c < n) {
                const double2 x = *reinterpret_cast<const double2*>(a + k * ld + c);
                const double2 y = *reinterpret_cast<const double2*>(b + k * ld + c);
                s = s + x.x * y.x;
                s = s + x.y * y.y;
            }
        }
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = tot;
    fin_fused(fin, partial);
}

// FIRST: the first iteration from x = 0, r = b -- reads b instead of r and does
// not read x; x = 0 + alpha p and r = b - alpha q are the same operations.
// PART: 0 both updates, 1 r only (with the partial <r, r>), 2 x only (the
// PCG defers it to a side stream under the V-cycle's coarse tail).
template <bool FIRST, int PART = 0>
__global__ void __launch_bounds__(kVecBlock) k_update_xr(double* __restrict__ x, double* __restrict__ r,
                                                         const double* __restrict__ p, const double* __restrict__ q,
                                                         const double* __restrict__ rin, int64_t n, int64_t ld, int nz,
                                                         const PcgScalars* sc, double* __restrict__ partial,
                                                         FinArgs fin = FinArgs()) {
    __shared__ double red[kVecBlock / 32], red2[kVecBlock / 32];
    const double alpha = sc->alpha;
    const VecRange v = vec_range(nz);
    // FIRST with kFinRRBB: <b, b> as well (the PCG's ||b||, no separate dot)
    const bool with_bb = FIRST && PART != 2 && fin.op == kFinRRBB;
    double s = 0.0, sb = 0.0;
    for (int k = v.k0; k < v.k1; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = v.c0 + h * 2 * kVecBlock;
            if (c < n) {
                const int64_t i = k * ld + c;
                if (PART != 1) {
                    double2 xx = FIRST ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(x + i);
                    const double2 pp = *reinterpret_cast<const double2*>(p + i);
                    xx.x = xx.x + alpha * pp.x;
                    xx.y = xx.y + alpha * pp.y;
                    *reinterpret_cast<double2*>(x + i) = xx;
                }
                if (PART != 2) {
                    double2 rr = *reinterpret_cast<const double2*>((FIRST ? rin : r) + i);
                    if (with_bb) {
                        sb = sb + rr.x * rr.x;
                        sb = sb + rr.y * rr.y;
                    }
                    const double2 qq = *reinterpret_cast<const double2*>(q + i);
                    rr.x = rr.x - alpha * qq.x;
                    rr.y = rr.y - alpha * qq.y;
                    *reinterpret_cast<double2*>(r + i) = rr;
                    s = s + rr.x * rr.x;
                    s = s + rr.y * rr.y;
                }
            }
        }
    if (PART == 2) return;
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = tot;
    if (with_bb) {
        const double totb = block_sum(sb, red2);
        if (threadIdx.x == 0) partial[gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = totb;
    }
    fin_fused(fin, partial);
}

__device__ __forceinline__ void scalar_op(PcgScalars* sc, int op, double S) { pcg_scalar_op(sc, op, S); }

// pub: non-null for the scalars the host reads (||b||^2, ||r||^2 with the
// singular-pivot flag): the updated struct is also written to mapped pinned
// host memory, so the host's read needs no copy-engine transfer (which would
// queue behind a large device->host copy on another stream)
__device__ __forceinline__ void publish(const PcgScalars* sc, PcgScalars* pub) {
    if (pub) *pub = *sc;
}

__global__ void __launch_bounds__(kFinThreads) k_finalize(const double* __restrict__ partial, int np, int op,
                                                          PcgScalars* __restrict__ sc, PcgScalars* pub) {
    __shared__ double red[kFinThreads / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += kFinThreads) s = s + partial[i];
    const double S = block_sum(s, red);
    if (threadIdx.x != 0) return;
    if (op < 0) {                 // rank-local total, to be all-reduced
        sc->tmp = S;
        return;
    }
    scalar_op(sc, op, S);
    publish(sc, pub);
}

__global__ void k_scalar_op(PcgScalars* __restrict__ sc, int op, PcgScalars* pub) {
    scalar_op(sc, op, sc->tmp);
    publish(sc, pub);
}

__global__ void k_copy_rows(const double* __restrict__ src, int64_t sld, double* __restrict__ dst, int64_t dld,
                            int64_t n) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c < n) dst[k * dld + c] = src[k * sld + c];
}

inline unsigned blocks(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// Vertical chunks for the column kernels: 1 on levels with enough columns to
// fill the GPU; on small (coarse) levels split the layers so that the
// sequential per-thread loop is short (these levels are latency-bound).
unsigned vchunks(int64_t n, int nz) {
    const int64_t target = 148LL * 1024;
    int64_t c = (target + n - 1) / n;
    if (c > nz / 4) c = nz / 4;
    return c < 1 ? 1u : (unsigned)c;
}

int sweep_block(int nz) {
    int t = 4096 / nz;             // 2 * nz * t * 8 B = 64 KB of Thomas state per block
    t = t < 32 ? 32 : (t > 128 ? 128 : t);
    return t & ~31;
}

template <bool Z, bool P>
void set_smem_attr() {
    static bool done = false;
    if (!done) {
        cudaFuncSetAttribute(k_sweep<Z, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        done = true;
    }
}

}  // namespace

ProfScope::ProfScope(const Hierarchy& h, int cls, int ref, cudaStream_t st) : H(h), s(st) {
    Profiler& P = H.prof;
    if (!P.on) return;
    if ((P.only_cls >= 0 && cls != P.only_cls) || (P.only_ref >= 0 && ref != P.only_ref)) return;
    if (P.used + 2 > P.pool.size()) {
        for (int i = 0; i < 256; ++i) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return;
            P.pool.push_back(e);
        }
    }
    cudaEvent_t start = P.pool[P.used];
    stop = P.pool[P.used + 1];
    P.used += 2;
    P.cls.push_back(cls);
    P.ref.push_back(ref);
    cudaEventRecord(start, s);
}

ProfScope::~ProfScope() {
    if (stop) cudaEventRecord(stop, s);
}

// Sum of the per-block partials into the PCG scalar `op`; across ranks
// (multi-GPU) the rank-local totals are all-reduced first.
FinArgs fin_take(const Hierarchy& H) {
    FinArgs f;
    if (H.fin_op >= 0) {
        f.op = H.fin_op;
        f.sc = H.scal;
        f.pub = (f.op == kFinBB || f.op == kFinRR || f.op == kFinRRBB) ? H.scal_pub : nullptr;
        H.fin_fused = true;
    }
    H.fin_op = -1;
    return f;
}

void fin_begin(const Hierarchy& H, int op) {
    H.fin_op = (!H.comm || (H.nranks == 1 && !H.force_coll)) ? op : -1;
    H.fin_fused = false;
}

void finalize_parts(const Hierarchy& H, int nparts, int op, cudaStream_t s) {
    H.fin_op = -1;
    if (H.fin_fused) {                 // the partial-sum launch finalized itself
        H.fin_fused = false;
        return;
    }
    PcgScalars* pub = (op == kFinBB || op == kFinRR) ? H.scal_pub : nullptr;
    if (!H.comm || (H.nranks == 1 && !H.force_coll)) {
        k_finalize<<<1, kFinThreads, 0, s>>>(H.partials, nparts, op, H.scal, pub);
        ++H.launches;
        return;
    }
    k_finalize<<<1, kFinThreads, 0, s>>>(H.partials, nparts, -1, H.scal, nullptr);
    ++H.launches;
    dist_allreduce_tmp(H, s);
    k_scalar_op<<<1, 1, 0, s>>>(H.scal, op, pub);
    ++H.launches;
}

int partials_needed(int64_t n, int nz) {
    const int a = (int)(blocks(n, kApplyBlock) * vchunks(n, nz)), v = (int)blocks(n, kVecCells);
    return a > v ? a : v;
}

void launch_coarsen_lam(const Hierarchy& H, const DevLevel& F, const DevLevel& C, cudaStream_t s) {
    dim3 g(blocks(C.n, 256), H.nz);
    k_coarsen_lam<<<g, 256, 0, s>>>(F.lam, F.ld, C.lam, C.ld, C.n);
    ++H.launches;
}

// Edge-deduplicated couplings: H_e[k][e] = H_j[k][a] for the owner (a, j) of
// edge e (a copy of the band value; the other cell's band holds the same
// bits, the assembly being bitwise symmetric).
__global__ void k_edge_h(const int32_t* __restrict__ own, int64_t ne, int64_t ldE, int64_t ld, int nz,
                         const double* __restrict__ bands, double* __restrict__ hedge) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (e >= ne) return;
    const int64_t a = own[e], j = own[ldE + e];
    hedge[k * ldE + e] = bands[((2 + j) * nz + k) * ld + a];
}

void launch_edge_h(const Hierarchy& H, const DevLevel& L, int64_t nedges, cudaStream_t s) {
    dim3 g(blocks(nedges, 256), H.nz);
    k_edge_h<<<g, 256, 0, s>>>(L.edge_own, nedges, L.edge.ldE, L.ld, H.nz, L.bands, L.hedge);
    ++H.launches;
}

void launch_assemble(const Hierarchy& H, const DevLevel& L, cudaStream_t s) {
    dim3 g(blocks(L.n, 256), H.nz);
    k_assemble<<<g, 256, 0, s>>>(L.n, L.ld, H.nz, L.nbr, L.geom, L.lam, H.w2, H.dz, H.sn, L.bands);
    ++H.launches;
}

void launch_apply(const Hierarchy& H, const DevLevel& L, const double* x, double* y, cudaStream_t s) {
    ProfScope ps(H, kKApply, L.ref, s);
    if (!H.matrix_free && apply_st_supported(H, L)) {
        launch_apply_st(H, L, x, y, false, s);
        return;
    }
    dim3 g(blocks(L.n, kApplyBlock), vchunks(L.n, H.nz));
    if (H.matrix_free)
        k_apply_mf<false, false><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), L.geom, L.lam, H.w2, H.dz, x, y, nullptr,
                                                           nullptr, nullptr, nullptr);
    else
        k_apply_t<false, false><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), x, y, nullptr, nullptr, nullptr, nullptr);
    ++H.launches;
}

void launch_apply_dot(const Hierarchy& H, const DevLevel& L, const double* x, double* y, cudaStream_t s) {
    ProfScope ps(H, kKApply, L.ref, s);
    if (!H.matrix_free && apply_st_supported(H, L)) {
        fin_begin(H, kFinPQ);
        const int n = launch_apply_st(H, L, x, y, true, s);
        finalize_parts(H, n, kFinPQ, s);
        return;
    }
    dim3 g(blocks(L.n, kApplyBlock), vchunks(L.n, H.nz));
    if (H.matrix_free)
        k_apply_mf<true, false><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), L.geom, L.lam, H.w2, H.dz, x, y, H.partials,
                                                          nullptr, nullptr, nullptr);
    else
        k_apply_t<true, false><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), x, y, H.partials, nullptr, nullptr, nullptr);
    ++H.launches;
    finalize_parts(H, (int)(g.x * g.y), kFinPQ, s);
}

void launch_sweep(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin,
                  const double* uc, double* uout, double omega, cudaStream_t s) {
    ProfScope ps(H, !uin ? kKSweepZero : (uc ? kKSweepProlong : kKSweep), L.ref, s);
    if (H.use_small_sweep && sweep_small_supported(H, L)) {
        launch_sweep_small(H, L, b, uin, uc, uout, omega, 1, s);
        return;
    }
    if ((uin || H.matrix_free) && !L.fden && H.use_tc_sweep && sweep_st_supported(H, L)) {
        launch_sweep_st(H, L, b, uin, uc, uout, omega, s);
        return;
    }
    if (H.use_tc_sweep && sweep_tc_supported(H, L)) {
        launch_sweep_tc(H, L, b, uin, uc, uout, omega, s);
        return;
    }
    const int T = sweep_block(H.nz);
    const size_t smem = (size_t)2 * H.nz * T * sizeof(double);
    const unsigned g = blocks(L.n, T);
    unsigned long long* bad = &H.scal->bad;
    const int64_t ldc = uc ? H.lev[L.ref - 1].ld : 0;
    if (!uin) {
        set_smem_attr<true, false>();
        k_sweep<true, false><<<g, T, smem, s>>>(L.view(H.nz), b, nullptr, nullptr, 0, uout, omega, L.ref, bad);
    } else if (uc) {
        set_smem_attr<false, true>();
        k_sweep<false, true><<<g, T, smem, s>>>(L.view(H.nz), b, uin, uc, ldc, uout, omega, L.ref, bad);
    } else {
        set_smem_attr<false, false>();
        k_sweep<false, false><<<g, T, smem, s>>>(L.view(H.nz), b, uin, nullptr, 0, uout, omega, L.ref, bad);
    }
    ++H.launches;
}

void launch_apply_pupdate_dot(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                              double* q, cudaStream_t s) {
    ProfScope ps(H, kKApplyP, L.ref, s);
    if (!H.matrix_free && apply_st_supported(H, L)) {
        fin_begin(H, kFinPQ);
        const int n = launch_apply_pupdate_st(H, L, z, pold, pnew, q, s);
        finalize_parts(H, n, kFinPQ, s);
        return;
    }
    dim3 g(blocks(L.n, kApplyBlock), vchunks(L.n, H.nz));
    if (H.matrix_free)
        k_apply_mf<true, true><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), L.geom, L.lam, H.w2, H.dz, pold, q, H.partials,
                                                         z, pnew, H.scal);
    else
        k_apply_t<true, true><<<g, kApplyBlock, 0, s>>>(L.view(H.nz), pold, q, H.partials, z, pnew, H.scal);
    ++H.launches;
    finalize_parts(H, (int)(g.x * g.y), kFinPQ, s);
}

void launch_restrict(const Hierarchy& H, const DevLevel& F, const double* r, double* bc, cudaStream_t s) {
    ProfScope ps(H, kKRestrict, F.ref, s);
    const DevLevel& C = H.lev[F.ref - 1];
    dim3 g(blocks(F.n / 4, 256), H.nz);
    k_restrict<<<g, 256, 0, s>>>(r, F.ld, bc, C.ld, F.n / 4, F.dist.coff);
    ++H.launches;
}

void launch_resid_restrict(const Hierarchy& H, const DevLevel& F, const double* b, const double* u,
                           double* bc, cudaStream_t s) {
    ProfScope ps(H, kKResidRestrict, F.ref, s);
    const DevLevel& C = H.lev[F.ref - 1];
    if (resid_st_supported(H, F)) {
        launch_resid_restrict_st(H, F, b, u, bc, C.ld, F.dist.coff, s);
        return;
    }
    dim3 g(blocks(F.n, kApplyBlock), vchunks(F.n, H.nz));
    k_resid_restrict<<<g, kApplyBlock, 0, s>>>(F.view(H.nz), b, u, bc, C.ld, F.dist.coff);
    ++H.launches;
}

void launch_prolong_add(const Hierarchy& H, const DevLevel& F, const double* uin, const double* uc,
                        double* uout, cudaStream_t s) {
    ProfScope ps(H, kKProlong, F.ref, s);
    const DevLevel& C = H.lev[F.ref - 1];
    dim3 g(blocks(F.n, 256), H.nz);
    k_prolong_add<<<g, 256, 0, s>>>(uin, uc, uout, F.ld, C.ld, F.n, F.dist.coff);
    ++H.launches;
}

// Grid of the vector kernels: column blocks x layer chunks, ~8 blocks per SM.
dim3 vec_grid(int64_t n, int nz) {
    const unsigned gx = blocks(n, kVecCells);
    unsigned gy = (unsigned)((148 * 8 + gx - 1) / gx);
    if (gy > (unsigned)nz) gy = (unsigned)nz;
    return dim3(gx, gy < 1 ? 1 : gy);
}

void launch_dot(const Hierarchy& H, const DevLevel& L, const double* a, const double* b, cudaStream_t s) {
    ProfScope ps(H, kKVector, H.fine_ref, s);
    k_dot<<<vec_grid(L.n, H.nz), kVecBlock, 0, s>>>(a, b, L.n, L.ld, H.nz, H.partials, fin_take(H));
    ++H.launches;
}

void launch_finalize(const Hierarchy& H, int op, cudaStream_t s) {
    const DevLevel& L = H.lev[H.fine_ref];
    const dim3 g = vec_grid(L.n, H.nz);
    finalize_parts(H, (int)(g.x * g.y), op, s);
}

void launch_finalize_local(const Hierarchy& H, int nparts, cudaStream_t s) {
    k_finalize<<<1, kFinThreads, 0, s>>>(H.partials, nparts, -1, H.scal, nullptr);
    ++H.launches;
}

void launch_scalar_op(const Hierarchy& H, int op, cudaStream_t s) {
    k_scalar_op<<<1, 1, 0, s>>>(H.scal, op, nullptr);
    ++H.launches;
}

void launch_halo_pack(const Hierarchy& H, const DevLevel& L, const double* v, cudaStream_t s) {
    const int64_t tot = L.dist.send_total * H.nz;
    if (tot == 0) return;
    k_halo_pack<<<blocks(tot, 256), 256, 0, s>>>(v, L.ld, H.nz, L.dist.send_idx, L.dist.send_total, L.dist.sendbuf);
    ++H.launches;
}

void launch_halo_unpack(const Hierarchy& H, const DevLevel& L, double* v, cudaStream_t s) {
    const int64_t tot = L.dist.n_halo * H.nz;
    if (tot == 0) return;
    k_halo_unpack<<<blocks(tot, 256), 256, 0, s>>>(L.dist.recvbuf, L.dist.n_halo, H.nz, v, L.ld, L.n);
    ++H.launches;
}

void launch_gather_pack(const Hierarchy& H, const DevLevel& C, const double* v, int64_t off, int64_t cnt,
                        cudaStream_t s) {
    dim3 g(blocks(cnt, 256), H.nz);
    k_gather_pack<<<g, 256, 0, s>>>(v, C.ld, off, cnt, H.gbuf_send);
    ++H.launches;
}

void launch_gather_unpack(const Hierarchy& H, const DevLevel& C, double* v, int64_t cnt, cudaStream_t s) {
    dim3 g(blocks(cnt, 256), H.nz, H.nranks);
    k_gather_unpack<<<g, 256, 0, s>>>(H.gbuf_recv, cnt, H.nz, v, C.ld);
    ++H.launches;
}

void launch_halo_pupdate(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                         cudaStream_t s) {
    const int64_t tot = L.dist.n_halo * H.nz;
    if (tot == 0) return;
    k_halo_pupdate<<<blocks(tot, 256), 256, 0, s>>>(z, pold, pnew, L.n, L.dist.n_halo, L.ld, H.nz, H.scal);
    ++H.launches;
}

void launch_update_p(const Hierarchy& H, const DevLevel& L, double* p, const double* z, cudaStream_t s) {
    ProfScope ps(H, kKVector, L.ref, s);
    dim3 g(blocks(L.n, 256), H.nz);
    k_update_p<<<g, 256, 0, s>>>(p, z, L.n, L.ld, H.scal);
    ++H.launches;
    ++H.launches;
}

void launch_update_xr(const Hierarchy& H, const DevLevel& L, double* x, const double* p, cudaStream_t s) {
    ProfScope ps(H, kKVector, H.fine_ref, s);
    k_update_xr<false><<<vec_grid(L.n, H.nz), kVecBlock, 0, s>>>(x, H.r, p, H.q, nullptr, L.n, L.ld, H.nz, H.scal,
                                                                 H.partials, fin_take(H));
    ++H.launches;
}

// x = x + alpha p (FIRST: x = 0 + alpha p) over every padded row, grid-stride:
// the deferred CG update on the side stream, launched with few CTAs so that it
// trickles through the V-cycle's latency-bound coarse part instead of
// contending with it at full bandwidth (same values as k_update_xr's x part)
template <bool FIRST>
__global__ void __launch_bounds__(256) k_update_x_slow(double* __restrict__ x, const double* __restrict__ p,
                                                       int64_t n, int64_t ld, int nz, const PcgScalars* __restrict__ sc) {
    const double alpha = sc->alpha;
    double2* x2 = reinterpret_cast<double2*>(x);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const int64_t hn = n / 2, total = hn * nz;          // pairs of cells per layer (n is even); padding untouched
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / hn, q = k * (ld / 2) + (t - k * hn);
        double2 xx = FIRST ? make_double2(0.0, 0.0) : x2[q];
        const double2 pp = p2[q];
        xx.x = xx.x + alpha * pp.x;
        xx.y = xx.y + alpha * pp.y;
        x2[q] = xx;
    }
}

// part 1: r = r - alpha q (first: r = b - alpha q) with partial <r, r>;
// part 2: x = x + alpha p (first: x = 0 + alpha p); part 3: the same as 2 by
// k_update_x_slow with `slow_blocks` CTAs
void launch_update_part(const Hierarchy& H, const DevLevel& L, int part, bool first, double* x, const double* p,
                        const double* b, cudaStream_t s) {
    ProfScope ps(H, kKVector, H.fine_ref, s);
    const dim3 g = vec_grid(L.n, H.nz);
    if (part == 1) {
        const FinArgs f = fin_take(H);
        if (first) k_update_xr<true, 1><<<g, kVecBlock, 0, s>>>(x, H.r, p, H.q, b, L.n, L.ld, H.nz, H.scal, H.partials, f);
        else k_update_xr<false, 1><<<g, kVecBlock, 0, s>>>(x, H.r, p, H.q, b, L.n, L.ld, H.nz, H.scal, H.partials, f);
    }
    if (part == 2 && first) k_update_xr<true, 2><<<g, kVecBlock, 0, s>>>(x, H.r, p, H.q, b, L.n, L.ld, H.nz, H.scal, H.partials);
    if (part == 2 && !first) k_update_xr<false, 2><<<g, kVecBlock, 0, s>>>(x, H.r, p, H.q, b, L.n, L.ld, H.nz, H.scal, H.partials);
    if (part == 3) {
        const unsigned nb = (unsigned)(H.x_slow_blocks > 0 ? H.x_slow_blocks : 1);
        if (first) k_update_x_slow<true><<<nb, 256, 0, s>>>(x, p, L.n, L.ld, H.nz, H.scal);
        else k_update_x_slow<false><<<nb, 256, 0, s>>>(x, p, L.n, L.ld, H.nz, H.scal);
    }
    ++H.launches;
}

void launch_update_xr_first(const Hierarchy& H, const DevLevel& L, double* x, const double* p, const double* b,
                            cudaStream_t s) {
    ProfScope ps(H, kKVector, H.fine_ref, s);
    k_update_xr<true><<<vec_grid(L.n, H.nz), kVecBlock, 0, s>>>(x, H.r, p, H.q, b, L.n, L.ld, H.nz, H.scal,
                                                                H.partials, fin_take(H));
    ++H.launches;
}

void launch_copy_pad(const Hierarchy& H, const DevLevel& L, const double* src, int64_t src_ld, double* dst,
                     int64_t dst_ld, cudaStream_t s) {
    dim3 g(blocks(L.n, 256), H.nz);
    k_copy_rows<<<g, 256, 0, s>>>(src, src_ld, dst, dst_ld, L.n);
    ++H.launches;
}

}  // namespace hmg
