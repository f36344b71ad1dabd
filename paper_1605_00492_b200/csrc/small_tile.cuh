// One damped line-Jacobi sweep on a TW-column tile (TW = 32, or 16 / 8 for
// deep columns) whose whole operand set is resident in shared memory (lane =
// column; lanes >= TW idle).  Shared by the
// small-level sweep kernel (sweep_small.cu) and the cooperative coarse tail
// (coarse_coop.cu).
//
// Same operation (Eq. 10 read with Eq. 13, readings R5-R7) and the same
// operation order as every other sweep; bit-identical results.  The sweep is
// split into passes with independent work batched into registers: all
// residuals (independent per layer), then the z recurrence (the only serial
// chain: 5 dependent fp64 ops per layer), then back substitution.  All passes
// run over nzp = nz rounded up to 8 layers with no per-layer branches; rows
// >= nz hold zeros and their results never reach a layer < nz (their 'slow'
// flags are masked, and back substitution restarts at nz - 1).
#pragma once
#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {

constexpr int kTileW = kSmallTile;   // widest tile: 32 columns, one warp
constexpr int kHaloW = kSmallHaloMax;  // width of the halo plane (<= 32 off-tile neighbours per tile)

#ifdef HMG_TIMING
__device__ unsigned long long g_tile_slow_count;   // diagnostics: exact-division redos
__device__ unsigned long long g_tile_phase[5];     // CTA 0 thread 0: residual pass, forward, backward cycles; calls; forward waits
#define TSTAMP(v) long long v = clock64()
#define TACC(i, a, b) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tile_phase[i] += (unsigned long long)((b) - (a)); } while (0)
#else
#define TSTAMP(v) do {} while (0)
#define TACC(i, a, b) do {} while (0)
#endif

// Shared-memory planes of one tile, each [nzp][TW] (nzp = nz rounded up to 8);
// the halo plane is [nzp][kHaloW].
struct TileSmem {
    const double* D;
    const double* U;
    const double* H0;
    const double* H1;
    const double* H2;
    const double* den;   // Thomas pivots den_k (precomputed at setup, same formulas)
    const double* y;     // refined reciprocals of den_k
    const double* g;     // multipliers g_k = U_k / den_k
    const double* b;     // right-hand side
    double* u;           // iterate: in on entry, out on exit
    const double* hu;    // off-tile neighbour values [nz][kHaloW] (halo slot h at column h)
    double* z;           // scratch
};

// neighbour value of local slot l at layer k (in-tile slot < TW, else halo)
template <int TW>
__device__ __forceinline__ double tile_nb(const TileSmem& S, int k, int l) {
    return l < TW ? S.u[k * TW + l] : S.hu[k * kHaloW + (l - TW)];
}

// pass 1: r_k = b_k - (H^ u)_k for every layer into S.z (zero guess: r = b)
template <int TW = kTileW>
__device__ __forceinline__ void tile_residuals(const TileSmem& S, int nz, int j, int l0, int l1, int l2, bool zero) {
    const int nzp = (nz + 7) & ~7;
    if (zero) {
        for (int k0 = 0; k0 < nzp; k0 += 8) {
            double r[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = S.b[(k0 + i) * TW + j];
#pragma unroll
            for (int i = 0; i < 8; ++i) S.z[(k0 + i) * TW + j] = r[i];
        }
        return;
    }
    for (int k0 = 0; k0 < nzp; k0 += 8) {
        double r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + i;
            const int q = k * TW + j;
            const int qm = k > 0 ? q - TW : q;          // in-range address; term skipped at k = 0
            const int qp = k < nzp - 1 ? q + TW : q;
            double acc = S.D[q] * S.u[q];
            const double lo = S.U[qm] * S.u[qm];
            const double hi = S.U[q] * S.u[qp];
            acc = (k > 0) ? acc + lo : acc;
            acc = (k < nz - 1) ? acc + hi : acc;
            acc = acc + S.H0[q] * tile_nb<TW>(S, k, l0);
            acc = acc + S.H1[q] * tile_nb<TW>(S, k, l1);
            acc = acc + S.H2[q] * tile_nb<TW>(S, k, l2);
            r[i] = S.b[q] - acc;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) S.z[(k0 + i) * TW + j] = r[i];
    }
}

// One sweep: S.u <- S.u + omega T^{-1}(b - H^ S.u)   (zero: S.u <- omega T^{-1} b).
// Warp-synchronous; every lane of the warp must call it.
template <int TW = kTileW>
__device__ __forceinline__ void tile_sweep(const TileSmem& S, int nz, int j, int l0, int l1, int l2, bool zero,
                                           double omega, bool valid) {
    const int nzp = (nz + 7) & ~7;
    tile_residuals<TW>(S, nz, j, l0, l1, l2, zero);
    // pass 2: z_k = (r_k - U_{k-1} z_{k-1}) / den_k, operands of 8 layers per batch
    bool slow = false;
    double zprev = 0.0;
    for (int k0 = 0; k0 < nzp; k0 += 8) {
        double rr[8], um[8], dd[8], yy[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + i;
            const int q = k * TW + j;
            rr[i] = S.z[q];
            um[i] = S.U[k > 0 ? q - TW : q];
            dd[i] = S.den[q];
            yy[i] = S.y[q];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + i;
            const double num = (k == 0) ? rr[i] : rr[i] - um[i] * zprev;
            bool sl = false;
            const double zk = div_fast_z(num, dd[i], yy[i], sl);
            slow = slow || (sl && k < nz);
            rr[i] = zk;
            zprev = zk;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) S.z[(k0 + i) * TW + j] = rr[i];
    }
    if (__any_sync(0xffffffffu, slow && valid)) {  // rare: recompute with '/' (bitwise the same as the oracle)
#ifdef HMG_TIMING
        if (j == 0) atomicAdd(&g_tile_slow_count, 1ull);
#endif
        __syncwarp();
        tile_residuals<TW>(S, nz, j, l0, l1, l2, zero);
        zprev = 0.0;
        for (int k = 0; k < nz; ++k) {
            const int q = k * TW + j;
            const double num = (k == 0) ? S.z[q] : S.z[q] - S.U[q - TW] * zprev;
            const double zk = num / S.den[q];
            S.z[q] = zk;
            zprev = zk;
        }
    }
    __syncwarp();                                   // every lane's residual pass has read S.u
    // pass 3: back substitution, u' = u + omega delta, into S.u
    double dl = 0.0;
    for (int k1 = nzp - 1; k1 >= 0; k1 -= 8) {
        double zz[8], gg[8], uo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int q = (k1 - i) * TW + j;
            zz[i] = S.z[q];
            gg[i] = S.g[q];
            uo[i] = S.u[q];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k1 - i;
            dl = (k >= nz - 1) ? zz[i] : zz[i] - gg[i] * dl;
            uo[i] = zero ? omega * dl : uo[i] + omega * dl;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) S.u[(k1 - i) * TW + j] = uo[i];
    }
    __syncwarp();
}

// Back substitution of one 8-layer batch (top layer k1): delta_k = z_k - g_k
// delta_{k+1} (delta_{nz-1} = z_{nz-1}; TOP: the batch holding nz - 1 and the
// padding rows, the only one that needs the select), u' = u + omega delta.
template <int TW, bool TOP>
__device__ __forceinline__ void tile_back_batch(const TileSmem& S, int nz, int j, int k1, bool zero, double omega,
                                                double& dl) {
    double zz[8], gg[8], uo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int q = (k1 - i) * TW + j;
        zz[i] = S.z[q];
        gg[i] = S.g[q];
        uo[i] = S.u[q];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = k1 - i;
        if (TOP)
            dl = (k >= nz - 1) ? zz[i] : zz[i] - gg[i] * dl;
        else
            dl = zz[i] - gg[i] * dl;
        uo[i] = zero ? omega * dl : uo[i] + omega * dl;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) S.u[(k1 - i) * TW + j] = uo[i];
}

// The same sweep for a CTA of kTileWarps warps on one tile: the residual pass
// (independent per layer; issue-bound for a single warp) is split over the
// warps by 8-layer batches, then warp 0 alone runs the serial z recurrence and
// back substitution (latency-bound: more warps cannot shorten a column's
// chain).  Every thread of the CTA must call it; `lane` is the column.
constexpr int kTileWarps = 4;
template <int TW = kTileW>
__device__ __forceinline__ void tile_residuals_cta(const TileSmem& S, int nz, int warp, int j, int l0, int l1, int l2,
                                                   bool zero) {
    const int nzp = (nz + 7) & ~7;
    for (int k0 = 8 * warp; k0 < nzp; k0 += 8 * kTileWarps) {
        double r[8];
        if (zero) {
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = S.b[(k0 + i) * TW + j];
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = k0 + i;
                const int q = k * TW + j;
                const int qm = k > 0 ? q - TW : q;          // in-range address; term skipped at k = 0
                const int qp = k < nzp - 1 ? q + TW : q;
                double acc = S.D[q] * S.u[q];
                const double lo = S.U[qm] * S.u[qm];
                const double hi = S.U[q] * S.u[qp];
                acc = (k > 0) ? acc + lo : acc;
                acc = (k < nz - 1) ? acc + hi : acc;
                acc = acc + S.H0[q] * tile_nb<TW>(S, k, l0);
                acc = acc + S.H1[q] * tile_nb<TW>(S, k, l1);
                acc = acc + S.H2[q] * tile_nb<TW>(S, k, l2);
                r[i] = S.b[q] - acc;
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) S.z[(k0 + i) * TW + j] = r[i];
    }
}

// NB residual rows k0 .. k0 + NB - 1 into S.z (as tile_residuals_cta's batches)
template <int TW, int NB>
__device__ __forceinline__ void tile_residual_rows(const TileSmem& S, int nz, int nzp, int j, int k0, int l0, int l1,
                                                   int l2, bool zero) {
    double r[NB];
    if (zero) {
#pragma unroll
        for (int i = 0; i < NB; ++i) r[i] = S.b[(k0 + i) * TW + j];
    } else {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int k = k0 + i;
            const int q = k * TW + j;
            const int qm = k > 0 ? q - TW : q;          // in-range address; term skipped at k = 0
            const int qp = k < nzp - 1 ? q + TW : q;
            double acc = S.D[q] * S.u[q];
            const double lo = S.U[qm] * S.u[qm];
            const double hi = S.U[q] * S.u[qp];
            acc = (k > 0) ? acc + lo : acc;
            acc = (k < nz - 1) ? acc + hi : acc;
            acc = acc + S.H0[q] * tile_nb<TW>(S, k, l0);
            acc = acc + S.H1[q] * tile_nb<TW>(S, k, l1);
            acc = acc + S.H2[q] * tile_nb<TW>(S, k, l2);
            r[i] = S.b[q] - acc;
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) S.z[(k0 + i) * TW + j] = r[i];
}

// Named barriers 1 .. 15 hand residual batch b (8 layers) from the warp that
// formed it to the chain warp: the overlapped form below serves nzp <= 128.
constexpr int kOverlapMaxLayers = 128;
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int TW = kTileW>
__device__ __forceinline__ void tile_sweep_cta(const TileSmem& S, int nz, int warp, int j, int l0, int l1, int l2,
                                               bool zero, double omega, bool valid) {
    const int nzp = (nz + 7) & ~7;
    const int nb = nzp / 8;
    // The residual rows are independent per layer, the z recurrence is serial:
    // with nzp <= 128 the rows are formed WHILE warp 0 runs the recurrence --
    // batch 0 by all four warps (two layers each), batches 1 .. nb-1 by warps
    // 1-3 in turn, each released to warp 0 by its own named barrier.
    const bool overlap = nzp <= kOverlapMaxLayers && kTileWarps == 4;
    TSTAMP(p0);
    if (overlap) {
        tile_residual_rows<TW, 2>(S, nz, nzp, j, 2 * warp, l0, l1, l2, zero);
        __syncthreads();
        if (warp > 0)
            for (int bt = warp; bt < nb; bt += kTileWarps - 1) {
                tile_residual_rows<TW, 8>(S, nz, nzp, j, 8 * bt, l0, l1, l2, zero);
                named_arrive(bt, 64);
            }
    } else {
        tile_residuals_cta<TW>(S, nz, warp, j, l0, l1, l2, zero);
        __syncthreads();
    }
    TSTAMP(p1);
    TACC(0, p0, p1);
    if (warp == 0) {
        bool slow = false;
        double zprev = 0.0;
        for (int k0 = 0; k0 < nzp; k0 += 8) {
            if (overlap && k0 > 0) named_sync(k0 / 8, 64);   // residual batch k0 / 8 is formed
            double rr[8], um[8], dd[8], yy[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = k0 + i;
                const int q = k * TW + j;
                rr[i] = S.z[q];
                um[i] = S.U[k > 0 ? q - TW : q];
                dd[i] = S.den[q];
                yy[i] = S.y[q];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = k0 + i;
                const double num = (k == 0) ? rr[i] : rr[i] - um[i] * zprev;
                bool sl = false;
                const double zk = div_fast_z(num, dd[i], yy[i], sl);
                slow = slow || (sl && k < nz);
                rr[i] = zk;
                zprev = zk;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) S.z[(k0 + i) * TW + j] = rr[i];
        }
        TSTAMP(p2);
        TACC(1, p1, p2);
        if (__any_sync(0xffffffffu, slow && valid)) {  // rare: recompute with '/' (bitwise the same as the oracle)
#ifdef HMG_TIMING
            if (j == 0) atomicAdd(&g_tile_slow_count, 1ull);
#endif
            __syncwarp();
            tile_residuals<TW>(S, nz, j, l0, l1, l2, zero);
            zprev = 0.0;
            for (int k = 0; k < nz; ++k) {
                const int q = k * TW + j;
                const double num = (k == 0) ? S.z[q] : S.z[q] - S.U[q - TW] * zprev;
                const double zk = num / S.den[q];
                S.z[q] = zk;
                zprev = zk;
            }
        }
        __syncwarp();
        // back substitution: only the top batch (layer nz - 1 and the padding
        // rows) needs the select; below it the chain is select-free (the select
        // costs the single chain warp ~12 cycles per layer, tools/micro/chain4.cu)
        double dl = 0.0;
        tile_back_batch<TW, true>(S, nz, j, nzp - 1, zero, omega, dl);
        for (int k1 = nzp - 9; k1 >= 0; k1 -= 8) tile_back_batch<TW, false>(S, nz, j, k1, zero, omega, dl);
        TSTAMP(p3);
        TACC(2, p2, p3);
        if (blockIdx.x == 0 && threadIdx.x == 0) TACC(3, 0, 1);
    }
    __syncthreads();
}

}  // namespace hmg
