// Fused line-Jacobi sweep for sm_100a: TMA-tiled layer blocks, TMEM-resident
// Thomas state.
//
// Computes exactly what k_sweep (kernels.cu) computes -- for every column
//   r = b - H^ u,  delta = T^{-1} r (Thomas),  u' = u + omega delta
// (Eq. 10 read with Eq. 13; readings R5-R7), same operation order,
// no FMA contraction -- but is organised for HBM bandwidth:
//
//  * a CTA owns a tile of kTile = 128 consecutive columns (4 consumer warps,
//    one thread per column) plus one producer warp;
//  * the producer streams blocks of G layers x 128 cells of every array
//    (D, U, H0, H1, H2, b, and the u rows) with 2-D TMA tensor copies
//    (cp.async.bulk.tensor.2d; one instruction per array per G layers) into an
//    S-stage shared-memory ring guarded by full/empty mbarriers, and gathers
//    the tile's off-tile neighbour values ("halo", <= 64 cells, table built at
//    setup) with 8-byte cp.async into the same stage;
//  * the whole tile's u rows stay resident in shared memory, so in-tile
//    neighbour reads and the back substitution's u_old come from on-chip;
//  * the Thomas forward state (z_k, g_k: 2 doubles per layer per column) is
//    kept in tensor memory (tcgen05.st / tcgen05.ld, lane = column), which
//    leaves shared memory to the streaming ring: 2 CTAs per SM;
//  * both quotients of a layer divide by the same pivot den_k and share one
//    reciprocal (div_fast: bit-identical to '/').
// HBM traffic per dof: u, b, D, U, H0, H1, H2 read once, u' written once
// (64 B/dof); zero-guess form: b, D, U in, u' out (32 B/dof).
#include <cuda.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {
namespace {

constexpr int kTile = kSweepTile;          // columns per CTA
constexpr int kConsumerWarps = kTile / 32;
constexpr int kThreads = kTile + 32;

__device__ __forceinline__ bool pivot_ok(double den) { return den > 0.0 && den <= DBL_MAX; }

// Tensor maps of one launch: bands (per level) + vectors (per call).
// The band planes D, U, H0, H1, H2 are contiguous ([5][nz][ld]), and so are the
// precomputed factors ([3][nz][ld]): one 3-D box moves every band (or factor)
// of G layers in a single TMA instruction -- per-instruction latency, not
// bytes, limits a CTA's TMA stream, so fewer, larger copies matter.
struct SweepMaps {
    CUtensorMap bands;  // 3-D (cell, layer, band), box kTile x G x nb  (nb = 2: D, U; 5: D..H2)
    CUtensorMap b;      // right-hand side, box kTile x G
    CUtensorMap fact;   // 3-D factors den, y, g, box kTile x G x 3 (FACT only)
    CUtensorMap u;      // incoming iterate (box kTile x G)
    CUtensorMap uc;     // coarse correction (box kTile/4 x G), PROLONG only
};

struct SweepSmem {
    int S, nrows, stage_doubles, rows_pad;
    size_t off_u, off_uc, off_stage, total;
};

__host__ __device__ inline SweepSmem sweep_layout(int nz, bool zero, bool prolong, bool fact, int S, int G) {
    SweepSmem L;
    L.S = S;
    L.nrows = (zero ? 3 : 6) + (fact ? 3 : 0);
    L.rows_pad = ((nz + G - 1) / G) * G;
    L.stage_doubles = L.nrows * G * kTile + (zero ? 0 : G * kHaloMax) + (prolong ? G * kHaloMax : 0);
    size_t off = 1024;  // barriers + TMEM slot
    L.off_u = off;
    if (!zero) off += sizeof(double) * L.rows_pad * kTile;
    L.off_uc = off;
    if (prolong) off += sizeof(double) * L.rows_pad * (kTile / 4);
    L.off_stage = off;
    off += sizeof(double) * (size_t)S * L.stage_doubles;
    L.total = off;
    return L;
}

#ifdef HMG_TIMING
__device__ long long g_tc_timing[16];
#define TSTAMP(i) do { if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 128)) g_tc_timing[i] = clock64(); } while (0)
#else
#define TSTAMP(i) do {} while (0)
#endif

template <bool ZERO, bool PROLONG, bool FACT, int G, bool CHK = true>
__global__ void __launch_bounds__(kThreads, 2)
    k_sweep_tc(const __grid_constant__ SweepMaps maps, LevelView L, TileHalo th, const double* __restrict__ bvec,
               const double* __restrict__ uin, const double* __restrict__ uc, int64_t ldc,
               const double* __restrict__ fdp, const double* __restrict__ fgp, double* __restrict__ uout,
               double omega, int ref, unsigned long long* __restrict__ bad, int S, uint32_t tmem_cols,
               int pf_groups) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    const int nz = L.nz;
    const int64_t ld = L.ld;
    const int ngroups = (nz + G - 1) / G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const SweepSmem lay = sweep_layout(nz, ZERO, PROLONG, FACT, S, G);
    constexpr int kFactRow = ZERO ? 3 : 6;                            // den, y, g rows (FACT)
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
    uint64_t* empty = full + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + S);
    const int ntiles = (int)((L.n + kTile - 1) / kTile);
    double* utile = reinterpret_cast<double*>(smraw + lay.off_u);     // [rows_pad][kTile]
    double* uctile = reinterpret_cast<double*>(smraw + lay.off_uc);   // [rows_pad][kTile/4]
    double* stages = reinterpret_cast<double*>(smraw + lay.off_stage);
    const int row_block = G * kTile;                                  // doubles per array per stage

    TSTAMP(0);
    ptx::pdl_trigger();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kConsumerWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(tmem_slot, tmem_cols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    ptx::pdl_wait();
    TSTAMP(1);

    if (warp == kConsumerWarps) {
        // ======================= producer warp =======================
        // persistent: tiles blockIdx.x, blockIdx.x + gridDim.x, ...; the ring
        // runs on across tile boundaries, so the next tile's first stages
        // stream while the consumers finish the current tile
        const uint32_t ublock = (uint32_t)(sizeof(double) * G * kTile);
        const uint32_t ucblock = (uint32_t)(sizeof(double) * G * (kTile / 4));
        int s = 0;
        uint32_t phase = 0;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t c0 = (int64_t)tile * kTile;
        int hcount = 0;
        int32_t h0 = 0, h1 = 0;
        if (!ZERO) {
            hcount = th.count[tile];
            if (lane < hcount) h0 = th.cells[tile * kHaloMax + lane];
            if (lane + 32 < hcount) h1 = th.cells[tile * kHaloMax + lane + 32];
        }
        const int x = (int)c0, xc = (int)(c0 / 4);
        for (int gi = 0; gi < ngroups; ++gi, (++s == S ? (s = 0, phase ^= 1u) : 0)) {
            ptx::mbar_wait(&empty[s], phase ^ 1u);
            double* st = stages + (size_t)s * lay.stage_doubles;
            if (!ZERO) {
                double* hu = st + lay.nrows * row_block;
                for (int kk = 0; kk < G; ++kk) {
                    const int k = gi * G + kk;
                    if (k >= nz) break;
                    const double* src = uin + (int64_t)k * ld;
                    if (lane < hcount) ptx::cp_async8(&hu[kk * kHaloMax + lane], src + h0);
                    if (lane + 32 < hcount) ptx::cp_async8(&hu[kk * kHaloMax + lane + 32], src + h1);
                    if (PROLONG) {
                        double* huc = hu + G * kHaloMax;
                        const double* srcc = uc + (int64_t)k * ldc;
                        if (lane < hcount) ptx::cp_async8(&huc[kk * kHaloMax + lane], srcc + (h0 >> 2));
                        if (lane + 32 < hcount) ptx::cp_async8(&huc[kk * kHaloMax + lane + 32], srcc + (h1 >> 2));
                    }
                }
                ptx::cp_async_arrive(&full[s]);
            }
            __syncwarp();
            if (lane == 0 && pf_groups > 0) {
                // L2 prefetch pf_groups stages ahead: the ring's copies then see
                // L2 instead of HBM latency (smem caps the ring's depth)
                const int gp = gi + pf_groups;
                if (gp < ngroups) {
                    constexpr int nbp = ZERO ? 2 : 5;
                    (void)nbp;
                    ptx::tma_prefetch_3d(&maps.bands, x, gp * G, 0);
                    ptx::tma_prefetch_2d(&maps.b, x, gp * G);
                    if (!ZERO) ptx::tma_prefetch_2d(&maps.u, x, (gp + 1) * G);
                    if (FACT) ptx::tma_prefetch_3d(&maps.fact, x, gp * G, 0);
                }
            }
            if (lane == 0) {
                uint32_t bytes = (uint32_t)lay.nrows * ublock;   // bands + b (+ factors)
                const bool u0 = !ZERO && gi == 0;
                const bool unext = !ZERO && gi + 1 < ngroups;
                if (u0) bytes += ublock + (PROLONG ? ucblock : 0);
                if (unext) bytes += ublock + (PROLONG ? ucblock : 0);
                ptx::mbar_arrive_expect_tx(&full[s], bytes);
                constexpr int nb = ZERO ? 2 : 5;
                ptx::tma_load_3d(st, &maps.bands, x, gi * G, 0, &full[s]);
                ptx::tma_load_2d(st + nb * row_block, &maps.b, x, gi * G, &full[s]);
                if (FACT) ptx::tma_load_3d(st + (nb + 1) * row_block, &maps.fact, x, gi * G, 0, &full[s]);
                (void)it;   // only the zero-guess form (no u tile) runs persistent, see launch_tc
                if (u0) {
                    ptx::tma_load_2d(utile, &maps.u, x, 0, &full[s]);
                    if (PROLONG) ptx::tma_load_2d(uctile, &maps.uc, xc, 0, &full[s]);
                }
                if (unext) {
                    const int y = (gi + 1) * G;
                    ptx::tma_load_2d(utile + (size_t)y * kTile, &maps.u, x, y, &full[s]);
                    if (PROLONG) ptx::tma_load_2d(uctile + (size_t)y * (kTile / 4), &maps.uc, xc, y, &full[s]);
                }
            }
        }
        }
    } else {
        // ======================= consumer warps: one column per thread =======================
        const int j = threadIdx.x;
        int s = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = (int64_t)tile * kTile;
        const int64_t c = c0 + j;
        const bool valid = c < L.n;
        uint32_t loc = 0;
        if (!ZERO) loc = th.loc[valid ? c : L.n - 1];
        const int l0 = loc & 0xff, l1 = (loc >> 8) & 0xff, l2 = (loc >> 16) & 0xff;
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        const uint32_t gcol = 2u * (uint32_t)nz;   // g_k at columns 2nz + 2k, z_k at 2k

        // u value (with the fused prolongation) of in-tile local cell l at layer kk
        auto UV = [&](int kk, int l) -> double {
            double v = utile[(size_t)kk * kTile + l];
            if (PROLONG) v = v + uctile[(size_t)kk * (kTile / 4) + (l >> 2)];
            return v;
        };
        auto NBR = [&](int kk, int l, const double* hu) -> double {
            if (l < kTile) return UV(kk, l);
            double v = hu[l - kTile];
            if (PROLONG) v = v + hu[G * kHaloMax + l - kTile];
            return v;
        };

        // Thomas forward elimination, reading R6 order: den_0 = D_0; for k >= 1
        // den_k = D_k - U_{k-1} g_{k-1}; z_k = (r_k - U_{k-1} z_{k-1}) / den_k;
        // g_k = U_k / den_k.  One layer of it, from already-loaded operands;
        // EXACT selects the '/' operator, otherwise the shared-reciprocal
        // division whose rare invalid cases are flagged in `slow` (the whole
        // column is then redone exactly, below, so the hot loop has no branch).
        double um = 0.0, uk = 0.0, Um = 0.0, gprev = 0.0, zprev = 0.0;
        bool ok = true, slow = false;
        auto layer = [&](int k, double Dk, double Uk, double r, double fden, double fy, double fg, bool exact) {
            const double num = (k == 0) ? r : r - Um * zprev;
            const bool has_g = k < nz - 1;
            double den, z, g = 0.0;
            if (FACT) {                           // pivots precomputed at setup (matrix-only)
                den = fden;
                g = fg;
                z = exact ? num / den : div_fast_z(num, den, fy, slow);
            } else {
                den = (k == 0) ? Dk : Dk - Um * gprev;
                if (exact) {
                    z = num / den;
                    if (has_g) g = Uk / den;
                } else {
                    const double y = div_recip(den);
                    z = div_fast_z(num, den, y, slow);
                    if (has_g) g = div_fast(Uk, den, y, slow);
                }
                ok = ok && pivot_ok(den);
            }
            ptx::tmem_st_f64(tl + 2u * (uint32_t)k, z);
            if (has_g) ptx::tmem_st_f64(tl + gcol + 2u * (uint32_t)k, g);
            zprev = z;
            gprev = g;
        };
#ifdef HMG_TIMING
        long long wait_acc = 0;
#endif
        for (int gi = 0; gi < ngroups; ++gi, (++s == S ? (s = 0, phase ^= 1u) : 0)) {
#ifdef HMG_TIMING
            long long tw0 = clock64();
#endif
            ptx::mbar_wait(&full[s], phase);
#ifdef HMG_TIMING
            wait_acc += clock64() - tw0;
#endif
            if (gi == 0) TSTAMP(2);
            const double* st = stages + (size_t)s * lay.stage_doubles;
            if (ZERO && !FACT && gi > 0 && (gi + 1) * G < nz) {
                // interior stage of the zero-guess form: 0 < k < nz - 1 for every
                // layer, so the Thomas step runs without boundary tests
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const int k = gi * G + kk;
                    const double* sr = st + kk * kTile + j;
                    const double Dk = sr[0];
                    const double Uk = sr[row_block];
                    const double num = sr[2 * row_block] - Um * zprev;
                    const double den = Dk - Um * gprev;
                    const double y = div_recip(den);
                    const double z = div_fast_z(num, den, y, slow);
                    // CHK = false: pivots and every g_k's fast path verified at build (k_pivot_check)
                    const double g = CHK ? div_fast(Uk, den, y, slow) : div_fast_unchecked(Uk, den, y);
                    if (CHK) ok = ok && pivot_ok(den);
                    ptx::tmem_st_f64(tl + 2u * (uint32_t)k, z);
                    ptx::tmem_st_f64(tl + gcol + 2u * (uint32_t)k, g);
                    zprev = z;
                    gprev = g;
                    Um = Uk;
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
                continue;
            }
#pragma unroll
            for (int kk = 0; kk < G; ++kk) {
                const int k = gi * G + kk;
                if (k >= nz) break;
                const double* sr = st + kk * kTile + j;
                const double Dk = sr[0];
                const double Uk = sr[row_block];
                double r;
                double up = 0.0;
                if (ZERO) {
                    r = sr[2 * row_block];
                } else {
                    const double* hu = st + lay.nrows * row_block + kk * kHaloMax;
                    if (k == 0) uk = UV(0, j);
                    if (k < nz - 1) up = UV(k + 1, j);
                    double acc = Dk * uk;
                    if (k > 0) acc = acc + Um * um;
                    if (k < nz - 1) acc = acc + Uk * up;
                    acc = acc + sr[2 * row_block] * NBR(k, l0, hu);
                    acc = acc + sr[3 * row_block] * NBR(k, l1, hu);
                    acc = acc + sr[4 * row_block] * NBR(k, l2, hu);
                    r = sr[5 * row_block] - acc;
                }
                double fden = 0.0, fy = 0.0, fg = 0.0;
                if (FACT) {
                    fden = sr[kFactRow * row_block];
                    fy = sr[(kFactRow + 1) * row_block];
                    fg = sr[(kFactRow + 2) * row_block];
                }
                layer(k, Dk, Uk, r, fden, fy, fg, false);
                um = uk;
                uk = up;
                Um = Uk;
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
        }
        TSTAMP(3);
#ifdef HMG_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 0) g_tc_timing[8] = wait_acc;
#endif
        // Rare: a quotient left the fast path's exact range (e.g. a zero
        // numerator).  The warp recomputes its columns' forward pass from
        // global memory with the '/' operator (TMEM stores are warp-wide).
        if (__any_sync(0xffffffffu, slow && valid)) {
            const int64_t ce = valid ? c : L.n - 1;
            const int32_t g0 = ZERO ? 0 : L.nbr[ce], g1 = ZERO ? 0 : L.nbr[ld + ce], g2 = ZERO ? 0 : L.nbr[2 * ld + ce];
            auto GU = [&](int kk, int64_t cell) -> double {
                double v = uin[(int64_t)kk * ld + cell];
                if (PROLONG) v = v + uc[(int64_t)kk * ldc + (cell >> 2)];
                return v;
            };
            um = uk = Um = gprev = zprev = 0.0;
            if (!ZERO) uk = GU(0, ce);
            for (int k = 0; k < nz; ++k) {
                const int64_t i = (int64_t)k * ld + ce;
                const double Dk = L.D[i], Uk = L.U[i];
                double r, up = 0.0;
                if (ZERO) {
                    r = bvec[i];
                } else {
                    if (k < nz - 1) up = GU(k + 1, ce);
                    double acc = Dk * uk;
                    if (k > 0) acc = acc + Um * um;
                    if (k < nz - 1) acc = acc + Uk * up;
                    acc = acc + L.H0[i] * GU(k, g0);
                    acc = acc + L.H1[i] * GU(k, g1);
                    acc = acc + L.H2[i] * GU(k, g2);
                    r = bvec[i] - acc;
                }
                layer(k, Dk, Uk, r, FACT ? fdp[i] : 0.0, 0.0, FACT ? fgp[i] : 0.0, true);
                um = uk;
                uk = up;
                Um = Uk;
            }
        }
        if (valid && !ok) atomicMin(bad, ((unsigned long long)ref << 40) | (unsigned long long)c);
        ptx::tmem_wait_st();
        TSTAMP(4);

        // back substitution from the top layer, 8 layers of (z, g) per TMEM load
        double dl = 0.0;
        int k = nz - 1;
        while (k >= 0) {
            const int k0 = (k >= 7) ? k - 7 : 0;
            if (k - k0 == 7) {
                uint32_t zr[16], gr[16];
                ptx::tmem_ld_8f64(tl + 2u * (uint32_t)k0, zr);
                ptx::tmem_ld_8f64(tl + gcol + 2u * (uint32_t)k0, gr);
                ptx::tmem_wait_ld();
                if (k0 + 7 < nz - 1) {                  // below the top layer: no boundary test
#pragma unroll
                    for (int i = 7; i >= 0; --i) {
                        const int kk = k0 + i;
                        dl = ptx::f64_from(zr[2 * i], zr[2 * i + 1]) - ptx::f64_from(gr[2 * i], gr[2 * i + 1]) * dl;
                        const double o = ZERO ? omega * dl : UV(kk, j) + omega * dl;
                        if (valid) uout[(int64_t)kk * ld + c] = o;
                    }
                } else {
#pragma unroll
                    for (int i = 7; i >= 0; --i) {
                        const int kk = k0 + i;
                        const double zk = ptx::f64_from(zr[2 * i], zr[2 * i + 1]);
                        if (kk == nz - 1)
                            dl = zk;
                        else
                            dl = zk - ptx::f64_from(gr[2 * i], gr[2 * i + 1]) * dl;
                        const double o = ZERO ? omega * dl : UV(kk, j) + omega * dl;
                        if (valid) uout[(int64_t)kk * ld + c] = o;
                    }
                }
            } else {
                for (int kk = k; kk >= k0; --kk) {
                    uint32_t zr[2], gr[2];
                    ptx::tmem_ld_1f64(tl + 2u * (uint32_t)kk, zr);
                    ptx::tmem_ld_1f64(tl + gcol + 2u * (uint32_t)kk, gr);
                    ptx::tmem_wait_ld();
                    const double zk = ptx::f64_from(zr[0], zr[1]);
                    if (kk == nz - 1)
                        dl = zk;
                    else
                        dl = zk - ptx::f64_from(gr[0], gr[1]) * dl;
                    const double o = ZERO ? omega * dl : UV(kk, j) + omega * dl;
                    if (valid) uout[(int64_t)kk * ld + c] = o;
                }
            }
            k = k0 - 1;
        }
        }
    }
    TSTAMP(5);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, tmem_cols);
    TSTAMP(6);
}

__global__ void k_selftest_div(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ fast, double* __restrict__ ref) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool slow = false;
    const double y = div_recip(b[i]);
    double q = div_fast(a[i], b[i], y, slow);
    if (slow) q = a[i] / b[i];
    fast[i] = q;
    ref[i] = a[i] / b[i];
}

// ---- host: tensor-map encoding through the driver entry point ---------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// Map over `planes` consecutive layer-major [rows][ld] fp64 arrays (planes = 1:
// 2-D, else 3-D with plane stride rows*ld); box = box_x cells x G layers x planes.
// Out-of-range box elements (tail tile, layers >= rows) are zero-filled.
CUtensorMap encode_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes, int64_t width) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[3] = {(cuuint64_t)(width > 0 ? width : ld), (cuuint64_t)rows, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)(ld * sizeof(double)), (cuuint64_t)(rows * ld * sizeof(double))};
    const cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)G, (cuuint32_t)planes};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, planes == 1 ? 2 : 3, const_cast<double*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
    return m;
}

// Encoding a tensor map costs host microseconds; the V-cycle and PCG reuse the
// same few buffers every call, so maps are cached by (base, ld, rows, box).
struct MapKey {
    const double* base;
    int64_t ld, rows;
    int box_x, G, planes;
    int64_t width;
    bool operator==(const MapKey& o) const {
        return base == o.base && ld == o.ld && rows == o.rows && box_x == o.box_x && G == o.G && planes == o.planes &&
               width == o.width;
    }
};
// width > 0: the map's row extent (columns past it are neither read nor
// written), else the row stride ld
CUtensorMap make_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes = 1,
                     int64_t width = 0) {
    constexpr int kCache = 128;
    static thread_local MapKey keys[kCache];
    static thread_local CUtensorMap maps[kCache];
    static thread_local int used = 0, next = 0;
    const MapKey k{base, ld, rows, box_x, G, planes, width};
    for (int i = 0; i < used; ++i)
        if (keys[i] == k) return maps[i];
    const int slot = used < kCache ? used++ : (next++ % kCache);
    keys[slot] = k;
    maps[slot] = encode_map(base, ld, rows, box_x, G, planes, width);
    return maps[slot];
}

uint32_t tmem_cols_for(int nz) {
    uint32_t need = 4u * (uint32_t)nz, c = 32;
    while (c < need) c <<= 1;
    return c;
}

template <bool Z, bool P, bool F, int G, bool CK = true>
void launch_tc(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
               double* uout, double omega, cudaStream_t s) {
    const int nz = H.nz;
    const uint32_t cols = tmem_cols_for(nz);
    // Budget: 2 CTAs per SM when the tile's TMEM share allows it (<= 256 columns).
    const unsigned grid = (unsigned)((L.n + kTile - 1) / kTile);
    // 2 CTAs per SM when the tile's TMEM share allows it (<= 256 columns) and
    // the grid fills the GPU; small (coarse) grids get one CTA per SM and a
    // deeper ring instead (they are latency-bound).
    const size_t budget = (cols <= 256 && grid > 148) ? 110 * 1024 : 220 * 1024;
    SweepSmem lay = sweep_layout(nz, Z, P, F, 2, G);
    const size_t per_stage = sizeof(double) * lay.stage_doubles;
    int S = (int)((budget - lay.off_stage) / per_stage);
    S = S < 2 ? 2 : (S > 32 ? 32 : S);
    lay = sweep_layout(nz, Z, P, F, S, G);
    size_t smem = lay.total;
    // never let a third CTA onto an SM (its TMEM allocation would have to wait)
    const size_t floor_smem = (cols <= 256 && grid > 148) ? 80 * 1024 : 120 * 1024;
    if (smem < floor_smem) smem = floor_smem;
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_sweep_tc<Z, P, F, G, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_done = true;
    }
    SweepMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const LevelView V = L.view(nz);
    maps.bands = make_map(V.D, L.ld, nz, kTile, G, Z ? 2 : 5);
    maps.b = make_map(b, L.ld, nz, kTile, G);
    if (F) maps.fact = make_map(L.fden, L.ld, nz, kTile, G, 3);
    if (!Z) maps.u = make_map(uin, L.ld, nz, kTile, G);
    int64_t ldc = 0;
    if (P) {
        const DevLevel& C = H.lev[L.ref - 1];
        ldc = C.ld;
        maps.uc = make_map(uc, C.ld, nz, kTile / 4, G);
    }
    // The zero-guess form (no resident u tile) runs persistent CTAs, two per SM,
    // each looping over tiles: the producer streams the next tile's first
    // stages while the consumers finish the current tile's back substitution.
    // The other forms keep one tile per CTA (their u tile rows would have to
    // be released before the next tile's could land; measured slower).
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
    unsigned cap = Z ? (unsigned)((cols <= 256 && grid > (unsigned)sms) ? 2 * sms : sms) : grid;
    launch_pdl(H, k_sweep_tc<Z, P, F, G, CK>, dim3(grid < cap ? grid : cap), dim3(kThreads), smem, s, maps, V, L.halo, b,
               uin, uc, ldc, L.fden, L.fg, uout, omega, L.ref, &H.scal->bad, S, cols, H.l2_prefetch_groups);
}

}  // namespace

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes) {
    return make_map(base, ld, rows, box_x, G, planes);
}
CUtensorMap make_store_map(double* base, int64_t ld, int64_t width, int64_t rows, int box_x, int G) {
    return make_map(base, ld, rows, box_x, G, 1, width);
}

#ifdef HMG_TIMING
extern "C" void hmg_debug_tc_timing(long long* out) { cudaMemcpyFromSymbol(out, g_tc_timing, sizeof(long long) * 16); }
#endif

void launch_selftest_div(int64_t n, const double* a, const double* b, double* fast, double* ref, cudaStream_t s) {
    k_selftest_div<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, a, b, fast, ref);
}

bool sweep_tc_supported(const Hierarchy& H, const DevLevel& L) {
    return H.nz <= 128 && L.halo.loc != nullptr;
}

thread_local std::string g_launch_error;

const char* take_launch_error() {
    static thread_local std::string last;
    last.swap(g_launch_error);
    g_launch_error.clear();
    return last.empty() ? nullptr : last.c_str();
}

bool tensor_maps_available() {
    try {
        encode_fn();
        return true;
    } catch (const std::exception&) {
        return false;
    }
}

void launch_sweep_tc(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                     double* uout, double omega, cudaStream_t s) {
    try {
        const bool fact = L.fden != nullptr;   // small (latency-bound) levels carry precomputed pivots
        if (fact) {
            if (!uin)
                launch_tc<true, false, true, 4>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_tc<false, true, true, 2>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_tc<false, false, true, 2>(H, L, b, uin, nullptr, uout, omega, s);
        } else {
            if (!uin && L.g_safe)
                launch_tc<true, false, false, 4, false>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (!uin)
                launch_tc<true, false, false, 4>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_tc<false, true, false, 2>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_tc<false, false, false, 2>(H, L, b, uin, nullptr, uout, omega, s);
        }
    } catch (const std::exception& e) {
        g_launch_error = std::string("sweep launch: ") + e.what();
    }
    ++H.launches;
}

}  // namespace hmg
