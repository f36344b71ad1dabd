// Line-Jacobi sweeps on small (latency-bound) levels: one warp per 32-column
// tile, the tile's whole operand set resident in shared memory.
//
// Same operation (Eq. 10 read with Eq. 13, readings R5-R7) and the same
// operation order as every other sweep kernel; bit-identical results.  What
// differs is the schedule, tuned for levels with few columns where a sweep is
// bounded by the length of each column's sequential Thomas recurrence, not by
// HBM bandwidth:
//  * prologue: 3-4 TMA tensor copies bring all layers of the tile's bands,
//    right-hand side, precomputed pivots (den, y, g) and iterate into shared
//    memory in one shot; the <= 32 off-tile neighbour cells ("halo") come with
//    8-byte cp.async, one halo cell per lane;
//  * the sweep itself (tile_sweep, small_tile.cuh) is split into passes with
//    independent work batched into registers, so the only serial chain is
//    z_k's (5 dependent fp64 ops);
//  * the coarsest level (one tile) runs all n_coarse sweeps in one launch,
//    iterating in shared memory.
#include <cuda.h>

#include <cstring>
#include <stdexcept>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"
#include "small_tile.cuh"

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);

namespace {

constexpr int kTS = kSmallTile;   // 32 columns per CTA, one warp

struct SmallMaps {
    CUtensorMap bands;  // 3-D box 32 x nz x 5 (D, U, H0, H1, H2)
    CUtensorMap fact;   // 3-D box 32 x nz x 3 (den, y, g)
    CUtensorMap b;      // 2-D box 32 x nz
    CUtensorMap u;      // 2-D box 32 x nz (incoming iterate; unused for the zero guess)
    CUtensorMap uc;     // 2-D box 8 x nz (coarse correction; PROLONG only)
};

struct SmallSmem {
    size_t bands, fact, b, u, uc, hu, huc, z, bar, total;
};

__host__ __device__ inline SmallSmem small_layout(int nz) {
    SmallSmem L;
    const size_t plane = sizeof(double) * (size_t)((nz + 7) & ~7) * kTS;   // layers padded to 8
    size_t off = 0;
    L.bands = off; off += 5 * plane;
    L.fact = off;  off += 3 * plane;
    L.b = off;     off += plane;
    L.u = off;     off += plane;
    L.uc = off;    off += plane / 4;
    L.hu = off;    off += plane;          // [nz][32] halo slots
    L.huc = off;   off += plane;
    L.z = off;     off += plane;
    L.bar = off;   off += 64;
    L.total = off;
    return L;
}

#ifdef HMG_TIMING
__device__ long long g_sm_timing[64];
#define SSTAMP(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_sm_timing[i] = clock64(); } while (0)
#else
#define SSTAMP(i) do {} while (0)
#endif

template <bool ZERO, bool PROLONG>
__global__ void __launch_bounds__(kTS, 1)
    k_sweep_small(const __grid_constant__ SmallMaps maps, LevelView L, SmallHalo sh, const double* __restrict__ bvec,
                  const double* __restrict__ uin, const double* __restrict__ uc, int64_t ldc,
                  double* __restrict__ uout, double omega, int nsweeps) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    const int nz = L.nz;
    const int64_t ld = L.ld;
    const int j = threadIdx.x;
    const int64_t c0 = (int64_t)blockIdx.x * kTS, c = c0 + j;
    const bool valid = c < L.n;
    const SmallSmem lay = small_layout(nz);
    double* sB = reinterpret_cast<double*>(smraw + lay.bands);
    double* sF = reinterpret_cast<double*>(smraw + lay.fact);
    double* sb = reinterpret_cast<double*>(smraw + lay.b);
    double* su = reinterpret_cast<double*>(smraw + lay.u);
    double* suc = reinterpret_cast<double*>(smraw + lay.uc);
    double* shu = reinterpret_cast<double*>(smraw + lay.hu);
    double* shuc = reinterpret_cast<double*>(smraw + lay.huc);
    double* sz = reinterpret_cast<double*>(smraw + lay.z);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + lay.bar);
    const int P = ((nz + 7) & ~7) * kTS;               // doubles per plane (layers padded to 8)
    const double* __restrict__ D = sB;
    const double* __restrict__ U = sB + P;
    const double* __restrict__ H0 = sB + 2 * P;
    const double* __restrict__ H1 = sB + 3 * P;
    const double* __restrict__ H2 = sB + 4 * P;
    const double* __restrict__ den = sF;
    const double* __restrict__ yv = sF + P;
    const double* __restrict__ g = sF + 2 * P;

    SSTAMP(0);
    // ---- prologue: everything of the tile into shared memory ----
    const int hcount = ZERO ? 0 : sh.count[blockIdx.x];
    const int32_t hcell = (!ZERO && j < hcount) ? sh.cells[blockIdx.x * kSmallHaloMax + j] : 0;
    if (j == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    if (j == 0) {
        const uint32_t plane_bytes = (uint32_t)(sizeof(double) * P);
        uint32_t bytes = 9 * plane_bytes;
        if (!ZERO) bytes += plane_bytes;
        if (PROLONG) bytes += plane_bytes / 4;
        ptx::mbar_arrive_expect_tx(bar, bytes);
        ptx::tma_load_3d(sB, &maps.bands, (int)c0, 0, 0, bar);
        ptx::tma_load_3d(sF, &maps.fact, (int)c0, 0, 0, bar);
        ptx::tma_load_2d(sb, &maps.b, (int)c0, 0, bar);
        if (!ZERO) ptx::tma_load_2d(su, &maps.u, (int)c0, 0, bar);
        if (PROLONG) ptx::tma_load_2d(suc, &maps.uc, (int)(c0 / 4), 0, bar);
    }
    if (!ZERO && j < hcount) {
        for (int k = 0; k < nz; ++k) {
            ptx::cp_async8(&shu[k * kTS + j], uin + (int64_t)k * ld + hcell);
            if (PROLONG) ptx::cp_async8(&shuc[k * kTS + j], uc + (int64_t)k * ldc + (hcell >> 2));
        }
    }
    uint32_t loc = 0;
    if (!ZERO || nsweeps > 1) loc = sh.loc[valid ? c : L.n - 1];
    const int l0 = loc & 0xff, l1 = (loc >> 8) & 0xff, l2 = (loc >> 16) & 0xff;
    asm volatile("cp.async.wait_all;" ::: "memory");
    ptx::mbar_wait(bar, 0);
    __syncwarp();
    if (PROLONG) {                                     // fused prolongation: u <- u + P u_c (same addition)
        for (int k = 0; k < nz; ++k) {
            su[k * kTS + j] = su[k * kTS + j] + suc[k * (kTS / 4) + (j >> 2)];
            if (j < hcount) shu[k * kTS + j] = shu[k * kTS + j] + shuc[k * kTS + j];
        }
        __syncwarp();
    }
    SSTAMP(1);
    const TileSmem S{D, U, H0, H1, H2, den, yv, g, sb, su, shu, sz};
    for (int sweep = 0; sweep < nsweeps; ++sweep)   // later sweeps of a multi-sweep launch use u
        tile_sweep(S, nz, j, l0, l1, l2, ZERO && sweep == 0, omega, valid);
    if (valid)
        for (int k = 0; k < nz; ++k) uout[(int64_t)k * ld + c] = su[k * kTS + j];
}

#ifdef HMG_TIMING
}  // namespace
extern "C" void hmg_debug_sm_timing(long long* out) { cudaMemcpyFromSymbol(out, g_sm_timing, sizeof(long long) * 64); }
namespace {
#endif

template <bool Z, bool P>
void launch_small_t(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                    double* uout, double omega, int nsweeps, cudaStream_t s) {
    const int nz = H.nz;
    const SmallSmem lay = small_layout(nz);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sweep_small<Z, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    SmallMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const LevelView V = L.view(nz);
    const int nzp = (nz + 7) & ~7;                 // box rows >= nz are zero-filled by the TMA
    maps.bands = make_tensor_map(V.D, L.ld, nz, kTS, nzp, 5);
    maps.fact = make_tensor_map(L.fden, L.ld, nz, kTS, nzp, 3);
    maps.b = make_tensor_map(b, L.ld, nz, kTS, nzp, 1);
    if (!Z) maps.u = make_tensor_map(uin, L.ld, nz, kTS, nzp, 1);
    int64_t ldc = 0;
    if (P) {
        const DevLevel& C = H.lev[L.ref - 1];
        ldc = C.ld;
        maps.uc = make_tensor_map(uc, C.ld, nz, kTS / 4, nzp, 1);
    }
    const unsigned grid = (unsigned)((L.n + kTS - 1) / kTS);
    k_sweep_small<Z, P><<<grid, kTS, lay.total, s>>>(maps, V, L.small, b, uin, uc, ldc, uout, omega, nsweeps);
}

}  // namespace

bool sweep_small_supported(const Hierarchy& H, const DevLevel& L) {
    // one 32-column tile per SM (the tile's operands fill shared memory): use it
    // while the level fits in a single wave
    return L.fden != nullptr && L.small.loc != nullptr && H.nz <= 256 && small_layout(H.nz).total <= 227 * 1024 &&
           (L.n + kTS - 1) / kTS <= 148;
}

void launch_sweep_small(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                        double* uout, double omega, int nsweeps, cudaStream_t s) {
    if (!uin)
        launch_small_t<true, false>(H, L, b, nullptr, nullptr, uout, omega, nsweeps, s);
    else if (uc)
        launch_small_t<false, true>(H, L, b, uin, uc, uout, omega, nsweeps, s);
    else
        launch_small_t<false, false>(H, L, b, uin, nullptr, uout, omega, nsweeps, s);
    ++H.launches;
}

}  // namespace hmg
