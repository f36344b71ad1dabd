// Operator apply y = H^ x (reading R5) streamed through a TMA ring:
// persistent CTAs, 128-column tiles, one producer warp, four consumer warps.
//
// Same operation order as k_apply_t (kernels.cu), so bitwise the same result:
//   y = ((((D x_k + U_{k-1} x_{k-1}) + U_k x_{k+1}) + H0 x_N0) + H1 x_N1) + H2 x_N2.
// What differs is the data movement.  The thread-per-column k_apply_t keeps
// only a few layers' loads in flight per thread and gathers the face
// neighbours from L2 (ncu: ~50 cycles per issued instruction, long-scoreboard
// bound, 0.64-0.71 of the HBM peak).  Here a producer warp streams, per stage
// of G layers, one 3-D TMA box with the five bands, G + 1 rows of x (row k + 1
// of the own column is needed at layer k) and the tile's <= 64 off-tile
// neighbours (8-byte cp.async); in-tile neighbours come from shared memory.
//  * PUPD (CG): the operand is p = z + beta p_old formed on the fly for the
//    cell and its neighbours (the same addition as a separate update) and
//    written back -- the p update fused into q = H^ p; rows of both z and
//    p_old travel in the stage.
//  * DOT: <x, H^ x> accumulated per thread, reduced per CTA in a fixed order.
//  * D is not streamed (except with the p update): the consumers re-form D_k
//    from the column's prism volume and the streamed couplings in
//    k_assemble's order (bitwise the stored diagonal), so a stage carries the
//    U, H0, H1, H2 rows only.  The p-update variant streams D: re-forming it
//    there measured slower (C2b 223 -> 266 us).
// HBM traffic per dof: 48 B (x, U, H0-H2 in; y out), 72 B with the p update;
// with the edge store 36 / 60 B.
#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);
extern thread_local std::string g_launch_error;
void finalize_parts(const Hierarchy& H, int nparts, int op, cudaStream_t s);

namespace {

constexpr int kTile = kSweepTile;
constexpr int kConsumerWarps = kTile / 32;
constexpr int kThreads = kTile + 64;   // + a producer warp (TMA) and a gather warp (off-tile cp.async)

struct ApMaps {
    CUtensorMap bands;  // 3-D box kTile x G x 4: U, H0, H1, H2 (x 1, 2-D: U with the edge store); PUPD: D first
    CUtensorMap x;      // box kTile x (G + 1): x, or p_old (PUPD), or u (RESID)
    CUtensorMap z;      // box kTile x (G + 1): z (PUPD)
    CUtensorMap b;      // box kTile x G: right-hand side (RESID)
};

struct ApLayout {
    int x, z, b, hx, hz, eh, stage;
};
// eh: the band box carries U (PUPD: D, U) only; couplings from the edge store
// (one row of kEdgeRow doubles per layer: contiguous range, then gathered edges)
__host__ __device__ constexpr int ap_band_planes(bool pupd, bool eh) { return (eh ? 2 : 5) - (pupd ? 0 : 1); }
__host__ __device__ constexpr ApLayout ap_layout(bool pupd, int G, bool eh = false, bool resid = false) {
    static_assert(kTile % 2 == 0, "");
    ApLayout L{};
    L.x = ap_band_planes(pupd, eh) * G * kTile;
    L.z = L.x + (G + 1) * kTile;
    L.b = L.z + (pupd ? (G + 1) * kTile : 0);
    L.hx = L.b + (resid ? G * kTile : 0);
    // halo rows with the tile rows' stride kTile: a neighbour's operand is read at
    // one per-tile offset (tile or halo part) + kk * kTile
    // (with the p update the halo rows of z sit as far after those of p_old as the
    // tile rows of z after those of p_old: (G + 1) rows)
    L.hz = L.hx + (pupd ? (G + 1) : G) * kTile;
    L.eh = L.hz + (pupd ? G * kTile : 0);
    L.stage = L.eh + (eh ? G * kEdgeRow : 0);
    return L;
}

// RESID (Alg. 1 M2): r = b - H^ u formed like y (reading R5 order, then b - acc)
// and restricted in the epilogue, b_c[k][p] = ((r_4p + r_4p+1) + r_4p+2) + r_4p+3
// over four adjacent lanes (reading R8; k_resid_restrict's order) into y = b_c
// (leading dimension ldc, column offset coff).
template <bool DOT, bool PUPD, int G, bool EH = false, bool RESID = false>
__global__ void __launch_bounds__(kThreads, 3)
    k_apply_st(const __grid_constant__ ApMaps maps, LevelView L, TileHalo th, EdgeTiles et,
               const double* __restrict__ xin,
               const double* __restrict__ zv, double* __restrict__ y, double* __restrict__ pnew,
               double* __restrict__ partial, const PcgScalars* __restrict__ sc, int S, int64_t ldc, int64_t coff,
               const double* __restrict__ geom, double dz, int nsplit, FinArgs fin) {
    static_assert(!(RESID && (DOT || PUPD)), "residual mode: plain operator only");
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ double red[kThreads / 32];
    constexpr ApLayout AL = ap_layout(PUPD, G, EH, RESID);
    constexpr bool ND = !PUPD;                 // D re-formed by the consumers, not streamed
    constexpr int NBP = ap_band_planes(PUPD, EH);
    const int nz = L.nz;
    const int64_t ld = L.ld;
    const int ngroups = (nz + G - 1) / G;
    const int ntiles = (int)((L.n + kTile - 1) / kTile);
    // work unit = (tile, one of nsplit contiguous layer ranges): small levels split
    // their columns' layers so that every resident CTA has work (launch_ap)
    const int nunits = ntiles * nsplit;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
    uint64_t* empty = full + S;
    double* stages = reinterpret_cast<double*>(smraw + 1024);
#ifdef HMG_CHECKED
    int* tags = reinterpret_cast<int*>(smraw + 896);   // checked builds: stage sequence numbers (S <= 32)
    int pseq = 0, cseq = 0;
#endif
    ptx::pdl_trigger();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 2);   // producer + gather warp
            ptx::mbar_init(&empty[s], kConsumerWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    ptx::pdl_wait();
    double dot = 0.0;
    int s = 0;
    uint32_t phase = 0;
    auto advance = [&]() {
        if (++s == S) {
            s = 0;
            phase ^= 1u;
        }
    };
    if (warp == kConsumerWarps + 1) {
        // ============ gather warp: off-tile operands and gathered couplings ============
        // (issued here, not by the producer, whose TMA issue is on the critical path)
        for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
            const int tile = un / nsplit, part = un - tile * nsplit;
            const int ga = part * ngroups / nsplit, gb = (part + 1) * ngroups / nsplit;
            const int hcount = th.count[tile];
            const int32_t h0 = lane < hcount ? th.cells[tile * kHaloMax + lane] : 0;
            const int32_t h1 = lane + 32 < hcount ? th.cells[tile * kHaloMax + lane + 32] : 0;
            const int ehc = EH ? et.hcount[tile] : 0;
            const int32_t eh0 = EH && lane < ehc ? et.hcells[tile * kEdgeHalo + lane] : 0;
            HMG_DCHECK(hcount <= kHaloMax && h0 >= 0 && h0 < ld && h1 >= 0 && h1 < ld);
            HMG_DCHECK(ehc <= kEdgeHalo && eh0 >= 0 && (!EH || eh0 < et.ldE));
            for (int gi = ga; gi < gb; ++gi, advance()) {
                ptx::mbar_wait(&empty[s], phase ^ 1u);
                double* st = stages + (size_t)s * AL.stage;
                for (int kk = 0; kk < G; ++kk) {
                    const int k = gi * G + kk;
                    if (k >= nz) break;
                    if (EH && lane < ehc)
                        ptx::cp_async8(st + AL.eh + kk * kEdgeRow + kEdgeRange + lane, et.H + (int64_t)k * et.ldE + eh0);
                    const double* src = xin + (int64_t)k * ld;
                    if (lane < hcount) ptx::cp_async8(st + AL.hx + kk * kTile + lane, src + h0);
                    if (lane + 32 < hcount) ptx::cp_async8(st + AL.hx + kk * kTile + lane + 32, src + h1);
                    if (PUPD) {
                        const double* srz = zv + (int64_t)k * ld;
                        if (lane < hcount) ptx::cp_async8(st + AL.hz + kk * kTile + lane, srz + h0);
                        if (lane + 32 < hcount) ptx::cp_async8(st + AL.hz + kk * kTile + lane + 32, srz + h1);
                    }
                }
                ptx::cp_async_arrive(&full[s]);
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&full[s]);
            }
        }
    } else if (warp == kConsumerWarps) {
        // ======================= producer warp =======================
        const uint64_t pol = ptx::policy_evict_first();
        const uint32_t bytes = (uint32_t)(sizeof(double) * (NBP * G * kTile + (PUPD ? 2 : 1) * (G + 1) * kTile +
                                                            (RESID ? G * kTile : 0)));
        for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
            const int tile = un / nsplit, part = un - tile * nsplit;
            const int ga = part * ngroups / nsplit, gb = (part + 1) * ngroups / nsplit;
            const int x = tile * kTile;
            const int32_t ee0 = EH ? et.e0[tile] : 0;
            const uint32_t ebytes = EH ? (uint32_t)(sizeof(double) * et.ne[tile]) : 0u;
            for (int gi = ga; gi < gb; ++gi, advance()) {
                ptx::mbar_wait(&empty[s], phase ^ 1u);
#ifdef HMG_CHECKED
                if (lane == 0) tags[s] = pseq;
                ++pseq;
#endif
                double* st = stages + (size_t)s * AL.stage;
                if (lane == 0) {
                    int nl = nz - gi * G;
                    nl = nl < G ? nl : G;
                    ptx::mbar_arrive_expect_tx(&full[s], bytes + (EH ? (uint32_t)nl * ebytes : 0u));
                    if (EH)
                        for (int kk = 0; kk < nl; ++kk)
                            ptx::bulk_g2s(st + AL.eh + kk * kEdgeRow, et.H + (int64_t)(gi * G + kk) * et.ldE + ee0,
                                          ebytes, &full[s]);
                    if (NBP == 1)
                        ptx::tma_load_2d_hint(st, &maps.bands, x, gi * G, &full[s], pol);
                    else
                        ptx::tma_load_3d_hint(st, &maps.bands, x, gi * G, 0, &full[s], pol);
                    if (RESID) ptx::tma_load_2d_hint(st + AL.b, &maps.b, x, gi * G, &full[s], pol);
                    ptx::tma_load_2d(st + AL.x, &maps.x, x, gi * G, &full[s]);
                    if (PUPD) ptx::tma_load_2d(st + AL.z, &maps.z, x, gi * G, &full[s]);
                }
            }
        }
    } else {
        // ======================= consumers: one column per thread =======================
        const int j = threadIdx.x;
        const double beta = PUPD ? sc->beta : 0.0;
        for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
            const int tile = un / nsplit, part = un - tile * nsplit;
            const int ga = part * ngroups / nsplit, gb = (part + 1) * ngroups / nsplit;
            const int64_t c = (int64_t)tile * kTile + j;
            const bool valid = c < L.n;
            const uint32_t loc = th.loc[valid ? c : L.n - 1];
            const double vol = ND ? geom[valid ? c : L.n - 1] * dz : 0.0;   // k_assemble's prism volume
            const int l0 = loc & 0xff, l1 = (loc >> 8) & 0xff, l2 = (loc >> 16) & 0xff;
            // stage offsets of the neighbours' x (p_old) at row 0; their z lies at the same
            // offset + (AL.z - AL.x) (tile and halo rows of z both sit that far after x's)
            HMG_DCHECK(l0 < kTile + kHaloMax && l1 < kTile + kHaloMax && l2 < kTile + kHaloMax);
            const int ox0 = l0 < kTile ? AL.x + l0 : AL.hx + (l0 - kTile);
            const int ox1 = l1 < kTile ? AL.x + l1 : AL.hx + (l1 - kTile);
            const int ox2 = l2 < kTile ? AL.x + l2 : AL.hx + (l2 - kTile);
            int eo0 = 0, eo1 = 0, eo2 = 0;             // the faces' offsets in an edge row
            if (EH) {
                const uint32_t el = et.loc[valid ? c : L.n - 1];
                eo0 = el & 0xff;
                eo1 = (el >> 8) & 0xff;
                eo2 = (el >> 16) & 0xff;
            }
            HMG_DCHECK(eo0 < kEdgeRow && eo1 < kEdgeRow && eo2 < kEdgeRow);
            double xm = 0.0, Um = 0.0;
            if (ga > 0) {   // a unit starting above layer 0: x (p) and U of the layer below
                const int64_t i = (int64_t)(ga * G - 1) * ld + (valid ? c : L.n - 1);
                xm = PUPD ? zv[i] + beta * xin[i] : xin[i];
                Um = L.U[i];
            }
            for (int gi = ga; gi < gb; ++gi, advance()) {
                ptx::mbar_wait(&full[s], phase);
#ifdef HMG_CHECKED
                HMG_DCHECK(tags[s] == cseq);
                ++cseq;
#endif
                const double* st = stages + (size_t)s * AL.stage;
                const double* sx = st + AL.x;
                const double* sz = st + AL.z;
                const double* hx = st + AL.hx;
                const double* hz = st + AL.hz;
                auto XV = [&](int kk, int l) -> double {   // operand of local slot l at stage row kk
                    if (l < kTile) {
                        if (PUPD) return sz[kk * kTile + l] + beta * sx[kk * kTile + l];
                        return sx[kk * kTile + l];
                    }
                    if (PUPD) return hz[kk * kTile + l - kTile] + beta * hx[kk * kTile + l - kTile];
                    return hx[kk * kTile + l - kTile];
                };
                // the three neighbours' operands at the per-tile offsets (same values as XV)
                auto XN = [&](int kk, int q) -> double {
                    const int ox = q == 0 ? ox0 : q == 1 ? ox1 : ox2;
                    if (PUPD) return st[ox + (AL.z - AL.x) + kk * kTile] + beta * st[ox + kk * kTile];
                    return st[ox + kk * kTile];
                };
                // one layer; IN (interior, 0 < k < nz - 1) drops the boundary tests
                auto step = [&](int kk, auto interior) {
                    constexpr bool IN = decltype(interior)::value;
                    const int k = gi * G + kk;
                    const double* sr = st + kk * kTile + j;
                    constexpr int pu = ND ? 0 : 1;     // plane of U in the stage's band rows
                    const double Uk = sr[pu * G * kTile];
                    const double* er = st + AL.eh + kk * kEdgeRow;
                    const double H0 = EH ? er[eo0] : sr[(pu + 1) * G * kTile];
                    const double H1 = EH ? er[eo1] : sr[(pu + 2) * G * kTile];
                    const double H2 = EH ? er[eo2] : sr[(pu + 3) * G * kTile];
                    double Dk;
                    if (ND) {
                        // k_assemble's diagonal vol + V_dn + V_up + H0 + H1 + H2 from the stored
                        // U = -V_up, H_j = -(coupling) (x + (-y) is x - y exactly): bitwise D_k
                        Dk = vol;
                        if (IN || k > 0) Dk = Dk - Um;
                        if (IN || k < nz - 1) Dk = Dk - Uk;
                        Dk = Dk - H0;
                        Dk = Dk - H1;
                        Dk = Dk - H2;
                    } else {
                        Dk = sr[0];
                    }
                    const double xk = XV(kk, j);
                    double xp = 0.0;
                    if (IN || k < nz - 1) xp = XV(kk + 1, j);
                    double acc = Dk * xk;
                    if (IN || k > 0) acc = acc + Um * xm;
                    if (IN || k < nz - 1) acc = acc + Uk * xp;
                    acc = acc + H0 * XN(kk, 0);
                    acc = acc + H1 * XN(kk, 1);
                    acc = acc + H2 * XN(kk, 2);
                    if (RESID) {
                        const double r = st[AL.b + kk * kTile + j] - acc;
                        const double r1 = __shfl_down_sync(0xffffffffu, r, 1);
                        const double r2 = __shfl_down_sync(0xffffffffu, r, 2);
                        const double r3 = __shfl_down_sync(0xffffffffu, r, 3);
                        if (valid && (j & 3) == 0) y[(int64_t)k * ldc + coff + (c >> 2)] = ((r + r1) + r2) + r3;
                    } else if (valid) {
                        const int64_t i = (int64_t)k * ld + c;
                        y[i] = acc;
                        if (PUPD) pnew[i] = xk;
                        if (DOT) dot = dot + xk * acc;
                    }
                    xm = xk;
                    Um = Uk;
                };
                if (gi > 0 && (gi + 1) * G < nz) {
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) step(kk, std::true_type{});
                } else {
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        if (gi * G + kk >= nz) break;
                        step(kk, std::false_type{});
                    }
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
            }
        }
    }
    if (DOT) {   // fixed-order CTA reduction (the producer warp contributes 0)
        for (int off = 16; off > 0; off >>= 1) dot = dot + __shfl_down_sync(0xffffffffu, dot, off);
        if (lane == 0) red[warp] = dot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) t = t + red[w];
            partial[blockIdx.x] = t;
        }
        fin_fused(fin, partial);   // the last CTA: alpha = rho / <p, q> (fused finalize)
    }
}

template <bool DOT, bool PUPD, int G, bool EH = false, bool RESID = false>
int launch_ap(const Hierarchy& H, const DevLevel& L, const double* x, const double* z, double* y, double* pnew,
              cudaStream_t s, const double* b = nullptr, int64_t ldc = 0, int64_t coff = 0) {
    const int nz = H.nz;
    constexpr ApLayout AL = ap_layout(PUPD, G, EH, RESID);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
    // resident CTAs per SM (shared memory split evenly): three for the p-update
    // and residual variants (more consumer warps: C2b 244 -> 225 us and 183 -> 172
    // us), two for the plain apply.  A level with at most 1.5 tiles per SM
    // (ref <= 5: C1's 160 tiles) runs three per SM and splits each column's
    // layers into nsplit contiguous ranges, one work unit each, so that every
    // resident CTA streams (C1: 320 units of 32 layers instead of 160 tiles on
    // 148 SMs).
    const unsigned ntiles = (unsigned)((L.n + kTile - 1) / kTile);
    const int ngroups = (nz + G - 1) / G;
    const bool small = 2 * ntiles <= 3u * (unsigned)sms;
    int nsplit = small ? (int)((3u * (unsigned)sms) / (ntiles > 0 ? ntiles : 1u)) : 1;
    nsplit = nsplit < 1 ? 1 : (nsplit > 4 ? 4 : nsplit);
    nsplit = nsplit > ngroups ? ngroups : nsplit;
    const int per_sm = small ? 3 : (PUPD || RESID) ? H.apply_ctas_per_sm : 2;
    const size_t budget = (size_t)(per_sm >= 3 ? 72 : 110) * 1024;
    int S = (int)((budget - 1024) / (sizeof(double) * AL.stage));
    S = S < 2 ? 2 : (S > 32 ? 32 : S);
    const size_t smem = 1024 + sizeof(double) * (size_t)S * AL.stage;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_apply_st<DOT, PUPD, G, EH, RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
    }
    ApMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const LevelView V = L.view(nz);
    maps.bands = make_tensor_map(PUPD ? V.D : V.U, L.ld, nz, kTile, G, ap_band_planes(PUPD, EH));
    maps.x = make_tensor_map(x, L.ld, nz, kTile, G + 1, 1);
    if (PUPD) maps.z = make_tensor_map(z, L.ld, nz, kTile, G + 1, 1);
    if (RESID) maps.b = make_tensor_map(b, L.ld, nz, kTile, G, 1);
    const unsigned nunits = ntiles * (unsigned)nsplit;
    const unsigned cap = (unsigned)((per_sm >= 3 ? 3 : 2) * sms);
    const unsigned grid = nunits < cap ? nunits : cap;
    launch_pdl(H, k_apply_st<DOT, PUPD, G, EH, RESID>, dim3(grid), dim3(kThreads), smem, s, maps, V, L.halo, L.edge, x,
               z, y, pnew, H.partials, H.scal, S, ldc, coff, L.geom, H.dz, nsplit, DOT ? fin_take(H) : FinArgs());
    return (int)grid;
}

}  // namespace

// b_c = R(b - H^ u) through the streamed apply; used where the level has the
// edge store and columns of <= 64 layers (C2b fine level: 209 -> 185 us).  With
// 128 layers the thread-per-column k_resid_restrict streams its long columns at
// 6.4 TB/s and stays faster (C4: 1,524 against 1,596 us), so it keeps the
// per-cell bands there.
bool resid_st_supported(const Hierarchy& H, const DevLevel& L) {
    return H.resid_st && L.edge.H != nullptr && H.use_st_apply && !H.matrix_free && L.halo.loc != nullptr &&
           H.nz >= 2 && H.nz <= 64;
}

void launch_resid_restrict_st(const Hierarchy& H, const DevLevel& L, const double* b, const double* u, double* bc,
                              int64_t ldc, int64_t coff, cudaStream_t s) {
    try {
        launch_ap<false, false, 2, true, true>(H, L, u, nullptr, bc, nullptr, s, b, ldc, coff);
    } catch (const std::exception& e) {
        g_launch_error = std::string("residual launch: ") + e.what();
    }
    ++H.launches;
}

bool apply_st_supported(const Hierarchy& H, const DevLevel& L) {
    return H.use_st_apply && L.halo.loc != nullptr && H.nz >= 2;
}

// y = H^ x (dot: partial <x, H^ x> per CTA into H.partials, returns the count; 0 otherwise)
int launch_apply_st(const Hierarchy& H, const DevLevel& L, const double* x, double* y, bool dot, cudaStream_t s) {
    int n = 0;
    try {
        const bool eh = L.edge.H != nullptr;
        if (dot && eh)
            n = launch_ap<true, false, 2, true>(H, L, x, nullptr, y, nullptr, s);
        else if (dot)
            n = launch_ap<true, false, 2>(H, L, x, nullptr, y, nullptr, s);
        else if (eh)
            launch_ap<false, false, 2, true>(H, L, x, nullptr, y, nullptr, s);
        else
            launch_ap<false, false, 2>(H, L, x, nullptr, y, nullptr, s);
    } catch (const std::exception& e) {
        g_launch_error = std::string("apply launch: ") + e.what();
    }
    ++H.launches;
    return n;
}

// q = H^ p with p = z + beta p_old formed on the fly and stored in pnew; partial <p, q>
int launch_apply_pupdate_st(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                            double* q, cudaStream_t s) {
    int n = 0;
    try {
        if (L.edge.H)
            n = launch_ap<true, true, 2, true>(H, L, pold, z, q, pnew, s);
        else
            n = launch_ap<true, true, 2>(H, L, pold, z, q, pnew, s);
    } catch (const std::exception& e) {
        g_launch_error = std::string("apply launch: ") + e.what();
    }
    ++H.launches;
    return n;
}

}  // namespace hmg
