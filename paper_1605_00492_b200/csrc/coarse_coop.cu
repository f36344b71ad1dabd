// Coarse levels of the V-cycle in ONE cooperative kernel launch, with the
// operands of each 32-column tile resident in shared memory.
//
// Alg. 1 below the level `top` (default: ref 4, the first level
// whose sweeps are bounded by the length of the column recurrences rather
// than by HBM bandwidth; the paper saw the same coarse-level inefficiency on
// CPUs): presmoothing, residual restriction, the coarsest level's
// n_coarse sweeps (BASELINE.json: 20) and the postsmoothing with the fused
// prolongation.  Each CTA is one warp owning 32-column tiles; per level it
// brings the tile's bands and precomputed Thomas factors into shared memory
// with two TMA tensor copies, and each dependent step (a sweep, a restriction)
// ends in a grid barrier (~1.2 us on B200) instead of a kernel boundary
// (~3 us per dependent launch plus the TMA prologue of a fresh CTA).  Between
// steps, values cross tiles through global memory (L2): every step reloads
// the tile's iterate and its <= 32 off-tile neighbour cells.
//
// Arithmetic: tile_sweep (small_tile.cuh), identical in operation order to
// every other sweep (readings R5-R9), so the result is bitwise the oracle's.
#include <cuda.h>

#include <cooperative_groups.h>
#include <cstring>
#include <stdexcept>

#include "hmg_internal.h"
#include "small_tile.cuh"
#include "sm100_ptx.cuh"

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);

namespace {

constexpr int kCoopLevels = 5;

#ifdef HMG_TIMING
__device__ long long g_coop_timing[512];
__device__ int g_coop_label[512];
// label: 0 start, 1 operands loaded, 2 tile sweep done, 3 grid barrier passed, 4 coarsest sweeps done
#define CSTAMP(lbl)                                                           \
    do {                                                                      \
        if (blockIdx.x == 0 && threadIdx.x == 0 && nst < 512) {               \
            g_coop_label[nst] = (lbl);                                        \
            g_coop_timing[nst++] = clock64();                                 \
        }                                                                     \
    } while (0)
#else
#define CSTAMP(lbl) do {} while (0)
#endif   // levels top..coarsest handled (index = ref - coarsest)

struct CoopLevel {
    LevelView V;
    SmallHalo sh;
    double *wa, *wb, *b, *u;
    int ntiles;
};

struct CoopParams {
    CUtensorMap bands[kCoopLevels];   // 3-D box 32 x nzp x 5 (D, U, H0, H1, H2)
    CUtensorMap fact[kCoopLevels];    // 3-D box 32 x nzp x 3 (den, y, g)
    CoopLevel lev[kCoopLevels];
    int nz, top, coarsest, nu_pre, nu_post, n_coarse;
    double omega;
    const double* b_top;
    double* out_top;
};

struct CoopSmem {
    size_t bands, fact, b, u, hu, z, uc, huc, bar, total;
};

// TW-column tiles: TW = 32 while the tile's operands fit in shared memory
// (nz <= 64), 16 up to nz = 128, 8 up to nz = 256; lanes >= TW idle.
__host__ __device__ inline CoopSmem coop_layout(int nz, int TW) {
    CoopSmem L;
    const size_t rows = (size_t)((nz + 7) & ~7);            // layers padded to 8
    const size_t plane = sizeof(double) * rows * TW;
    const size_t hplane = sizeof(double) * rows * kHaloW;   // halo planes: <= 32 off-tile cells
    size_t off = 0;
    L.bands = off; off += 5 * plane;
    L.fact = off;  off += 3 * plane;
    L.b = off;     off += plane;
    L.u = off;     off += plane;
    L.hu = off;    off += hplane;
    L.z = off;     off += plane;
    L.uc = off;    off += plane / 4;      // [nz][TW/4] parents of the tile (prolongation)
    L.huc = off;   off += hplane;         // [nz][kHaloW] parents of the halo cells
    L.bar = off;   off += 64;
    L.total = off;
    return L;
}

constexpr int kCoopThreads = 32 * kTileWarps;   // 4 warps per tile

template <int TW>
__global__ void __launch_bounds__(kCoopThreads, 1) k_coarse_coop(const __grid_constant__ CoopParams P) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int nz = P.nz, nzp = (nz + 7) & ~7;
    const int tid = threadIdx.x, warp = tid >> 5;
    // j: the column of this lane; lanes >= TW repeat column TW - 1 (identical
    // values written to identical addresses) and never store to global memory
    const int lane = tid & 31;
    const int j = lane < TW ? lane : TW - 1;
    const bool jlane = lane < TW;
    const CoopSmem lay = coop_layout(nz, TW);
    const int PL = nzp * TW;                           // doubles per plane
    double* sB = reinterpret_cast<double*>(smraw + lay.bands);
    double* sF = reinterpret_cast<double*>(smraw + lay.fact);
    double* sb = reinterpret_cast<double*>(smraw + lay.b);
    double* su = reinterpret_cast<double*>(smraw + lay.u);
    double* shu = reinterpret_cast<double*>(smraw + lay.hu);
    double* sz = reinterpret_cast<double*>(smraw + lay.z);
    double* suc = reinterpret_cast<double*>(smraw + lay.uc);
    double* shuc = reinterpret_cast<double*>(smraw + lay.huc);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + lay.bar);
    const TileSmem S{sB, sB + PL, sB + 2 * PL, sB + 3 * PL, sB + 4 * PL, sF, sF + PL, sF + 2 * PL, sb, su, shu, sz};
    if (tid == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
    }
    // padding rows (layers nz..nzp-1) of the vector planes stay zero
    for (int q = nz * TW + tid; q < PL; q += kCoopThreads) sb[q] = su[q] = 0.0;
    for (int q = nz * kHaloW + tid; q < nzp * kHaloW; q += kCoopThreads) shu[q] = 0.0;
    __syncthreads();
#ifdef HMG_TIMING
    int nst = 0;
#endif
    CSTAMP(0);
    uint32_t phase = 0;
    int loaded_l = -1, loaded_tile = -1;               // which tile's bands/factors are in shared memory

    // bands + factors of (level l, tile t): two TMA tensor copies (the caller
    // has synchronised the CTA since the planes were last read)
    auto load_static = [&](int l, int t) {
        if (loaded_l == l && loaded_tile == t) return;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads before async writes
        if (tid == 0) {
            ptx::mbar_arrive_expect_tx(bar, (uint32_t)(8 * sizeof(double) * PL));
            ptx::tma_load_3d(sB, &P.bands[l - P.coarsest], t * TW, 0, 0, bar);
            ptx::tma_load_3d(sF, &P.fact[l - P.coarsest], t * TW, 0, 0, bar);
        }
        ptx::mbar_wait(bar, phase);
        phase ^= 1u;
        loaded_l = l;
        loaded_tile = t;
    };
    const CoopLevel* LV = P.lev - P.coarsest;          // LV[ref]
    // Vector loads are asynchronous copies (one round trip for a whole tile):
    // rows of w columns starting at col0 of v (leading dimension ld) into the
    // plane dst [nz][w], 16 bytes per copy (w = 32 or 8).  Columns beyond n are
    // padding and only feed lanes whose results are discarded.
    auto cp_rows = [&](double* dst, const double* v, int64_t ld, int64_t col0, int w) {
        const int cpr = w / 2;                          // 16-byte chunks per row
        for (int q = tid; q < nz * cpr; q += kCoopThreads) {
            const int k = q / cpr, ch = q - k * cpr;
            ptx::cp_async16(dst + k * w + 2 * ch, v + k * ld + col0 + 2 * ch);
        }
    };
    // Tile metadata (the column's neighbour slots, the halo cell list) of the
    // (level, tile) last visited, kept in registers: a CTA that owns one tile of
    // a level reads it from global memory once per level, not once per step
    // (three dependent L2 round trips at the start of every step otherwise).
    const CoopLevel* m_lev = nullptr;
    int m_t = -1, m_hcount = 0;
    uint32_t m_loc = 0;
    int32_t m_hc = 0;
    auto meta = [&](const CoopLevel& L, int t) {
        if (m_lev == &L && m_t == t) return;
        const int64_t c = (int64_t)t * TW + j;
        const uint32_t loc = L.sh.loc[c < L.V.n ? c : L.V.n - 1];
        const int hcount = L.sh.count[t];
        const int32_t hc = L.sh.cells[t * kSmallHaloMax + lane];   // slots past hcount: unused
        HMG_DCHECK(hcount <= kSmallHaloMax && (lane >= hcount || (hc >= 0 && hc < L.V.ld)));
        HMG_DCHECK((loc & 0xff) < TW + kHaloW && ((loc >> 8) & 0xff) < TW + kHaloW && ((loc >> 16) & 0xff) < TW + kHaloW);
        m_loc = loc;
        m_hcount = hcount;
        m_hc = lane < hcount ? hc : 0;
        m_lev = &L;
        m_t = t;
    };
    // off-tile neighbour values of v (cell >> shift) into the plane dst: lane h
    // of every warp gathers halo cell h, warps split the layers
    auto cp_halo = [&](double* dst, const double* v, const CoopLevel& L, int t, int shift, int64_t ldv) {
        meta(L, t);
        if (lane < m_hcount) {
            const int32_t hc = m_hc >> shift;
            for (int k = warp; k < nz; k += kTileWarps) ptx::cp_async8(dst + k * kHaloW + lane, v + k * ldv + hc);
        }
    };
    auto cp_wait = [&]() {
        ptx::cp_async_wait_all();
        __syncthreads();
    };
    auto store_own = [&](double* dst, const CoopLevel& L, int64_t c) {
        if (jlane && c < L.V.n)
            for (int k = warp; k < nz; k += kTileWarps) dst[k * L.V.ld + c] = su[k * TW + j];
    };
    auto slots = [&](const CoopLevel& L, int64_t c, int& l0, int& l1, int& l2) {   // c = t * TW + j
        meta(L, (int)(c / TW));
        l0 = m_loc & 0xff;
        l1 = (m_loc >> 8) & 0xff;
        l2 = (m_loc >> 16) & 0xff;
    };
    // What the vector planes hold: sb = tile res_t of res_b, su = the same tile
    // of res_u (the iterate this CTA last wrote or read for it).  A CTA that
    // owns a single tile of a level keeps both across that level's steps and
    // gathers only the off-tile neighbours again.
    const double* res_b = nullptr;
    const double* res_u = nullptr;
    int res_t = -1;
    auto load_vectors = [&](const CoopLevel& L, int t, const double* bl, const double* uin) {
        const bool keep_b = t == res_t && bl == res_b;
        if (!keep_b) cp_rows(sb, bl, L.V.ld, (int64_t)t * TW, TW);
        if (uin) {
            if (!(keep_b && uin == res_u)) cp_rows(su, uin, L.V.ld, (int64_t)t * TW, TW);
            cp_halo(shu, uin, L, t, 0, L.V.ld);
        }
    };
    auto resident = [&](int t, const double* bl, const double* u) {
        res_t = t;
        res_b = bl;
        res_u = u;
    };
    // A CTA with several tiles of a level visits them in alternating order from
    // one step to the next, so the tile it finished last (operands resident in
    // shared memory) is the first of the next step.
    bool rev = false;
    auto my_tiles = [&](const CoopLevel& L) {
        rev = !rev;
        return L.ntiles > (int)blockIdx.x ? (L.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    };
    // one damped sweep of level l from iterate uin (nullptr: zero guess) to uout, all tiles
    auto sweep_step = [&](int l, const double* bl, const double* uin, double* uout) {
        const CoopLevel& L = LV[l];
        const int cnt = my_tiles(L);
        for (int i = 0; i < cnt; ++i) {
            const int t = (int)blockIdx.x + (int)gridDim.x * (rev ? cnt - 1 - i : i);
            const int64_t c = (int64_t)t * TW + j;
            int l0, l1, l2;
            slots(L, c, l0, l1, l2);
            __syncthreads();                           // every thread is done with the previous tile's planes
            load_vectors(L, t, bl, uin);
            load_static(l, t);
            cp_wait();
            CSTAMP(1);
            tile_sweep_cta<TW>(S, nz, warp, j, l0, l1, l2, uin == nullptr, P.omega, jlane && c < L.V.n);
            CSTAMP(2);
            store_own(uout, L, c);
            resident(t, bl, uout);
        }
    };

    const double* cur[kMaxRef + 1];
    // ---- down leg: presmooth, restrict the residual ----
    for (int l = P.top; l > P.coarsest; --l) {
        const CoopLevel& L = LV[l];
        const CoopLevel& C = LV[l - 1];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        const double* c_in = nullptr;
        for (int s = 0; s < P.nu_pre; ++s) {
            double* dst = (c_in == L.wa) ? L.wb : L.wa;
            sweep_step(l, bl, c_in, dst);
            grid.sync();
            CSTAMP(3);
            c_in = dst;
        }
        cur[l] = c_in;
        const int cnt = my_tiles(L);
        for (int i = 0; i < cnt; ++i) {
            const int t = (int)blockIdx.x + (int)gridDim.x * (rev ? cnt - 1 - i : i);
            const int64_t c = (int64_t)t * TW + j;
            int l0, l1, l2;
            slots(L, c, l0, l1, l2);
            __syncthreads();
            load_vectors(L, t, bl, c_in);
            load_static(l, t);
            cp_wait();
            resident(t, bl, c_in);
            CSTAMP(1);
            tile_residuals_cta<TW>(S, nz, warp, j, l0, l1, l2, c_in == nullptr);   // r = b - H^ u (r = b from zero)
            __syncthreads();
            // b_c[k][p] = ((r0 + r1) + r2) + r3 over the children 4p..4p+3: thread = (parent, layer phase)
            constexpr int PT = TW / 4;                 // parents per tile
            const int pp = tid % PT, kph = tid / PT;
            const int64_t p = (int64_t)t * PT + pp;
            if (p < C.V.n)
                for (int k = kph; k < nz; k += kCoopThreads / PT) {
                    const double* r = sz + k * TW + 4 * pp;
                    C.b[k * C.V.ld + p] = ((r[0] + r[1]) + r[2]) + r[3];
                }
        }
        grid.sync();
        CSTAMP(3);
    }
    // ---- coarsest level: n_coarse sweeps from zero ----
    {
        const int l = P.coarsest;
        const CoopLevel& L = LV[l];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        double* out = (l == P.top) ? P.out_top : L.u;
        if (L.ntiles == 1) {
            // one tile: every sweep stays in shared memory (no off-tile neighbours)
            if (blockIdx.x == 0) {
                const int64_t c = j;
                int l0, l1, l2;
                slots(L, c, l0, l1, l2);
                __syncthreads();
                cp_rows(sb, bl, L.V.ld, 0, TW);
                load_static(l, 0);
                cp_wait();
                CSTAMP(1);
                for (int s = 0; s < P.n_coarse; ++s)
                    tile_sweep_cta<TW>(S, nz, warp, j, l0, l1, l2, s == 0, P.omega, jlane && c < L.V.n);
                CSTAMP(4);
                store_own(out, L, c);
                resident(0, bl, out);
            }
        } else {
            const double* c_in = nullptr;
            for (int s = 0; s < P.n_coarse; ++s) {
                double* dst = (s == P.n_coarse - 1) ? out : ((c_in == L.wa) ? L.wb : L.wa);
                sweep_step(l, bl, c_in, dst);
                if (s < P.n_coarse - 1) grid.sync();
                c_in = dst;
            }
        }
        grid.sync();
        CSTAMP(3);
    }
    // ---- up leg: prolongation fused into the first postsmoothing sweep ----
    for (int l = P.coarsest + 1; l <= P.top; ++l) {
        const CoopLevel& L = LV[l];
        const CoopLevel& C = LV[l - 1];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        double* out = (l == P.top) ? P.out_top : L.u;
        const double* c_in = cur[l];                   // presmoothed iterate (nullptr: zero)
        // first step: u = c_in + P u_c formed in shared memory for the tile and its halo
        double* dst = (P.nu_post <= 1) ? out : ((c_in == L.wa) ? L.wb : L.wa);
        const int cnt = my_tiles(L);
        for (int i = 0; i < cnt; ++i) {
            const int t = (int)blockIdx.x + (int)gridDim.x * (rev ? cnt - 1 - i : i);
            const int64_t c = (int64_t)t * TW + j;
            const bool valid = c < L.V.n;
            int l0, l1, l2;
            slots(L, c, l0, l1, l2);
            const int64_t c0 = (int64_t)t * TW;
            __syncthreads();
            cp_rows(sb, bl, L.V.ld, c0, TW);
            if (c_in) {
                cp_rows(su, c_in, L.V.ld, c0, TW);
                cp_halo(shu, c_in, L, t, 0, L.V.ld);
            }
            cp_rows(suc, C.u, C.V.ld, c0 / 4, TW / 4);
            cp_halo(shuc, C.u, L, t, 2, C.V.ld);
            load_static(l, t);
            cp_wait();
            // u + P u_c, the addition of the prolongation (0 + u_c from a zero iterate)
            meta(L, t);
            const int hcount = m_hcount;
            for (int k = warp; k < nz; k += kTileWarps) {
                if (jlane) {
                    const double v = c_in ? su[k * TW + j] : 0.0;
                    su[k * TW + j] = v + suc[k * (TW / 4) + (j >> 2)];
                }
                if (lane < hcount) {
                    const double h = c_in ? shu[k * kHaloW + lane] : 0.0;
                    shu[k * kHaloW + lane] = h + shuc[k * kHaloW + lane];
                }
            }
            __syncthreads();
            CSTAMP(1);
            if (P.nu_post > 0) tile_sweep_cta<TW>(S, nz, warp, j, l0, l1, l2, false, P.omega, jlane && valid);
            CSTAMP(2);
            store_own(dst, L, c);
            resident(t, bl, dst);
        }
        grid.sync();
        CSTAMP(3);
        const double* prev = dst;
        for (int s = 1; s < P.nu_post; ++s) {
            double* d2 = (s == P.nu_post - 1) ? out : ((prev == L.wa) ? L.wb : L.wa);
            sweep_step(l, bl, prev, d2);
            grid.sync();
            CSTAMP(3);
            prev = d2;
        }
    }
}

#ifdef HMG_TIMING
}  // namespace
extern "C" void hmg_debug_coop_timing(long long* out) { cudaMemcpyFromSymbol(out, g_coop_timing, sizeof(long long) * 512); }
extern "C" void hmg_debug_coop_labels(int* out) { cudaMemcpyFromSymbol(out, g_coop_label, sizeof(int) * 512); }
extern "C" void hmg_debug_tile_phase(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_tile_phase, sizeof(unsigned long long) * 5);
}
extern "C" unsigned long long hmg_debug_tile_slow() {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_tile_slow_count, sizeof(v));
    return v;
}
namespace {
#endif

int coop_tile_width(int nz) {
    for (int tw : {32, 16, 8})
        if (coop_layout(nz, tw).total <= 227 * 1024) return tw;
    return 0;
}

template <int TW>
void launch_coop_tw(const Hierarchy& H, CoopParams& P, cudaStream_t s) {
    const int nz = H.nz, nzp = (nz + 7) & ~7;
    for (int r = H.coarsest_ref; r <= H.coop_ref; ++r) {
        const DevLevel& L = H.lev[r];
        const int i = r - H.coarsest_ref;
        CoopLevel& C = P.lev[i];
        C.ntiles = (int)((L.n + TW - 1) / TW);
        P.bands[i] = make_tensor_map(C.V.D, L.ld, nz, TW, nzp, 5);
        P.fact[i] = make_tensor_map(L.fden, L.ld, nz, TW, nzp, 3);
    }
    const size_t smem = coop_layout(nz, TW).total;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_coarse_coop<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_coop<TW>, kCoopThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
    // as many rounds of tiles on the top level as the resident CTAs need, the
    // tiles dealt evenly (C2b: 160 tiles -> 80 CTAs x 2 instead of 148 CTAs of
    // which 12 take a second tile -- the same critical path, and 68 SMs stay
    // free for the PCG's deferred x update on the side stream)
    const int ntop = P.lev[H.coop_ref - H.coarsest_ref].ntiles;
    const int cap = (per_sm < 1 ? 1 : per_sm) * sms;
    const int rounds = (ntop + cap - 1) / cap;
    const int grid = (ntop + rounds - 1) / rounds;
    ProfScope ps(H, kKCoarseTail, H.coop_ref, s);
    void* args[] = {&P};
    cudaLaunchCooperativeKernel((const void*)k_coarse_coop<TW>, dim3(grid), dim3(kCoopThreads), args, smem, s);
    ++H.launches;
}

}  // namespace

int coarse_coop_tile_width(int nz) { return coop_tile_width(nz); }

bool coarse_coop_supported(const Hierarchy& H) {
    if (H.coop_ref < 0) return false;
    if (H.coop_ref - H.coarsest_ref + 1 > kCoopLevels) return false;
    if (coop_tile_width(H.nz) == 0) return false;
    for (int r = H.coarsest_ref; r <= H.coop_ref; ++r) {
        const DevLevel& L = H.lev[r];
        if (!L.fden || !L.coop_halo.loc) return false;
    }
    return true;
}

void launch_coarse_coop(const Hierarchy& H, const hmg_mg_params& p, const double* b_top, double* out_top,
                        cudaStream_t s) {
    static_assert(sizeof(CoopParams) <= 4096, "kernel parameter block");
    CoopParams P;
    std::memset(&P, 0, sizeof(P));
    P.nz = H.nz;
    P.top = H.coop_ref;
    P.coarsest = H.coarsest_ref;
    P.nu_pre = p.nu_pre;
    P.nu_post = p.nu_post;
    P.n_coarse = p.n_coarse;
    P.omega = p.omega;
    P.b_top = b_top;
    P.out_top = out_top;
    for (int r = H.coarsest_ref; r <= H.coop_ref; ++r) {
        const DevLevel& L = H.lev[r];
        CoopLevel& C = P.lev[r - H.coarsest_ref];
        C.V = L.view(H.nz);
        C.sh = L.coop_halo;
        C.wa = L.wa;
        C.wb = L.wb;
        C.b = L.b;
        C.u = L.u;
    }
    switch (coop_tile_width(H.nz)) {
        case 32: launch_coop_tw<32>(H, P, s); break;
        case 16: launch_coop_tw<16>(H, P, s); break;
        default: launch_coop_tw<8>(H, P, s); break;
    }
}

}  // namespace hmg
