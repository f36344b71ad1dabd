// Fused line-Jacobi sweep with a non-zero iterate, fully streamed: persistent
// CTAs, no shared-memory-resident tile of the iterate.
//
// Computes exactly what k_sweep (kernels.cu) and k_sweep_tc (sweep_tc.cu)
// compute for every column -- r = b - H^ u, delta = T^{-1} r (Thomas,
// P:741-744), u' = u + omega delta (Eq. 10 read with Eq. 13; readings R5-R7),
// with the prolongation u <- u + P u_c optionally fused (Alg. 1 M4) -- in the
// same operation order, so the results are bitwise identical.  What differs
// from k_sweep_tc is the data movement:
//
//  * k_sweep_tc keeps the tile's u rows (64 KB at nz = 64) in shared memory
//    for the in-tile neighbours and the back substitution's u_old; that halves
//    its TMA ring and, with the fused prolongation, leaves two stages.  Here
//    the u rows travel in the ring like every other operand: a forward stage
//    carries G layers of the bands and b, G + 1 layers of u (layer k + 1 of the
//    own column is needed at layer k) and the <= 64 off-tile neighbours; a
//    backward stage brings 8 layers of u again for u' = u_old + omega delta.
//    That re-read is mostly an L2 hit: the forward copies of u use an
//    evict_last policy and the streamed-once bands an evict_first policy.
//  * Warp roles: 4 consumer warps (thread = column), a producer warp issuing
//    the TMA copies, and (stored bands, non-zero guess) a gather warp issuing
//    the off-tile cp.async gathers; the stage's full barrier counts both.
//  * CTAs are persistent (two per SM at nz <= 64).  With stored bands and a
//    non-zero guess (IL) pass p runs tile p's forward elimination and, one
//    8-layer chunk at a time, tile p - 1's back substitution; the Thomas state
//    (z_k, g_k) sits in tensor memory at slot k on even passes and nzp - 1 - k
//    on odd ones, so each slot is rewritten right after it was read.  The ring
//    keeps streaming through the back substitution, and the u' rows of a chunk
//    leave by one TMA store from its backward stage.
//  * D is not streamed: the consumers re-form D_k = ((((vol - U_{k-1}) - U_k)
//    - H0) - H1) - H2 from the column's prism volume and the streamed
//    couplings, k_assemble's sum term by term, so bitwise the stored D.
// HBM traffic per dof: u, b, U, H0, H1, H2 read once, u' written once
// (56 B/dof; the per-cell store's 64 of SURVEY 8(d) less D; 44 with the edge
// store; + 2 B/dof of u_c with the fused prolongation).
#include <cuda.h>

#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"
#include "mf_ops.cuh"

// Probe builds (tools/micro/st_probe.py only; never the product library):
// HMG_PROBE_NORES / NOCHAIN drop consumer work, NOHALO / NOBWD / NOEDGE drop
// parts of the data movement -- results are wrong, the timing says what bounds.
#if defined(HMG_PROBE_NOHALO) || defined(HMG_PROBE_NOBWD) || defined(HMG_PROBE_NOEDGE) || defined(HMG_PROBE_NOMOVE)
#define HMG_PROBE_NOCHAIN
#endif
#ifdef HMG_PROBE_NOMOVE
#define HMG_PROBE_NOHALO
#define HMG_PROBE_NOBWD
#define HMG_PROBE_NOEDGE
#endif
#ifndef HMG_ST_G
#define HMG_ST_G 2
#endif
#ifdef HMG_PROBE_NOHALO
constexpr bool kProbeHalo = false;
#else
constexpr bool kProbeHalo = true;
#endif
#ifdef HMG_PROBE_NOBWD
constexpr bool kProbeBwd = false;
#else
constexpr bool kProbeBwd = true;
#endif
#ifdef HMG_PROBE_NOEDGE
constexpr bool kProbeEdge = false;
#else
constexpr bool kProbeEdge = true;
#endif

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);
CUtensorMap make_store_map(double* base, int64_t ld, int64_t width, int64_t rows, int box_x, int G);
extern thread_local std::string g_launch_error;

namespace {

constexpr int kTile = kSweepTile;          // columns per tile (one consumer thread each)
constexpr int kConsumerWarps = kTile / 32;
constexpr int kThreads = kTile + 32;       // + one producer warp
constexpr int kMfWarps = kTile / 32;       // matrix-free: warps forming the couplings of each stage
constexpr int kThreadsMf = kThreads + 32 * kMfWarps;
constexpr int kThreadsSplit = kThreads + 32;  // stored bands, non-zero guess: + a gather warp for the halos
// threads of one CTA: the gather warp takes the off-tile cp.async gathers off
// the producer warp, whose TMA issue is on the sweep's critical path
__host__ __device__ constexpr int st_threads(bool zero, bool mf) { return mf ? kThreadsMf : zero ? kThreads : kThreadsSplit; }
constexpr int kBack = 8;                   // layers per backward stage
constexpr int kUcRow = 64;                 // forward u_c rows: 32 parents of the tile + the next 32 (so the
                                           // tile and halo parts of u_c share the row stride kHaloMax)

#ifdef HMG_TIMING
__device__ unsigned long long g_cta_ns[2 * 1024];   // per CTA: globaltimer at start and end
__device__ unsigned g_cta_sm[1024];
__device__ long long g_st_timing[12];  // CTA 0, thread 0: [0] total, [1] forward wait, [2] backward wait, [3] tiles;
                                       // producer lane 0: [8] total, [9] waiting for free slots, [10] stages
#endif

__device__ __forceinline__ bool pivot_ok(double den) { return den > 0.0 && den <= DBL_MAX; }

struct StMaps {
    CUtensorMap bands;  // 3-D box kTile x G x 5 (D, U, H0, H1, H2)     (stored bands)
    CUtensorMap lam;    // box kTile x (G + 1): coefficient rows          (matrix-free)
    CUtensorMap b;      // box kTile x G
    CUtensorMap uf;     // box kTile x (G + 1): forward u rows
    CUtensorMap ub;     // box kTile x 8: backward u rows
    CUtensorMap ucf;    // box kTile/4 x (G + 1)   (PROLONG)
    CUtensorMap ucb;    // box kTile/4 x 8         (PROLONG)
    CUtensorMap bb;     // box kTile x 8: backward b rows (DOT)
    CUtensorMap uo;     // box kTile x 8: u' rows stored from the backward stage (extent: the level's n columns)
};

// Doubles of one ring stage and the offsets of its parts.  Forward stage:
// operator rows (5 G band rows, or G + 1 lam rows), G rows of b, G + 1 rows
// of u (+ u_c), off-tile neighbour values (u, u_c, lam) of the G layers.
// Backward stage: [0, 8 kTile) u rows, then 8 kTile/4 u_c rows.
struct StLayout {
    int op, band, b, u, uc, hu, huc, hlam, eh, fwd, bwd, stage;
};
// eh: the band box carries D and U only; the couplings come from the edge
// store, one row of kEdgeRow doubles per layer (contiguous range, then gathered).
// Stored bands with a non-zero guess: the D rows are not streamed -- the
// consumers re-form D_k from the column's prism volume and the streamed
// couplings in k_assemble's order (st_band_planes).
__host__ __device__ constexpr int st_band_planes(bool zero, bool mf, bool eh) {
    return (eh ? 2 : 5) - ((!zero && !mf) ? 1 : 0);
}
__host__ __device__ constexpr StLayout st_layout(bool zero, bool prolong, bool mf, int G, bool dot = false,
                                                 bool eh = false) {
    StLayout L{};
    L.op = 0;                                        // band rows (stored), or lam rows (matrix-free)
    L.band = mf ? (G + 1) * kTile : 0;               // band rows as the consumers read them
    L.b = L.band + st_band_planes(zero, mf, eh) * G * kTile;
    L.u = L.b + G * kTile;
    L.uc = L.u + (zero ? 0 : (G + 1) * kTile);
    L.hu = L.uc + (prolong ? (G + 1) * kUcRow : 0);
    // halo rows of u: stride kTile where no prolongation / matrix-free parts use
    // them, so a neighbour is read at (tile or halo offset) + kk * kTile alike
    L.huc = L.hu + (zero ? 0 : G * (mf ? kHaloMax : kTile));
    L.hlam = L.huc + (prolong ? G * kHaloMax : 0);
    L.eh = L.hlam + (mf ? G * kHaloMax : 0);
    L.fwd = L.eh + (eh ? G * kEdgeRow : 0);
    L.bwd = zero ? 0 : kBack * kTile + (prolong ? kBack * (kTile / 4) : 0) + (dot ? kBack * kTile : 0);
    L.stage = L.fwd > L.bwd ? L.fwd : L.bwd;
    return L;
}

// Operator of one launch: the level's stored bands (view) or, matrix-free,
// its coefficient and geometry.
struct StOp {
    const double* lam;
    const double* geom;
    double w2, dz;
};

template <bool ZERO, bool PROLONG, bool MF, int G, bool CHK, bool DOT = false, bool EH = false>
__global__ void __launch_bounds__(st_threads(ZERO, MF), 2)
    k_sweep_st(const __grid_constant__ StMaps maps, LevelView L, StOp op, TileHalo th, EdgeTiles et,
               const double* __restrict__ bvec,
               const double* __restrict__ uin, const double* __restrict__ uc, int64_t ldc, double* __restrict__ uout,
               double omega, int ref, unsigned long long* __restrict__ bad, int S, uint32_t tmem_cols, int pf_groups,
               double* __restrict__ partial, FinArgs fin) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ double dred[kThreadsSplit / 32];
    static_assert(!(EH && (ZERO || MF)), "edge store: general stored-band sweeps only");
    constexpr StLayout SL = st_layout(ZERO, PROLONG, MF, G, DOT, EH);
    // ND: D_k is not streamed but re-formed by the consumers (st_band_planes);
    // the stage's band rows start at U
    constexpr bool ND = !ZERO && !MF;
    constexpr int NBP = st_band_planes(ZERO, MF, EH);
    double dotacc = 0.0;                               // DOT: this thread's sum of b_k u'_k
#ifdef HMG_TIMING
    long long tt0 = 0, wf = 0, wb = 0, ntl = 0, tfw = 0, tbk = 0, tfw0 = 0, tws = 0;
#endif
    constexpr bool HALO = !ZERO || MF;       // off-tile neighbour values needed
    constexpr int HS = MF ? kHaloMax : kTile;   // stride of the halo rows of u
    constexpr bool FLAT = !MF && !ZERO;         // neighbours read at per-tile offsets
    constexpr bool SPLIT = !MF && !ZERO;        // halo gathers issued by their own warp
    constexpr bool TSTORE = !ZERO;              // u' rows written back by TMA from the backward stage
    // IL: tile p's forward elimination interleaved with tile p - 1's back
    // substitution (see the consumers); stored bands and a non-zero guess
    constexpr bool IL = SPLIT;
    constexpr int kGpc = kBack / G;             // forward groups per 8-layer chunk
    static_assert(kBack % G == 0, "a chunk holds whole groups");
    static_assert(kUcRow == kHaloMax, "u_c tile and halo rows share one stride");
    const int nz = L.nz;
    const int64_t ld = L.ld;
    const int ngroups = (nz + G - 1) / G;
    const int nchunks = ZERO ? 0 : (nz + kBack - 1) / kBack;
    const int ntiles = (int)((L.n + kTile - 1) / kTile);
    const int ntc = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;   // my tiles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
    uint64_t* empty = full + S;
    uint64_t* mid = empty + S;                        // matrix-free: the stage's band rows are formed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mid + S);
    double* stages = reinterpret_cast<double*>(smraw + 1024);
#ifdef HMG_CHECKED
    int* tags = reinterpret_cast<int*>(smraw + 896);   // checked builds: stage sequence numbers (S <= 32)
    int pseq = 0, cseq = 0;
#define ST_TAG_SET() do { if (lane == 0) tags[s] = pseq; ++pseq; } while (0)
#define ST_TAG_CHECK() do { HMG_DCHECK(tags[s] == cseq); ++cseq; } while (0)
#else
#define ST_TAG_SET() do {} while (0)
#define ST_TAG_CHECK() do {} while (0)
#endif

    ptx::pdl_trigger();                                // the next kernel may start its prologue
#ifdef HMG_TIMING
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_cta_ns[2 * blockIdx.x] = t;
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_cta_sm[blockIdx.x] = sm;
    }
#endif
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], SPLIT ? 2 : 1);   // producer (+ gather warp)
            ptx::mbar_init(&empty[s], kConsumerWarps);
            ptx::mbar_init(&mid[s], kMfWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(tmem_slot, tmem_cols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    ptx::pdl_wait();                                   // the predecessor's results (b, u, u_c) are complete

    if (MF && warp > kConsumerWarps) {
        // ============ matrix-free warps: the couplings of each forward stage ============
        // Thread = column.  Writes D, U, H0, H1, H2 of the stage's G layers into
        // its band rows (k_assemble's values, bitwise) for the Thomas warps; passes
        // backward stages through.  A quotient outside the fast path's exact range
        // is recomputed with '/' on the spot (rare).
        const int j = threadIdx.x - 32 * (kConsumerWarps + 1);
        const int mlane = j & 31;
        const double ydz = div_recip(op.dz);
        int s = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        };
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t c = (int64_t)tile * kTile + j;
            const int64_t cv = c < L.n ? c : L.n - 1;
            const uint32_t loc = th.loc[cv];
            const int ls[3] = {(int)(loc & 0xff), (int)((loc >> 8) & 0xff), (int)((loc >> 16) & 0xff)};
            const ColumnGeom cg = column_geom(op.geom, ld, cv, op.w2, op.dz);
            double vdn = 0.0;
            for (int gi = 0; gi < ngroups; ++gi, advance()) {
                ptx::mbar_wait(&full[s], phase);
                double* st = stages + (size_t)s * SL.stage;
                const double* sl = st + SL.op;
                const double* hl = st + SL.hlam;
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const int k = gi * G + kk;
                    if (k >= nz) break;
                    const double lk = sl[kk * kTile + j];
                    bool slow = false;
                    double lp = 0.0, vup = 0.0;
                    if (k < nz - 1) {
                        lp = sl[(kk + 1) * kTile + j];
                        vup = mf_vcoup<false, CHK>(cg, lk, lp, op.dz, ydz, slow);
                    }
                    double hc[3], ln[3];
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        ln[q] = ls[q] < kTile ? sl[kk * kTile + ls[q]] : hl[kk * kHaloMax + ls[q] - kTile];
                        hc[q] = mf_hcoup<false, CHK>(cg, q, lk, ln[q], slow);
                    }
                    if (CHK && slow) {                     // rare: exact quotients
                        bool dummy = false;
                        if (k < nz - 1) vup = mf_vcoup<true>(cg, lk, lp, op.dz, ydz, dummy);
#pragma unroll
                        for (int q = 0; q < 3; ++q) hc[q] = mf_hcoup<true>(cg, q, lk, ln[q], dummy);
                    }
                    double* br = st + SL.band + kk * kTile + j;
                    br[0] = mf_diag(cg, k, nz, vdn, vup, hc[0], hc[1], hc[2]);
                    br[G * kTile] = (k < nz - 1) ? -vup : 0.0;
                    br[2 * G * kTile] = -hc[0];
                    br[3 * G * kTile] = -hc[1];
                    br[4 * G * kTile] = -hc[2];
                    vdn = vup;
                }
                __syncwarp();
                if (mlane == 0) ptx::mbar_arrive(&mid[s]);
            }
            for (int m = nchunks - 1; m >= 0; --m, advance()) {   // backward stages: pass through
                ptx::mbar_wait(&full[s], phase);
                __syncwarp();
                if (mlane == 0) ptx::mbar_arrive(&mid[s]);
            }
        }
    } else if (SPLIT && warp == kConsumerWarps + 1) {
        // ============ gather warp: off-tile u values and gathered couplings ============
        // Per forward stage: cp.async of the <= 64 halo u values and the <= 32
        // gathered edge couplings of each layer; the stage's full barrier counts
        // this warp's arrival after its copies are registered with it.
        int s = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        };
        // stage order of the interleaved schedule (IL, see the consumers): pass p
        // takes, per 8-layer chunk, tile p - 1's backward stage, then tile p's
        // forward stages of those layers
        for (int p = 0; p <= ntc; ++p) {
            const bool hasF = p < ntc, hasB = p > 0;
            const int tile = (int)blockIdx.x + p * (int)gridDim.x;
            int hcount = 0, ehc = 0;
            int32_t h0 = 0, h1 = 0, eh0 = 0;
            if (hasF) {
                hcount = th.count[tile];
                h0 = lane < hcount ? th.cells[tile * kHaloMax + lane] : 0;
                h1 = lane + 32 < hcount ? th.cells[tile * kHaloMax + lane + 32] : 0;
                ehc = EH ? et.hcount[tile] : 0;
                eh0 = EH && lane < ehc ? et.hcells[tile * kEdgeHalo + lane] : 0;
                HMG_DCHECK(hcount <= kHaloMax && h0 >= 0 && h0 < ld && h1 >= 0 && h1 < ld);
                HMG_DCHECK(ehc <= kEdgeHalo && eh0 >= 0 && (!EH || eh0 < et.ldE));
            }
            for (int ch = 0; ch < nchunks; ++ch) {
                if (hasB) {                                    // backward stage: one arrival
                    ptx::mbar_wait(&empty[s], phase ^ 1u);
                    if (lane == 0) ptx::mbar_arrive(&full[s]);
                    advance();
                }
                if (!hasF) continue;
                const int g1 = (ch + 1) * kGpc < ngroups ? (ch + 1) * kGpc : ngroups;
                for (int gi = ch * kGpc; gi < g1; ++gi, advance()) {
                    ptx::mbar_wait(&empty[s], phase ^ 1u);
                    double* st = stages + (size_t)s * SL.stage;
                    if (kProbeHalo) {
                        for (int kk = 0; kk < G; ++kk) {
                            const int k = gi * G + kk;
                            if (k >= nz) break;
                            if (EH && lane < ehc)
                                ptx::cp_async8(st + SL.eh + kk * kEdgeRow + kEdgeRange + lane,
                                               et.H + (int64_t)k * et.ldE + eh0);
                            const double* src = uin + (int64_t)k * ld;
                            if (lane < hcount) ptx::cp_async8(st + SL.hu + kk * HS + lane, src + h0);
                            if (lane + 32 < hcount) ptx::cp_async8(st + SL.hu + kk * HS + lane + 32, src + h1);
                            if (PROLONG) {
                                const double* srcc = uc + (int64_t)k * ldc;
                                if (lane < hcount)
                                    ptx::cp_async8(st + SL.huc + kk * kHaloMax + lane, srcc + (h0 >> 2));
                                if (lane + 32 < hcount)
                                    ptx::cp_async8(st + SL.huc + kk * kHaloMax + lane + 32, srcc + (h1 >> 2));
                            }
                        }
                        ptx::cp_async_arrive(&full[s]);
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&full[s]);
                }
            }
        }
    } else if (warp == kConsumerWarps) {
        // ======================= producer warp =======================
        const uint64_t pol_stream = ptx::policy_evict_first();
        const uint64_t pol_keep = ptx::policy_evict_last();
        constexpr int op_rows = MF ? (G + 1) * kTile : NBP * G * kTile;
        const uint32_t fwd_bytes =
            (uint32_t)(sizeof(double) * (op_rows + G * kTile + (ZERO ? 0 : (G + 1) * kTile) +
                                         (PROLONG ? (G + 1) * kUcRow : 0)));
        const uint32_t bwd_bytes = (uint32_t)(sizeof(double) * (kBack * kTile + (PROLONG ? kBack * (kTile / 4) : 0) +
                                                                (DOT ? kBack * kTile : 0)));
        int s = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        };
#ifdef HMG_TIMING
        long long p0 = clock64(), pw = 0, pn = 0, ph = 0;
#endif
        // one forward stage (group gi of the tile at column x)
        auto fwd_stage = [&](int tile, int gi, int hcount, int32_t h0, int32_t h1, int32_t ee0, uint32_t ebytes) {
            const int x = tile * kTile, xc = x / 4;
#ifdef HMG_TIMING
            long long q0 = clock64();
#endif
            ptx::mbar_wait(&empty[s], phase ^ 1u);
            ST_TAG_SET();
#ifdef HMG_TIMING
            pw += clock64() - q0;
            ++pn;
#endif
            double* st = stages + (size_t)s * SL.stage;
            if (HALO && !SPLIT && kProbeHalo) {
                for (int kk = 0; kk < G; ++kk) {          // off-tile neighbours of the G layers
                    const int k = gi * G + kk;
                    if (k >= nz) break;
                    if (!ZERO) {
                        const double* src = uin + (int64_t)k * ld;
                        if (lane < hcount) ptx::cp_async8(st + SL.hu + kk * HS + lane, src + h0);
                        if (lane + 32 < hcount) ptx::cp_async8(st + SL.hu + kk * HS + lane + 32, src + h1);
                    }
                    if (PROLONG) {
                        const double* srcc = uc + (int64_t)k * ldc;
                        if (lane < hcount) ptx::cp_async8(st + SL.huc + kk * kHaloMax + lane, srcc + (h0 >> 2));
                        if (lane + 32 < hcount)
                            ptx::cp_async8(st + SL.huc + kk * kHaloMax + lane + 32, srcc + (h1 >> 2));
                    }
                    if (MF) {
                        const double* srcl = op.lam + (int64_t)k * ld;
                        if (lane < hcount) ptx::cp_async8(st + SL.hlam + kk * kHaloMax + lane, srcl + h0);
                        if (lane + 32 < hcount) ptx::cp_async8(st + SL.hlam + kk * kHaloMax + lane + 32, srcl + h1);
                    }
                }
                ptx::cp_async_arrive(&full[s]);
            }
            __syncwarp();
            if (lane == 0) {
                if (pf_groups > 0 && gi + pf_groups < ngroups) {   // L2 prefetch a few stages ahead
                    const int gp = gi + pf_groups;
                    if (MF)
                        ptx::tma_prefetch_2d(&maps.lam, x, gp * G);
                    else if (NBP == 1)
                        ptx::tma_prefetch_2d(&maps.bands, x, gp * G);
                    else
                        ptx::tma_prefetch_3d(&maps.bands, x, gp * G, 0);
                    ptx::tma_prefetch_2d(&maps.b, x, gp * G);
                    if (!ZERO) ptx::tma_prefetch_2d(&maps.uf, x, gp * G);
                }
                int nl = nz - gi * G;
                nl = nl < G ? nl : G;
                ptx::mbar_arrive_expect_tx(&full[s], fwd_bytes + (EH && kProbeEdge ? (uint32_t)nl * ebytes : 0u));
                if (EH && kProbeEdge)
                    for (int kk = 0; kk < nl; ++kk)
                        ptx::bulk_g2s(st + SL.eh + kk * kEdgeRow, et.H + (int64_t)(gi * G + kk) * et.ldE + ee0,
                                      ebytes, &full[s]);
                if (MF)
                    ptx::tma_load_2d_hint(st + SL.op, &maps.lam, x, gi * G, &full[s], pol_stream);
                else if (NBP == 1)
                    ptx::tma_load_2d_hint(st + SL.op, &maps.bands, x, gi * G, &full[s], pol_stream);
                else
                    ptx::tma_load_3d_hint(st + SL.op, &maps.bands, x, gi * G, 0, &full[s], pol_stream);
                ptx::tma_load_2d_hint(st + SL.b, &maps.b, x, gi * G, &full[s], DOT ? pol_keep : pol_stream);
                if (!ZERO) ptx::tma_load_2d_hint(st + SL.u, &maps.uf, x, gi * G, &full[s], pol_keep);
                if (PROLONG) ptx::tma_load_2d_hint(st + SL.uc, &maps.ucf, xc, gi * G, &full[s], pol_keep);
            }
            advance();
        };
        // one backward stage: the u rows (u_c, b) of chunk m of the tile at column x, again
        auto bwd_stage = [&](int tile, int m) {
            const int x = tile * kTile, xc = x / 4;
#ifdef HMG_TIMING
            long long q0 = clock64();
#endif
            ptx::mbar_wait(&empty[s], phase ^ 1u);
            ST_TAG_SET();
#ifdef HMG_TIMING
            pw += clock64() - q0;
#endif
            double* st = stages + (size_t)s * SL.stage;
            if (lane == 0 && !kProbeBwd) ptx::mbar_arrive(&full[s]);
            if (lane == 0 && kProbeBwd) {
                ptx::mbar_arrive_expect_tx(&full[s], bwd_bytes);
                ptx::tma_load_2d_hint(st, &maps.ub, x, m * kBack, &full[s], pol_stream);
                if (PROLONG) ptx::tma_load_2d_hint(st + kBack * kTile, &maps.ucb, xc, m * kBack, &full[s], pol_stream);
                if (DOT) ptx::tma_load_2d_hint(st + kBack * kTile, &maps.bb, x, m * kBack, &full[s], pol_stream);
            }
            advance();
        };
        if (IL) {
            for (int p = 0; p <= ntc; ++p) {
                const bool hasF = p < ntc, hasB = p > 0;
                const int tile = (int)blockIdx.x + p * (int)gridDim.x;
                const int32_t ee0 = EH && hasF ? et.e0[tile] : 0;
                const uint32_t ebytes = EH && hasF ? (uint32_t)(sizeof(double) * et.ne[tile]) : 0u;
                for (int ch = 0; ch < nchunks; ++ch) {
                    if (hasB) bwd_stage(tile - (int)gridDim.x, nchunks - 1 - ch);
                    if (!hasF) continue;
                    const int g1 = (ch + 1) * kGpc < ngroups ? (ch + 1) * kGpc : ngroups;
                    for (int gi = ch * kGpc; gi < g1; ++gi) fwd_stage(tile, gi, 0, 0, 0, ee0, ebytes);
                }
            }
        } else {
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int hcount = HALO && !SPLIT ? th.count[tile] : 0;
                const int32_t h0 = lane < hcount ? th.cells[tile * kHaloMax + lane] : 0;
                const int32_t h1 = lane + 32 < hcount ? th.cells[tile * kHaloMax + lane + 32] : 0;
                // edge store: the tile's contiguous edge range (its gathered edges: gather warp)
                const int32_t ee0 = EH ? et.e0[tile] : 0;
                const uint32_t ebytes = EH ? (uint32_t)(sizeof(double) * et.ne[tile]) : 0u;
                for (int gi = 0; gi < ngroups; ++gi) fwd_stage(tile, gi, hcount, h0, h1, ee0, ebytes);
                for (int m = nchunks - 1; m >= 0; --m) bwd_stage(tile, m);   // u rows again for the back substitution
            }
        }
#ifdef HMG_TIMING
        if (blockIdx.x == 0 && lane == 0) {
            g_st_timing[8] = clock64() - p0;
            g_st_timing[9] = pw;
            g_st_timing[10] = pn;
            g_st_timing[11] = ph;
        }
#endif
    } else {
        // ======================= consumer warps: one column per thread =======================
        const int j = threadIdx.x;
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        const int nzp = nchunks * kBack;           // layers rounded up to whole chunks (>= nz)
        const uint32_t gcol = 2u * (uint32_t)(ZERO ? nz : nzp);   // g at TMEM columns gcol + 2 slot, z at 2 slot
        const double ydz = MF ? div_recip(op.dz) : 0.0;   // exact redo only
        int pend = -1;                                     // TSTORE: slot whose store may still read it
        int s = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        };
#ifdef HMG_TIMING
        tt0 = clock64();
#endif
        // IL schedule.  Pass p runs tile p's forward elimination and, chunk by
        // chunk (8 layers, top-down), tile p - 1's back substitution: before the
        // forward stages of layers 8c .. 8c+7, the back substitution of chunk
        // nchunks-1-c.  The (z, g) of layer k sit in TMEM slot k for even passes
        // and nzp - 1 - k for odd ones, so the forward pass writes each slot just
        // after the back substitution of the previous tile has read it: two
        // tiles' recurrences share one tile's TMEM, the loads stay continuous
        // through the back substitution, and its u' rows are written while the
        // next tile streams in.
        int btile = 0;
        bool bvalid = false, bodd = false;
        double bdl = 0.0;
        // the last pass has only back-substitution chunks: there thread 0 releases
        // a chunk's slot once the NEXT chunk's store is issued (the stores overlap
        // instead of each waiting for its copy to read the stage)
        bool blazy = false;
        int bpend = -1;
        const int mtop_il = nchunks - 1;
        auto bwd_chunk = [&](int m) {
            const int k0 = m * kBack;
            const int kt = (k0 + kBack - 1 < nz - 1) ? k0 + kBack - 1 : nz - 1;
            const uint32_t sb = bodd ? (uint32_t)(nzp - kBack - k0) : (uint32_t)k0;
            uint32_t zr[16], gr[16];
            ptx::tmem_ld_8f64(tl + 2u * sb, zr);
            ptx::tmem_ld_8f64(tl + gcol + 2u * sb, gr);
            ptx::mbar_wait(&full[s], phase);
            ST_TAG_CHECK();
            double* su = stages + (size_t)s * SL.stage;
            ptx::tmem_wait_ld();
            double zv[kBack], gv[kBack];                   // by layer k0 + i
#pragma unroll
            for (int i = 0; i < kBack; ++i) {
                const int q = bodd ? kBack - 1 - i : i;
                zv[i] = ptx::f64_from(zr[2 * q], zr[2 * q + 1]);
                gv[i] = ptx::f64_from(gr[2 * q], gr[2 * q + 1]);
            }
            auto finish = [&](int i) {
                double uo = su[i * kTile + j];
                if (PROLONG) uo = uo + su[kBack * kTile + i * (kTile / 4) + (j >> 2)];
                const double o = uo + omega * bdl;
                su[i * kTile + j] = o;
                if (DOT && bvalid) dotacc = dotacc + su[kBack * kTile + i * kTile + j] * o;
            };
            if (m < mtop_il) {                         // full chunk, every layer below nz - 1
#pragma unroll
                for (int i = kBack - 1; i >= 0; --i) {
                    bdl = zv[i] - gv[i] * bdl;
                    finish(i);
                }
            } else {
#pragma unroll
                for (int i = kBack - 1; i >= 0; --i) {
                    const int k = k0 + i;
                    if (k > kt) continue;
                    bdl = (k == nz - 1) ? zv[i] : zv[i] - gv[i] * bdl;
                    finish(i);
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::named_bar_sync(1, kTile);
            if (warp == 0) {
                if (lane == 0) {
                    ptx::tma_store_2d(&maps.uo, btile * kTile, k0, su);
                    ptx::bulk_commit_group();
                    if (!blazy) {
                        ptx::bulk_wait_group_read<0>();
                        ptx::mbar_arrive(&empty[s]);
                    } else {
                        if (bpend >= 0) {
                            ptx::bulk_wait_group_read<1>();
                            ptx::mbar_arrive(&empty[bpend]);
                        }
                        if (m == 0) {
                            ptx::bulk_wait_group_read<0>();
                            ptx::mbar_arrive(&empty[s]);
                        }
                    }
                }
                bpend = (blazy && m != 0) ? s : -1;
                __syncwarp();
            } else {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
            }
            advance();
        };
        const int npass = IL ? ntc + 1 : ntc;
        for (int pass = 0; pass < npass; ++pass) {
            const int tile = (int)blockIdx.x + pass * (int)gridDim.x;
            const bool hasF = pass < ntc, hasB = IL && pass > 0;
            const bool fodd = IL && (pass & 1);
            blazy = !hasF;
            // TMEM slot of layer k of this pass's tile
            auto fslot = [&](int k) -> uint32_t { return (uint32_t)(fodd ? nzp - 1 - k : k); };
#ifdef HMG_TIMING
            ++ntl;
            tfw0 = clock64();
#endif
            const int64_t c = (int64_t)tile * kTile + j;
            const bool valid = hasF && c < L.n;
            const int64_t cv = valid ? c : L.n - 1;
            int l0 = 0, l1 = 0, l2 = 0;
            if (HALO && hasF) {
                const uint32_t loc = th.loc[cv];
                l0 = loc & 0xff;
                l1 = (loc >> 8) & 0xff;
                l2 = (loc >> 16) & 0xff;
            }
#ifdef HMG_PROBE_NOCONFLICT
            l0 = j;
            l1 = (j + 1) & 127;
            l2 = (j + 2) & 127;
#endif
            // FLAT: stage offsets of the three neighbours' u at row 0 (tile row or halo row)
            HMG_DCHECK(l0 < kTile + kHaloMax && l1 < kTile + kHaloMax && l2 < kTile + kHaloMax);
            const int no0 = l0 < kTile ? SL.u + l0 : SL.hu + (l0 - kTile);
            const int no1 = l1 < kTile ? SL.u + l1 : SL.hu + (l1 - kTile);
            const int no2 = l2 < kTile ? SL.u + l2 : SL.hu + (l2 - kTile);
            // PROLONG: offsets of the neighbours' u_c (parent in the tile's rows, or halo row)
            const int nc0 = l0 < kTile ? SL.uc + (l0 >> 2) : SL.huc + (l0 - kTile);
            const int nc1 = l1 < kTile ? SL.uc + (l1 >> 2) : SL.huc + (l1 - kTile);
            const int nc2 = l2 < kTile ? SL.uc + (l2 >> 2) : SL.huc + (l2 - kTile);
            int eo0 = 0, eo1 = 0, eo2 = 0;                 // the faces' offsets in an edge row
            if (EH && hasF) {
                const uint32_t el = et.loc[cv];
                eo0 = el & 0xff;
                eo1 = (el >> 8) & 0xff;
                eo2 = (el >> 16) & 0xff;
            }
#ifdef HMG_PROBE_NOCONFLICT   // probe build only: lane-aligned gathers (wrong results, same instructions)
            eo0 = j;
            eo1 = j + 128;
            eo2 = (j + 64) & 255;
#endif
            HMG_DCHECK(eo0 < kEdgeRow && eo1 < kEdgeRow && eo2 < kEdgeRow);
            ColumnGeom cg{};
            const double vol = ND ? op.geom[cv] * op.dz : 0.0;   // k_assemble's prism volume

            // Thomas forward elimination, reading R6 order (as k_sweep_tc's `layer`)
            double um = 0.0, Um = 0.0, gprev = 0.0, zprev = 0.0, vdn = 0.0;
            bool ok = true, slow = false;
            auto layer = [&](int k, double Dk, double Uk, double r, bool exact) {
                const double num = (k == 0) ? r : r - Um * zprev;
                const bool has_g = k < nz - 1;
                const double den = (k == 0) ? Dk : Dk - Um * gprev;
                double z, g = 0.0;
                if (exact) {
                    z = num / den;
                    if (has_g) g = Uk / den;
                } else {
                    const double y = div_recip(den);
                    z = div_fast_z(num, den, y, slow);
                    if (has_g) g = div_fast(Uk, den, y, slow);
                }
                ok = ok && pivot_ok(den);
                ptx::tmem_st_f64(tl + 2u * fslot(k), z);
                if (has_g) ptx::tmem_st_f64(tl + gcol + 2u * fslot(k), g);
                zprev = z;
                gprev = g;
            };
            for (int ch = 0; ch < (IL ? nchunks : 1); ++ch) {
            if (hasB) bwd_chunk(nchunks - 1 - ch);
            const int ga = IL ? ch * kGpc : 0;
            const int gb = !hasF ? ga : !IL ? ngroups : ((ch + 1) * kGpc < ngroups ? (ch + 1) * kGpc : ngroups);
            for (int gi = ga; gi < gb; ++gi, advance()) {
#ifdef HMG_TIMING
                long long w0 = clock64();
#endif
                ptx::mbar_wait(MF ? &mid[s] : &full[s], phase);
                ST_TAG_CHECK();
#ifdef HMG_TIMING
                wf += clock64() - w0;
#endif
                const double* st = stages + (size_t)s * SL.stage;
                const double* su = st + SL.u;
                const double* suc = st + SL.uc;
                const double* hu = st + SL.hu;
                const double* huc = st + SL.huc;
                // u value (with the fused prolongation) of local slot l at stage row kk
                auto UV = [&](int kk, int l) -> double {
                    double v = su[kk * kTile + l];
                    if (PROLONG) v = v + suc[kk * kUcRow + (l >> 2)];
                    return v;
                };
                auto NBR = [&](int kk, int l) -> double {
                    if (l < kTile) return UV(kk, l);
                    double v = hu[kk * HS + l - kTile];
                    if (PROLONG) v = v + huc[kk * kHaloMax + l - kTile];
                    return v;
                };
                auto NBRF = [&](int kk, int q, int l) -> double {   // neighbour q (slot l) of the column
                    if (FLAT) {
                        double v = st[(q == 0 ? no0 : q == 1 ? no1 : no2) + kk * kTile];
                        if (PROLONG) v = v + st[(q == 0 ? nc0 : q == 1 ? nc1 : nc2) + kk * kUcRow];
                        return v;
                    }
                    return NBR(kk, l);
                };
                // One layer: residual row (reading R5 order) and Thomas step.  IN
                // (interior: 0 < k < nz - 1) drops every boundary test.
                auto step = [&](int kk, auto interior) {
                    constexpr bool IN = decltype(interior)::value;
                    const int k = gi * G + kk;
                    const double* sr = st + SL.band + kk * kTile + j;
                    constexpr int pu = ND ? 0 : 1;     // plane of U in the stage's band rows
                    const double Uk = sr[pu * G * kTile];
                    const double* er = st + SL.eh + kk * kEdgeRow;
                    const double H0 = EH ? er[eo0] : sr[(pu + 1) * G * kTile];
                    const double H1 = EH ? er[eo1] : sr[(pu + 2) * G * kTile];
                    const double H2 = EH ? er[eo2] : sr[(pu + 3) * G * kTile];
                    double Dk;
                    if (ND) {
                        // k_assemble's diagonal: vol + V_dn + V_up + H0 + H1 + H2 with the
                        // stored U = -V_up, H_j = -(coupling): x + (-y) is x - y exactly
                        double d = vol;
                        if (IN || k > 0) d = d - Um;
                        if (IN || k < nz - 1) d = d - Uk;
                        d = d - H0;
                        d = d - H1;
                        d = d - H2;
                        Dk = d;
                    } else {
                        Dk = sr[0];
                    }
                    const double bk = st[SL.b + kk * kTile + j];
                    double r;
                    if (ZERO) {
                        r = bk;
                    } else {
                        const double uk = UV(kk, j);
                        double up = 0.0;
                        if (IN || k < nz - 1) up = UV(kk + 1, j);
                        double acc = Dk * uk;
                        if (IN || k > 0) acc = acc + Um * um;
                        if (IN || k < nz - 1) acc = acc + Uk * up;
                        acc = acc + H0 * NBRF(kk, 0, l0);
                        acc = acc + H1 * NBRF(kk, 1, l1);
                        acc = acc + H2 * NBRF(kk, 2, l2);
                        r = bk - acc;
#if defined(HMG_PROBE_NORES) || defined(HMG_PROBE_NOCHAIN)
                        r = bk;   // probe build only: no residual work in the consumers (wrong results)
#endif
                        um = uk;
                    }
#ifdef HMG_PROBE_NOCHAIN
                    if (IN) {   // probe build only: no Thomas chain (wrong results, same data movement)
                        ptx::tmem_st_f64(tl + 2u * fslot(k), r);
                        ptx::tmem_st_f64(tl + gcol + 2u * fslot(k), Uk);
                        zprev = r;
                        gprev = Uk;
                    } else
#endif
                    if (IN) {
                        const double num = r - Um * zprev;
                        const double den = Dk - Um * gprev;
                        const double y = div_recip(den);
                        const double z = div_fast_z(num, den, y, slow);
                        // CHK = false: pivots and the fast-path exactness of every
                        // g_k were established at build time (k_pivot_check)
                        const double g = CHK ? div_fast(Uk, den, y, slow) : div_fast_unchecked(Uk, den, y);
                        if (CHK) ok = ok && pivot_ok(den);
                        ptx::tmem_st_f64(tl + 2u * fslot(k), z);
                        ptx::tmem_st_f64(tl + gcol + 2u * fslot(k), g);
                        zprev = z;
                        gprev = g;
                    } else {
                        layer(k, Dk, Uk, r, false);
                    }
                    Um = Uk;
                };
                if (gi > 0 && (gi + 1) * G < nz) {     // interior stage: no layer touches a boundary
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
            }   // chunks
#ifdef HMG_TIMING
            tfw += clock64() - tfw0;
            tfw0 = clock64();
#endif
            // Rare: a quotient left the fast path's exact range.  The warp redoes
            // its columns' forward pass from global memory with '/'.
#ifdef HMG_PROBE_NOREDO
            if (false) {
#else
            if (__any_sync(0xffffffffu, slow && valid)) {   // (valid implies this pass has a forward tile)
#endif
                const int32_t g0 = L.nbr[cv], g1 = L.nbr[ld + cv], g2 = L.nbr[2 * ld + cv];
                auto GU = [&](int kk, int64_t cell) -> double {
                    double v = uin[(int64_t)kk * ld + cell];
                    if (PROLONG) v = v + uc[(int64_t)kk * ldc + (cell >> 2)];
                    return v;
                };
                um = Um = gprev = zprev = vdn = 0.0;
                bool dummy = false;
                if (MF) cg = column_geom(op.geom, ld, cv, op.w2, op.dz);
                double uk = ZERO ? 0.0 : GU(0, cv);
                for (int k = 0; k < nz; ++k) {
                    const int64_t i = (int64_t)k * ld + cv;
                    double Dk, Uk, H0, H1, H2;
                    if (MF) {
                        const double lk = op.lam[i];
                        double vup = 0.0;
                        if (k < nz - 1) vup = mf_vcoup<true>(cg, lk, op.lam[i + ld], op.dz, ydz, dummy);
                        const double hc0 = mf_hcoup<true>(cg, 0, lk, op.lam[(int64_t)k * ld + g0], dummy);
                        const double hc1 = mf_hcoup<true>(cg, 1, lk, op.lam[(int64_t)k * ld + g1], dummy);
                        const double hc2 = mf_hcoup<true>(cg, 2, lk, op.lam[(int64_t)k * ld + g2], dummy);
                        Dk = mf_diag(cg, k, nz, vdn, vup, hc0, hc1, hc2);
                        Uk = (k < nz - 1) ? -vup : 0.0;
                        H0 = -hc0;
                        H1 = -hc1;
                        H2 = -hc2;
                        vdn = vup;
                    } else {
                        Dk = L.D[i];
                        Uk = L.U[i];
                        H0 = L.H0[i];
                        H1 = L.H1[i];
                        H2 = L.H2[i];
                    }
                    double r;
                    if (ZERO) {
                        r = bvec[i];
                    } else {
                        double up = 0.0;
                        if (k < nz - 1) up = GU(k + 1, cv);
                        double acc = Dk * uk;
                        if (k > 0) acc = acc + Um * um;
                        if (k < nz - 1) acc = acc + Uk * up;
                        acc = acc + H0 * GU(k, g0);
                        acc = acc + H1 * GU(k, g1);
                        acc = acc + H2 * GU(k, g2);
                        r = bvec[i] - acc;
                        um = uk;
                        uk = up;
                    }
                    layer(k, Dk, Uk, r, true);
                    Um = Uk;
                }
            }
            if (valid && !ok) atomicMin(bad, ((unsigned long long)ref << 40) | (unsigned long long)c);
            ptx::tmem_wait_st();
            if (IL) {                                  // this tile's back substitution: next pass
                btile = tile;
                bvalid = valid;
                bodd = fodd;
                bdl = 0.0;
                continue;
            }
#ifdef HMG_TIMING
            tws += clock64() - tfw0;
#endif

            // back substitution from the top: delta_{nz-1} = z_{nz-1},
            // delta_k = z_k - g_k delta_{k+1}; u' = u_old + omega delta (zero guess: omega delta)
            // The (z, g) of the next chunk down are loaded from TMEM while the
            // current chunk is computed (tcgen05.ld is asynchronous; only the top
            // chunk, possibly partial, is loaded synchronously).
            double dl = 0.0;
            const int mtop = (nz + kBack - 1) / kBack - 1;
            uint32_t zr[16], gr[16], zn[16], gn[16];
            {
                const int k0 = mtop * kBack;
                const int kt = nz - 1;
                if (kt - k0 == kBack - 1) {
                    ptx::tmem_ld_8f64(tl + 2u * (uint32_t)k0, zr);
                    ptx::tmem_ld_8f64(tl + gcol + 2u * (uint32_t)k0, gr);
                } else {
#pragma unroll
                    for (int i = 0; i < kBack; ++i) {      // partial top chunk
                        if (i > kt - k0) break;
                        uint32_t z2[2], g2[2];
                        ptx::tmem_ld_1f64(tl + 2u * (uint32_t)(k0 + i), z2);
                        ptx::tmem_ld_1f64(tl + gcol + 2u * (uint32_t)(k0 + i), g2);
                        ptx::tmem_wait_ld();
                        zr[2 * i] = z2[0];
                        zr[2 * i + 1] = z2[1];
                        gr[2 * i] = g2[0];
                        gr[2 * i + 1] = g2[1];
                    }
                }
                ptx::tmem_wait_ld();
            }
            double* const uo_row = uout + c;               // column c of row 0 (rows at stride ld)
            for (int m = mtop; m >= 0; --m) {
                const int k0 = m * kBack;
                const int kt = (k0 + kBack - 1 < nz - 1) ? k0 + kBack - 1 : nz - 1;   // top layer of the chunk
                if (m > 0) {                               // chunks below the top are full
                    ptx::tmem_ld_8f64(tl + 2u * (uint32_t)(k0 - kBack), zn);
                    ptx::tmem_ld_8f64(tl + gcol + 2u * (uint32_t)(k0 - kBack), gn);
                }
                double* su = nullptr;
                if (!ZERO) {
#ifdef HMG_TIMING
                    long long w0 = clock64();
#endif
                    ptx::mbar_wait(MF ? &mid[s] : &full[s], phase);
                    ST_TAG_CHECK();
#ifdef HMG_TIMING
                    wb += clock64() - w0;
#endif
                    su = stages + (size_t)s * SL.stage;
                }
                // the chunk's results: delta chain first (branch-free below the top
                // chunk), then u' = u_old + omega delta, the store and the fused dot
                auto finish = [&](int i, int k) {
                    double o;
                    if (ZERO) {
                        o = omega * dl;
                    } else {
                        double uo = su[i * kTile + j];
                        if (PROLONG) uo = uo + su[kBack * kTile + i * (kTile / 4) + (j >> 2)];
                        o = uo + omega * dl;
                    }
                    if (TSTORE) su[i * kTile + j] = o;     // u_old's place in the stage
                    if (valid) {
                        if (!TSTORE) uo_row[(int64_t)k * ld] = o;
                        if (DOT) dotacc = dotacc + su[kBack * kTile + i * kTile + j] * o;
                    }
                };
                if (m < mtop) {                            // full chunk, every layer below nz - 1
#pragma unroll
                    for (int i = kBack - 1; i >= 0; --i) {
                        dl = ptx::f64_from(zr[2 * i], zr[2 * i + 1]) - ptx::f64_from(gr[2 * i], gr[2 * i + 1]) * dl;
                        finish(i, k0 + i);
                    }
                } else {
#pragma unroll
                    for (int i = kBack - 1; i >= 0; --i) {
                        const int k = k0 + i;
                        if (k > kt) continue;
                        const double zk = ptx::f64_from(zr[2 * i], zr[2 * i + 1]);
                        if (k == nz - 1)
                            dl = zk;
                        else
                            dl = zk - ptx::f64_from(gr[2 * i], gr[2 * i + 1]) * dl;
                        finish(i, k);
                    }
                }
                if (TSTORE) {
                    // the chunk's 8 u' rows go out as one TMA box from the stage (clipped
                    // to the level's n columns and nz rows); thread 0 releases the slot
                    // once the copy has read it -- the previous chunk's here, this tile's
                    // last before the next tile's forward stages need the ring
                    ptx::fence_proxy_async_smem();
                    ptx::named_bar_sync(1, kTile);
                    if (warp == 0) {
                        if (lane == 0) {
                            ptx::tma_store_2d(&maps.uo, tile * kTile, k0, su);
                            ptx::bulk_commit_group();
                            if (pend >= 0) {
                                ptx::bulk_wait_group_read<1>();
                                ptx::mbar_arrive(&empty[pend]);
                            }
                            if (m == 0) {
                                ptx::bulk_wait_group_read<0>();
                                ptx::mbar_arrive(&empty[s]);
                            }
                        }
                        pend = m == 0 ? -1 : s;
                        __syncwarp();
                    } else {
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&empty[s]);
                    }
                    advance();
                } else if (!ZERO) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty[s]);
                    advance();
                }
                if (m > 0) {
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        zr[i] = zn[i];
                        gr[i] = gn[i];
                    }
                }
            }
#ifdef HMG_TIMING
            tbk += clock64() - tfw0;
#endif
        }
        if (TSTORE && threadIdx.x == 0) ptx::bulk_wait_group<0>();   // the u' rows are written before exit
    }
#ifdef HMG_TIMING
    if (warp < kConsumerWarps && blockIdx.x == 0 && threadIdx.x == 0) {
        g_st_timing[0] = clock64() - tt0;
        g_st_timing[1] = wf;
        g_st_timing[2] = wb;
        g_st_timing[3] = ntl;
        g_st_timing[4] = tfw;
        g_st_timing[5] = tbk;
        g_st_timing[6] = tws;
    }
#endif
    if (DOT) {   // fixed-order CTA reduction of <b, u'> (producer / coupling warps contribute 0)
        for (int off = 16; off > 0; off >>= 1) dotacc = dotacc + __shfl_down_sync(0xffffffffu, dotacc, off);
        if (lane == 0 && warp < kThreads / 32) dred[warp] = dotacc;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (DOT && threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t = t + dred[w];
        partial[blockIdx.x] = t;
    }
    if (warp == 0) ptx::tmem_dealloc(tbase, tmem_cols);
    if (DOT) fin_fused(fin, partial);   // the last CTA: beta, rho from <r, z> (fused finalize)
#ifdef HMG_TIMING
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_cta_ns[2 * blockIdx.x + 1] = t;
    }
#endif
}

uint32_t st_tmem_cols(int nz) {
    uint32_t need = 4u * (uint32_t)nz, c = 32;
    while (c < need) c <<= 1;
    return c;
}

template <bool Z, bool P, bool M, int G, bool CK = true, bool DOT = false, bool EH = false>
int launch_st(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
              double* uout, double omega, cudaStream_t s) {
    const int nz = H.nz;
    const uint32_t cols = st_tmem_cols(nz);
    constexpr StLayout SL = st_layout(Z, P, M, G, DOT, EH);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
    const unsigned ntiles = (unsigned)((L.n + kTile - 1) / kTile);
    const bool two = cols <= 256;                  // two CTAs' Thomas state fit one SM's tensor memory
    const size_t budget = two ? 110 * 1024 : 220 * 1024;
    int S = (int)((budget - 1024) / (sizeof(double) * SL.stage));
    S = S < 2 ? 2 : (S > 32 ? 32 : S);
    size_t smem = 1024 + sizeof(double) * (size_t)S * SL.stage;
    const size_t floor_smem = two ? 80 * 1024 : 120 * 1024;   // never a third CTA per SM (TMEM)
    if (smem < floor_smem) smem = floor_smem;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sweep_st<Z, P, M, G, CK, DOT, EH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             220 * 1024);
        attr = true;
    }
    StMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const LevelView V = L.view(nz);
    if (M)
        maps.lam = make_tensor_map(L.lam, L.ld, nz, kTile, G + 1, 1);
    else
        maps.bands = make_tensor_map(!Z ? V.U : V.D, L.ld, nz, kTile, G, st_band_planes(Z, M, EH));
    maps.b = make_tensor_map(b, L.ld, nz, kTile, G, 1);
    if (!Z) {
        maps.uf = make_tensor_map(uin, L.ld, nz, kTile, G + 1, 1);
        maps.ub = make_tensor_map(uin, L.ld, nz, kTile, kBack, 1);
    }
    int64_t ldc = 0;
    if (P) {
        const DevLevel& C = H.lev[L.ref - 1];
        ldc = C.ld;
        maps.ucf = make_tensor_map(uc, C.ld, nz, kUcRow, G + 1, 1);
        maps.ucb = make_tensor_map(uc, C.ld, nz, kTile / 4, kBack, 1);
    }
    if (DOT) maps.bb = make_tensor_map(b, L.ld, nz, kTile, kBack, 1);
    if (!Z) maps.uo = make_store_map(uout, L.ld, L.n, nz, kTile, kBack);
    const StOp op{L.lam, L.geom, H.w2, H.dz};
    // persistent grid: as many rounds of tiles as the resident CTAs need, with the
    // tiles dealt evenly (ref 6: 640 tiles -> 214 CTAs x 3 instead of 296 CTAs
    // with a last round 16% full)
    const unsigned cap = (unsigned)((two ? 2 : 1) * sms);
    const unsigned rounds = (ntiles + cap - 1) / cap;
    const unsigned grid = (ntiles + rounds - 1) / rounds;
    launch_pdl(H, k_sweep_st<Z, P, M, G, CK, DOT, EH>, dim3(grid), dim3(st_threads(Z, M)), smem, s, maps, V,
               op, L.halo, L.edge, b, uin, uc, ldc, uout, omega, L.ref, &H.scal->bad, S, cols, H.l2_prefetch_groups,
               H.partials, DOT ? fin_take(H) : FinArgs());
    return (int)grid;
}

#ifdef HMG_TIMING
}  // namespace
extern "C" void hmg_debug_st_timing(long long* out) { cudaMemcpyFromSymbol(out, g_st_timing, sizeof(long long) * 12); }
extern "C" void hmg_debug_st_cta(unsigned long long* ns, unsigned* sm) {
    cudaMemcpyFromSymbol(ns, g_cta_ns, sizeof(unsigned long long) * 2048);
    cudaMemcpyFromSymbol(sm, g_cta_sm, sizeof(unsigned) * 1024);
}
namespace {
#endif

}  // namespace

// The sweep reads the edge store only where two CTAs share an SM (nz <= 64):
// with one CTA per SM (nz = 128) its consumers are the bottleneck and the
// extra copies made the C4 sweep 25% slower (measured); the apply uses it always.
bool sweep_edge_store(const Hierarchy& H, const DevLevel& L) {
    return L.edge.H != nullptr && st_tmem_cols(H.nz) <= 256;
}

bool sweep_st_supported(const Hierarchy& H, const DevLevel& L) {
    return H.use_st_sweep && H.nz <= 128 && L.halo.loc != nullptr;
}

int launch_sweep_st_dot(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, double* uout,
                        double omega, cudaStream_t s) {
    int n = 0;
    try {
        const bool eh = sweep_edge_store(H, L);
        if (L.g_safe && eh)
            n = launch_st<false, false, false, 2, false, true, true>(H, L, b, uin, nullptr, uout, omega, s);
        else if (L.g_safe)
            n = launch_st<false, false, false, 2, false, true>(H, L, b, uin, nullptr, uout, omega, s);
        else if (eh)
            n = launch_st<false, false, false, 2, true, true, true>(H, L, b, uin, nullptr, uout, omega, s);
        else
            n = launch_st<false, false, false, 2, true, true>(H, L, b, uin, nullptr, uout, omega, s);
    } catch (const std::exception& e) {
        g_launch_error = std::string("sweep launch: ") + e.what();
    }
    ++H.launches;
    return n;
}

void launch_sweep_st(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                     double* uout, double omega, cudaStream_t s) {
    try {
        if (H.matrix_free && L.mf_safe && L.g_safe) {
            if (!uin)
                launch_st<true, false, true, 2, false>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_st<false, true, true, 2, false>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_st<false, false, true, 2, false>(H, L, b, uin, nullptr, uout, omega, s);
        } else if (H.matrix_free) {
            if (!uin)
                launch_st<true, false, true, 2>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_st<false, true, true, 2>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_st<false, false, true, 2>(H, L, b, uin, nullptr, uout, omega, s);
        } else if (uin && sweep_edge_store(H, L)) {   // edge-deduplicated couplings
            if (L.g_safe && uc)
                launch_st<false, true, false, 2, false, false, true>(H, L, b, uin, uc, uout, omega, s);
            else if (L.g_safe)
                launch_st<false, false, false, HMG_ST_G, false, false, true>(H, L, b, uin, nullptr, uout, omega, s);
            else if (uc)
                launch_st<false, true, false, 2, true, false, true>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_st<false, false, false, 2, true, false, true>(H, L, b, uin, nullptr, uout, omega, s);
        } else if (L.g_safe) {
            if (!uin)
                launch_st<true, false, false, 2, false>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_st<false, true, false, 2, false>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_st<false, false, false, 2, false>(H, L, b, uin, nullptr, uout, omega, s);
        } else {
            if (!uin)
                launch_st<true, false, false, 2>(H, L, b, nullptr, nullptr, uout, omega, s);
            else if (uc)
                launch_st<false, true, false, 2>(H, L, b, uin, uc, uout, omega, s);
            else
                launch_st<false, false, false, 2>(H, L, b, uin, nullptr, uout, omega, s);
        }
    } catch (const std::exception& e) {
        g_launch_error = std::string("sweep launch: ") + e.what();
    }
    ++H.launches;
}

}  // namespace hmg
