// Internal types of the CUDA path (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hmg.h"
#include "nccl_dyn.h"

namespace hmg {

constexpr int kMaxLayers = 256;   // Thomas state for a column lives in shared memory
constexpr int kMaxRef = 10;
// Checked builds (-DHMG_CHECKED, tools/checked_probe.py; never the product
// library): device-side bounds checks on gathered indices and a sequence tag
// on every ring stage (the producer writes the stage's number, the consumers
// check it) -- the stand-in for compute-sanitizer, which the GPU pool refuses.
#ifdef HMG_CHECKED
#define HMG_DCHECK(c)                                                                              \
    do {                                                                                           \
        if (!(c)) {                                                                                \
            printf("HMG_CHECKED: %s failed (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define HMG_DCHECK(c) \
    do {              \
    } while (0)
#endif

constexpr int kSweepTile = 128;   // columns per CTA of the TMA/TMEM sweep (sweep_tc.cu)
constexpr int kHaloMax = 64;
constexpr int64_t kFactMaxCells = 148 * 128;
constexpr int64_t kCoopMaxCells = 5120;   // default cooperative coarse tail: levels up to this size (ref 4)
constexpr int kSmallTile = 32;    // columns per CTA of the small-level sweep (sweep_small.cu)
constexpr int kSmallHaloMax = 32; // off-tile neighbours per 32-cell tile (24 observed)  // levels up to this size stream precomputed Thomas pivots      // max off-tile neighbour cells per tile (51 observed at ref >= 2)

// Per-level tile halo for the streamed sweep: for tile t (cells
// [t*kSweepTile, (t+1)*kSweepTile)), the sorted distinct neighbour cells
// outside the tile, and per cell the 3 neighbours' local slots packed in
// bytes (slot < kSweepTile: in-tile offset; else kSweepTile + halo index).
struct TileHalo {
    const int32_t* cells = nullptr;   // [ntiles][kHaloMax]
    const int32_t* count = nullptr;   // [ntiles]
    const uint32_t* loc = nullptr;    // [ld]
};

// Edge-deduplicated horizontal couplings for the streamed sweep (each face
// coupling stored once, 1.5 per cell instead of 3).  Edges are numbered by
// their lower cell, then its slot, so the edges owned by a 128-cell tile are
// one contiguous range (176-216 at ref >= 5; streamed with one bulk copy per
// layer); the <= 32 faces whose lower cell lies before the tile are gathered.
constexpr int kEdgeRange = 224;   // contiguous part of a stage row (doubles)
constexpr int kEdgeHalo = 32;     // gathered part
constexpr int kEdgeRow = kEdgeRange + kEdgeHalo;
struct EdgeTiles {
    const double* H = nullptr;        // [nz][ldE] coupling of each edge and layer
    int64_t ldE = 0;
    const int32_t* e0 = nullptr;      // [ntiles] first edge of the tile's range (even)
    const int32_t* ne = nullptr;      // [ntiles] edges per layer to copy (even)
    const int32_t* hcells = nullptr;  // [ntiles][kEdgeHalo] edges owned before the tile
    const int32_t* hcount = nullptr;  // [ntiles]
    const uint32_t* loc = nullptr;    // [ld] per cell: 3 x 8-bit offsets into a stage row
};

// Same for the 32-column tiles of the small-level sweep.
struct SmallHalo {
    const int32_t* cells = nullptr;   // [ntiles][kSmallHaloMax]
    const int32_t* count = nullptr;   // [ntiles]
    const uint32_t* loc = nullptr;    // [ld]: slot < 32 in-tile, else 32 + halo index
};

// Read-only view of one level's operator, passed by value to kernels.
// Bands are layer-major [nz][ld]; the neighbour table is SoA [3][ld].
struct LevelView {
    int64_t n;          // cells
    int64_t ld;         // leading dimension (multiple of 32)
    int nz;
    const int32_t* __restrict__ nbr;   // [3][ld]
    const double* __restrict__ D;
    const double* __restrict__ U;      // U[k] couples layers k and k+1; U[nz-1] = 0
    const double* __restrict__ H0;
    const double* __restrict__ H1;
    const double* __restrict__ H2;
};

// Distribution of one level: owned cells [0, n) in global order
// (global id off + c), halo slots [n, n + n_halo) grouped by owner rank.
struct DistLevel {
    bool on = false;                 // distributed level; false: single GPU or replicated level
    int64_t off = 0;                 // global id of local cell 0
    int64_t n_halo = 0;
    int64_t coff = 0;                // offset added to (c >> 2) to index the coarser level's vectors
    std::vector<int> peer_rank;
    std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;   // cells
    int64_t send_total = 0;
    int32_t* send_idx = nullptr;     // device, concatenated per peer
    double* sendbuf = nullptr;       // device [send_total][nz]
    double* recvbuf = nullptr;       // device [n_halo][nz]
};

struct DevLevel {
    int ref = 0;
    int64_t n = 0, ld = 0;
    int32_t* nbr = nullptr;     // [3][ld]
    double* geom = nullptr;     // [7][ld]: area, len0..2, cd0..2
    double* lam = nullptr;      // [nz][ld]
    double* bands = nullptr;    // [5][nz][ld]: D, U, H0, H1, H2
    double* wa = nullptr;       // V-cycle ping-pong work [nz][ld]
    double* wb = nullptr;
    double* b = nullptr;        // coarse-level right-hand side
    double* u = nullptr;        // coarse-level output (coarse correction)
    int32_t* halo_cells = nullptr;
    int32_t* halo_count = nullptr;
    uint32_t* halo_loc = nullptr;
    TileHalo halo;
    int32_t* small_cells = nullptr;
    int32_t* small_count = nullptr;
    uint32_t* small_loc = nullptr;
    SmallHalo small;
    // tiles of the cooperative coarse tail (width coarse_coop_tile_width(nz):
    // the 32-cell tables above when that is 32, else their own)
    int32_t* coop_cells = nullptr;
    int32_t* coop_count = nullptr;
    uint32_t* coop_loc = nullptr;
    SmallHalo coop_halo;
    // edge-deduplicated couplings (streamed-sweep levels; HMG_EDGE_H=0 disables)
    double* hedge = nullptr;
    int32_t *edge_e0 = nullptr, *edge_ne = nullptr, *edge_hcells = nullptr, *edge_hcount = nullptr;
    uint32_t* edge_loc = nullptr;
    int32_t* edge_own = nullptr;      // [2][ldE] owner cell and slot of each edge (setup)
    int64_t edge_count = 0;
    EdgeTiles edge;
    // Thomas factors (coarse-tail levels only): pivots, refined reciprocals, multipliers
    double* fden = nullptr;
    double* fy = nullptr;
    double* fg = nullptr;
    bool mf_safe = false;       // matrix-free quotients provably in the fast path's exact range (build_impl)
    bool g_safe = false;        // every Thomas pivot valid and every g_k exact by the fast path (k_pivot_check)
    DistLevel dist;
    LevelView view(int nz) const {
        const int64_t s = (int64_t)nz * ld;
        return LevelView{n, ld, nz, nbr, bands, bands + s, bands + 2 * s, bands + 3 * s, bands + 4 * s};
    }
};

// Device-resident PCG scalars: one struct so a single 64-byte D2H read per
// iteration returns the residual norm and the singular-pivot flag together.
struct PcgScalars {
    double rho, alpha, beta, pq, rr, rz, bb, tmp;
    unsigned long long bad;     // encoded (ref << 40 | column) of the first bad pivot, or ~0
    unsigned int fin_count;     // fused finalize: CTAs of the current partial-sum launch that are done
};

// Optional per-launch CUDA-event timing (hmg_profile_*): each instrumented
// launch records an event pair on its own stream; totals are read back per
// (kernel class, level).  Off by default; the benchmark turns it on for the
// timed region to report the dominant kernel's live duration.
enum KernelClass { kKApply = 0, kKSweepZero, kKSweep, kKSweepProlong, kKResidRestrict, kKRestrict, kKProlong,
                   kKVector, kKCoarseTail, kKApplyP, kKMixed, kKNumClasses };
struct Profiler {
    bool on = false;
    int only_cls = -1, only_ref = -1;   // hmg_profile_select: record only this class / level (-1: all)
    std::vector<cudaEvent_t> pool;   // pairs
    size_t used = 0;                 // events in use
    std::vector<int> cls, ref;       // per pair
};

// NEXT-4 mixed velocity-pressure system (mixed.cu): tables of the fine level,
// built on first use.  Vectors [U_h: nz x ldh | U_z: (nz-1) x ld | P: nz x ld].
struct MixedSystem {
    int64_t ne = 0, ldh = 0, off_z = 0, off_p = 0, ntot = 0;
    double omega = 0;
    int32_t *eca = nullptr, *ecb = nullptr, *esa = nullptr;   // [ldh]: cells a < b, slot of the edge in a
    int32_t* ee = nullptr;      // [6][ldh] edges of a's slots, then b's
    double* eg = nullptr;       // [6][ldh] RT0 mass rows (sign-adjusted Gram entries)
    int32_t* ce = nullptr;      // [3][ld] edge across each slot of a cell
    double* cs = nullptr;       // [3][ld] +1 / -1: the edge's flux leaves / enters the cell
    double* IL = nullptr;       // [off_p] lumped inverse mass of every velocity dof
    double* g = nullptr;        // [nz][ld] preconditioner: V-cycle right-hand side
    int nblocks = 0;
    double *part = nullptr, *dots = nullptr, *dots_host = nullptr;
    int m = 0;                  // GMRES workspace: basis V [m+1][ntot], w, z, t
    double *V = nullptr, *w = nullptr, *z = nullptr, *t = nullptr;
};

struct Hierarchy {
    mutable MixedSystem* mix = nullptr;
    mutable std::vector<double> res_hist;   // ||r_k|| / ||b|| of the last PCG solve, k = 0 .. iters
    int device = 0;
    int fine_ref = 0, coarsest_ref = 0, nz = 0;
    double thickness = 0, w2 = 0, dz = 0;
    double sn = 1.0;            // 1 + omega_N^2: the buoyancy factor of Eq. 5 / Eq. 8 (reading R24)
    std::vector<DevLevel> lev;  // index = ref
    // PCG workspace on the finest level
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *p2 = nullptr;
    double* partials = nullptr; // per-block partial sums (deterministic reductions)
    int npartials = 0;
    PcgScalars* scal = nullptr; // device
    PcgScalars* scal_host = nullptr;  // mapped pinned host memory, written by the finalize kernels
    PcgScalars* scal_pub = nullptr;   // its device alias
    double *hb = nullptr, *hx = nullptr;  // device staging for the host entry point
    // pipelined host batch (hmg_pcg_solve_host_batch): second staging pair,
    // copy-in / copy-out streams and their events
    double *hb1 = nullptr, *hx1 = nullptr;
    cudaStream_t cs_in = nullptr, cs_out = nullptr;
    // PCG: x = x + alpha p deferred to the side stream xs, launched when the
    // V-cycle reaches its latency-bound coarse part (idle HBM, free SMs)
    cudaStream_t xs = nullptr;
    cudaEvent_t ev_x_go = nullptr, ev_x_done = nullptr;
    struct PendingX {
        bool pending = false, first = false;
        double* x = nullptr;
        const double* p = nullptr;
    };
    mutable PendingX px;
    bool defer_x = true;        // HMG_DEFER_X=0: x and r updated by one kernel on the solve stream
    int x_slow_blocks = 148;    // HMG_X_BLOCKS=n: the deferred update by n grid-stride CTAs (0: the full vector grid)
    cudaEvent_t ev_in[2] = {}, ev_solved[2] = {}, ev_out[2] = {};
    int coop_ref = -1;          // levels <= coop_ref run in one cooperative smem-tile launch (-1: off)
    // multi-GPU (hmg_build_hierarchy_dist): levels > gather_ref are distributed
    int rank = 0, nranks = 1, gather_ref = -1;
    ncclComm_t comm = nullptr;
    bool force_coll = false;   // HMG_FORCE_COLLECTIVES=1: run the collectives even with one rank (tests)
    double *gbuf_send = nullptr, *gbuf_recv = nullptr;   // coarse-gather staging
    mutable int64_t launches = 0;
    // PCG: <r, z> fused into the preconditioner's last fine-level sweep (which
    // writes z and streams r as its right-hand side): pcg_impl sets rz_req, the
    // sweep launch that takes it writes per-CTA partial sums and sets rz_parts
    mutable bool rz_req = false;
    mutable int rz_parts = 0;
    mutable int rz_op = -1;           // the scalar op of that <r, z> (fused finalize)
    // fused finalize (FinArgs): op announced for the next partial-sum launch,
    // and whether that launch took it
    mutable int fin_op = -1;
    mutable bool fin_fused = false;
    bool fuse_rz = true;        // HMG_FUSE_RZ=0: separate dot kernel
    int64_t fact_max_cells = kFactMaxCells;   // levels up to this size carry precomputed Thomas factors
    bool check_skip = true;     // HMG_CHECK_SKIP=0: keep the per-layer pivot / g tests even where proven at build
    mutable Profiler prof;
    // diagnostics switches (environment, read at build time): HMG_SWEEP=simple
    // selects the reference-layout sweep kernel, HMG_SMALL=0 disables the
    // small-level kernel, HMG_L2PF sets the streamed sweep's L2 prefetch
    // distance in ring stages, HMG_TAIL_REF the one-launch coarse tail
    // Fixed choices of the measured design (DESIGN.md 7.1a lists the alternatives
    // that were measured; only the test knobs of README.md are read from the
    // environment, in build_impl).
    bool use_tc_sweep = true;   // TMEM/TMA sweeps (k_sweep_tc, k_sweep_st) instead of thread-per-column k_sweep
    bool use_st_sweep = true;   // non-zero-guess sweeps by the streamed k_sweep_st
    bool use_pdl = true;        // programmatic dependent launch of the persistent kernels
    bool use_st_apply = true;   // streamed k_apply_st instead of thread-per-column k_apply_t
    bool matrix_free = false;   // operator applies recompute the couplings from lam + geometry (NEXT-2; HMG_OPERATOR=free)
    bool use_small_sweep = true;
    bool edge_h = true;         // edge-deduplicated couplings on levels of >= edge_min_dofs (HMG_EDGE_MIN_DOFS)
    int64_t edge_min_dofs = 16LL << 20;
    bool resid_st = true;       // residual + restriction by the streamed apply on edge-store levels
    int apply_ctas_per_sm = 3;  // CTAs per SM of the p-update and residual applies
    int l2_prefetch_groups = 0;   // measured: the ring alone is as fast at ref 7 and faster at ref 6
};

// mixed.cu (NEXT-4)
std::string mixed_setup(const Hierarchy& H);   // "" on success
void mixed_free(MixedSystem* M);
void launch_mixed_apply(const Hierarchy& H, const double* x, double* y, cudaStream_t s);
void mixed_precond(const Hierarchy& H, const hmg_mg_params* p, const double* f, double* x, cudaStream_t s);
void mixed_dots(const Hierarchy& H, const double* w, const double* const* v, int nv, int dot, cudaStream_t s);
void mixed_update(const Hierarchy& H, const double* win, double* wout, const double* const* v, const double* c, int nv,
                  bool add, cudaStream_t s);
void mixed_vec(const Hierarchy& H, int op, const double* x, const double* b, double sc, double* y, cudaStream_t s);
int mixed_lin_max();
// api.cu: one V-cycle on the finest level (Alg. 1)
void vcycle_fine(const Hierarchy& H, const hmg_mg_params& p, const double* b, double* out, cudaStream_t s);

// kernels.cu
void launch_edge_h(const Hierarchy& H, const DevLevel& L, int64_t nedges, cudaStream_t s);
void launch_assemble(const Hierarchy& H, const DevLevel& L, cudaStream_t s);
void launch_coarsen_lam(const Hierarchy& H, const DevLevel& F, const DevLevel& C, cudaStream_t s);
void launch_apply(const Hierarchy& H, const DevLevel& L, const double* x, double* y, cudaStream_t s);
void launch_apply_dot(const Hierarchy& H, const DevLevel& L, const double* x, double* y,
                      cudaStream_t s);   // partial sums of x.y into H.partials
// One sweep: uout = uin(+P uc) + omega T^{-1}(b - H^ uin(+P uc)); uin == nullptr -> zero guess.
void launch_sweep(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin,
                  const double* uc, double* uout, double omega, cudaStream_t s);
void launch_restrict(const Hierarchy& H, const DevLevel& F, const double* r, double* bc, cudaStream_t s);
void launch_resid_restrict(const Hierarchy& H, const DevLevel& F, const double* b, const double* u,
                           double* bc, cudaStream_t s);
void launch_prolong_add(const Hierarchy& H, const DevLevel& F, const double* uin, const double* uc,
                        double* uout, cudaStream_t s);
// PCG vector kernels (scalars read from H.scal on the device)
void launch_dot(const Hierarchy& H, const DevLevel& L, const double* a, const double* b, cudaStream_t s);
void launch_finalize(const Hierarchy& H, int op, cudaStream_t s);
void launch_update_xr(const Hierarchy& H, const DevLevel& L, double* x, const double* p, cudaStream_t s);
void launch_update_part(const Hierarchy& H, const DevLevel& L, int part, bool first, double* x, const double* p,
                        const double* b, cudaStream_t s);
// first iteration from x = 0, r = b: x = 0 + alpha p, r = b - alpha q (reads b, not x or r)
void launch_update_xr_first(const Hierarchy& H, const DevLevel& L, double* x, const double* p, const double* b,
                            cudaStream_t s);
// q = H^ p_new with p_new = z + beta p_old formed on the fly and stored; partial <p_new, q> -> alpha
void launch_apply_pupdate_dot(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                              double* q, cudaStream_t s);
void launch_copy_pad(const Hierarchy& H, const DevLevel& L, const double* src, int64_t src_ld,
                     double* dst, int64_t dst_ld, cudaStream_t s);
int partials_needed(int64_t n, int nz);
// sweep_tc.cu: TMA-streamed, TMEM-state sweep (same arithmetic as launch_sweep's kernel)
bool sweep_tc_supported(const Hierarchy& H, const DevLevel& L);
void launch_sweep_tc(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                     double* uout, double omega, cudaStream_t s);

// sweep_st.cu: streamed persistent sweep with a non-zero iterate (same arithmetic)
bool sweep_st_supported(const Hierarchy& H, const DevLevel& L);
bool sweep_edge_store(const Hierarchy& H, const DevLevel& L);
void launch_sweep_st(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                     double* uout, double omega, cudaStream_t s);
// the same general sweep (non-zero iterate, no prolongation, stored bands) also
// accumulating <b, u'> per CTA into H.partials; returns the number of partials
int launch_sweep_st_dot(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, double* uout,
                        double omega, cudaStream_t s);

// apply_st.cu: TMA-streamed persistent operator apply (same arithmetic as k_apply_t);
// the dot forms return the number of per-CTA partial sums written to H.partials
bool apply_st_supported(const Hierarchy& H, const DevLevel& L);
bool resid_st_supported(const Hierarchy& H, const DevLevel& L);
void launch_resid_restrict_st(const Hierarchy& H, const DevLevel& L, const double* b, const double* u, double* bc,
                              int64_t ldc, int64_t coff, cudaStream_t s);
int launch_apply_st(const Hierarchy& H, const DevLevel& L, const double* x, double* y, bool dot, cudaStream_t s);
int launch_apply_pupdate_st(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                            double* q, cudaStream_t s);
void finalize_parts(const Hierarchy& H, int nparts, int op, cudaStream_t s);

// band.cu (NEXT-3 core: batched banded LU / solve / product, DG1 <-> DG0)
bool band_shape_supported(int kl, int ku);
void launch_band_factor(int64_t ncol, int m, int kl, int ku, double* ab, int64_t ld, int32_t* ipiv,
                        unsigned long long* bad, cudaStream_t s);
void launch_band_solve(int64_t ncol, int m, int kl, int ku, const double* ab, int64_t ld, const int32_t* ipiv,
                       const double* b, double* x, cudaStream_t s);
void launch_band_apply(int64_t ncol, int m, int kl, int ku, const double* ar, int64_t ld, const double* x, double* y,
                       cudaStream_t s);
void launch_p_restrict(int64_t ncol, int nz, const double* r1, int64_t ld, double* b0, cudaStream_t s);
void launch_p_prolong_add(int64_t ncol, int nz, const double* u0, int64_t ld, double* u1, cudaStream_t s);

// thomas_factor.cu
void launch_factor(const Hierarchy& H, const DevLevel& L, cudaStream_t s);
void launch_pivot_check(const Hierarchy& H, const DevLevel& L, unsigned int* gslow, cudaStream_t s);
// coarse_coop.cu: levels <= H.coop_ref in one cooperative launch (32-column smem tiles)
bool coarse_coop_supported(const Hierarchy& H);
int coarse_coop_tile_width(int nz);   // 32, 16 or 8 columns per tile (0: no fit)
void launch_coarse_coop(const Hierarchy& H, const hmg_mg_params& p, const double* b_top, double* out_top,
                        cudaStream_t s);
size_t coarsest_smem_bytes(int nz, int64_t n, int threads);
void launch_coarsest(const Hierarchy& H, const DevLevel& L, const double* b, double* out, int n_coarse, double omega,
                     cudaStream_t s);
// sweep_small.cu: small-level sweep (whole tile in shared memory); nsweeps > 1 only for a one-tile level
bool sweep_small_supported(const Hierarchy& H, const DevLevel& L);
void launch_sweep_small(const Hierarchy& H, const DevLevel& L, const double* b, const double* uin, const double* uc,
                        double* uout, double omega, int nsweeps, cudaStream_t s);
// Error raised on the host side of a launch (tensor-map encoding); nullptr if none.
const char* take_launch_error();
bool tensor_maps_available();
void launch_selftest_div(int64_t n, const double* a, const double* b, double* fast, double* ref, cudaStream_t s);

// Stream-ordered launch with programmatic dependent launch (PDL) allowed: the
// kernel may begin (prologue, SM placement) while its predecessor finishes;
// every kernel launched this way calls ptx::pdl_wait() before touching data a
// predecessor produced or consumes.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(const Hierarchy& H, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = H.use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// RAII event pair around one launch when profiling is on.
struct ProfScope {
    const Hierarchy& H;
    cudaStream_t s;
    cudaEvent_t stop = nullptr;
    ProfScope(const Hierarchy& h, int cls, int ref, cudaStream_t st);
    ~ProfScope();
};

// kFinRRBB: the first r update's two sums, <r, r> in partial[0, nb) and <b, b>
// in partial[nb, 2 nb) (fused finalize only)
enum FinalizeOp { kFinPQ = 0, kFinRR = 1, kFinRZ = 2, kFinRhoInit = 3, kFinBB = 4, kFinRRBB = 5 };

// Fused finalize (one rank): a kernel that writes one partial sum per CTA into
// `partial` also applies the PCG scalar update -- its last CTA to finish sums
// the partials in a fixed order (one warp: strided per lane, then a fixed
// shuffle tree) and does k_finalize's scalar op, so no single-block finalize
// launch follows.  op < 0: not fused (k_finalize or the all-reduce follows).
struct FinArgs {
    int op = -1;
    PcgScalars* sc = nullptr;
    PcgScalars* pub = nullptr;   // mapped host copy for the scalars the host reads
};
// The FinArgs of the next partial-sum launch: finalize_parts' op when the sum
// needs no all-reduce (pcg_impl announces it with fin_begin before the launch;
// the launch takes it with fin_take, and finalize_parts then launches nothing)
FinArgs fin_take(const Hierarchy& H);
void fin_begin(const Hierarchy& H, int op);

#ifdef __CUDACC__
__device__ __forceinline__ void pcg_scalar_op(PcgScalars* sc, int op, double S) {
    switch (op) {
        case kFinPQ: sc->pq = S; sc->alpha = sc->rho / S; break;
        case kFinRR: sc->rr = S; break;
        case kFinRZ: sc->rz = S; sc->beta = S / sc->rho; sc->rho = S; break;
        case kFinRhoInit: sc->rho = S; break;
        case kFinBB: sc->bb = S; break;
    }
}
// Every thread of the CTA calls it after the CTA's partial was stored by thread 0.
__device__ __forceinline__ void fin_fused(const FinArgs& f, const double* partial) {
    if (f.op < 0) return;
    __shared__ unsigned s_last;
    __syncthreads();
    const unsigned nb = gridDim.x * gridDim.y;
    if (threadIdx.x == 0) {
        __threadfence();                               // this CTA's partial before its arrival
        s_last = atomicAdd(&f.sc->fin_count, 1u) == nb - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    __threadfence();
    double v = 0.0, w = 0.0;
    for (unsigned i = threadIdx.x; i < nb; i += 32) v = v + __ldcg(partial + i);
    if (f.op == kFinRRBB)
        for (unsigned i = threadIdx.x; i < nb; i += 32) w = w + __ldcg(partial + nb + i);
    for (int off = 16; off > 0; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
    for (int off = 16; off > 0; off >>= 1) w = w + __shfl_down_sync(0xffffffffu, w, off);
    if (threadIdx.x == 0) {
        f.sc->fin_count = 0;
        if (f.op == kFinRRBB) {
            f.sc->rr = v;
            f.sc->bb = w;
        } else {
            pcg_scalar_op(f.sc, f.op, v);
        }
        if (f.pub) *f.pub = *f.sc;
    }
}
#endif

// multi-GPU helpers (kernels.cu)
void launch_halo_pack(const Hierarchy& H, const DevLevel& L, const double* v, cudaStream_t s);
void launch_halo_unpack(const Hierarchy& H, const DevLevel& L, double* v, cudaStream_t s);
void launch_gather_pack(const Hierarchy& H, const DevLevel& C, const double* v, int64_t off, int64_t cnt, cudaStream_t s);
void launch_gather_unpack(const Hierarchy& H, const DevLevel& C, double* v, int64_t cnt, cudaStream_t s);
void launch_update_p(const Hierarchy& H, const DevLevel& L, double* p, const double* z, cudaStream_t s);
// halo slots of p_new = z + beta p_old (multi-GPU fused CG direction update)
void launch_halo_pupdate(const Hierarchy& H, const DevLevel& L, const double* z, const double* pold, double* pnew,
                         cudaStream_t s);
// finalize of a dot when its partial sums are rank-local: local total into scal->tmp
void launch_finalize_local(const Hierarchy& H, int nparts, cudaStream_t s);
void launch_scalar_op(const Hierarchy& H, int op, cudaStream_t s);   // op on scal->tmp as the (global) sum
// api.cu: all-reduce (sum) of scal->tmp across the ranks on stream s
void dist_allreduce_tmp(const Hierarchy& H, cudaStream_t s);

}  // namespace hmg
