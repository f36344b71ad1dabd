/*
 * hmg.h -- C-ABI of the B200-native tensor-product multigrid Helmholtz solver
 * (hot path of arXiv:1605.00492, Mitchell & Mueller).
 *
 * Problem (Eq. 8 and P:626): solve  H^ P = R  for the DG0 pressure
 * P on an extruded icosahedral prism mesh of a thin spherical shell, with
 *   H^ = M3 + w_c^2 (Dh Minv_h Dh^T + Dz Minv_z Dz^T / (1 + w_N^2))
 * assembled with lumped two-point couplings (readings R1-R4):
 *   vertical   coupling  w2 * area * lamf / dz
 *   horizontal coupling  w2 * edge_len * dz * lamf / centroid_dist
 *   diagonal             prism volume + sum of couplings
 * by CG preconditioned with the tensor-product multigrid V-cycle of
 * Alg. 1 and Sec. 4.2.1: damped vertical line-Jacobi
 * smoother (Eq. 10/13), horizontal-only coarsening down the
 * icosahedral hierarchy (MeshHierarchy) with 4-child sum
 * restriction and injection prolongation.
 *
 * Conventions for every entry point
 *  - Return value: hmg_status; HMG_OK = 0.  On error a message naming the
 *    offending argument (or the singular column) is available from
 *    hmg_last_error() (thread-local, valid until the next call on the thread).
 *  - Vectors are fp64, LAYER-MAJOR [nlayers][ld] (cells contiguous within a
 *    layer), where ld is the level's leading dimension from hmg_level_info
 *    (ld = number of cells rounded up to a multiple of 32).  Entries with
 *    cell index >= ncells are padding: their values never affect a result
 *    (they may be read by row-block copies) and they are never written.
 *    Device vector pointers must be 16-byte aligned (HMG_ERR_INVALID_ARG).
 *  - Device pointers (everything except *_host arguments) are caller-owned
 *    CUDA device memory on the hierarchy's device; host pointers are plain
 *    host memory.  The library never frees caller memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls enqueue work on `stream` and return without
 *    synchronising unless stated otherwise.  A hierarchy is not re-entrant:
 *    do not use one hierarchy from two streams concurrently.
 *  - Input and output vectors of one call must not alias unless stated.
 *  - Cell numbering: the 20 icosahedron faces in the fixed order of reading
 *    R1; children of cell p at the next refinement are 4p+0..4p+3.
 */
#ifndef HMG_H
#define HMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HMG_OK = 0,
    HMG_ERR_INVALID_ARG = 1,     /* message names the argument */
    HMG_ERR_CUDA = 2,            /* CUDA runtime error (message has cudaGetErrorString) */
    HMG_ERR_NCCL = 3,            /* NCCL missing or a collective failed (multi-GPU) */
    HMG_ERR_SINGULAR_COLUMN = 4, /* a Thomas pivot was <= 0 or non-finite: "ref r column c" */
    HMG_ERR_NOT_CONVERGED = 5,   /* PCG hit maxit; outputs are still filled in */
    HMG_ERR_OOM = 6              /* device or host allocation failed */
} hmg_status;

/* Opaque hierarchy: owns every level's neighbour table, geometry, bands and
 * V-cycle workspaces (device memory), plus the PCG workspace. */
typedef struct hmg_hierarchy hmg_hierarchy;

/* Multigrid parameters.  The defaults of BASELINE.json are
 * {nu_pre = 2, nu_post = 2, n_coarse = 20, omega = 0.8}; the paper's own run
 * uses {1, 1, 2, 0.8}. */
typedef struct {
    int nu_pre;    /* presmoothing sweeps per level (>= 0) */
    int nu_post;   /* postsmoothing sweeps per level (>= 0) */
    int n_coarse;  /* sweeps from zero on the coarsest level (>= 1) */
    double omega;  /* damping of the line-Jacobi correction (reading R7) */
} hmg_mg_params;

/* Build the hierarchy ref fine_ref -> coarsest_ref (setup; synchronous).
 *  fine_ref      0..10, refinement of the icosahedron (20*4^fine_ref cells)
 *  coarsest_ref  0..fine_ref, coarsest multigrid level
 *  nlayers       >= 1 uniform layers; dz = thickness / nlayers
 *  thickness     > 0 shell thickness (unit sphere radius)
 *  w2            >= 0 coupling scale (w_c^2 of Eq. 8)
 *  lam_host      HOST array [nlayers][20*4^fine_ref] (dense, no padding) of
 *                per-dof coefficients, each finite and > 0; copied, not kept
 *  device        CUDA device ordinal
 *  out           receives the hierarchy; *out = NULL on failure
 * Coarse coefficients are the 4-child means (reading R3); every level is
 * rediscretised, not Galerkin.  The Thomas pivots of every column
 * of every level are checked here (they depend on the operator only): a
 * non-positive or non-finite pivot -> HMG_ERR_SINGULAR_COLUMN "ref r column c". */
hmg_status hmg_build_hierarchy(int fine_ref, int coarsest_ref, int nlayers, double thickness,
                               double w2, const double* lam_host, int device, hmg_hierarchy** out);

/* Multi-GPU (one process per GPU, the paper's horizontal domain
 * decomposition with halo exchanges).  Rank r of nranks
 * (nranks must divide 320) owns the ref-2 cells [r*320/nranks,
 * (r+1)*320/nranks) and, because children of p are 4p..4p+3, the contiguous
 * global cells [r*n/nranks, (r+1)*n/nranks) on every level ref > gather_ref.
 * Levels ref <= gather_ref (gather_ref in [max(2, coarsest_ref), fine_ref])
 * are replicated: their right-hand side is all-gathered and every rank runs
 * them redundantly (the coarse gather).  Vectors of a distributed level are
 * [nlayers][ld] with the owned cells first, in global order (local c = global
 * off + c), then the halo cells; halo slots are library scratch, written by
 * the library before it reads them (so inputs are written there too).
 * Transport: NCCL (libnccl.so.2 resolved at run time) -- grouped send/recv of
 * packed halos, all-reduce of CG inner products, all-gather at gather_ref. */
typedef struct {
    int rank;
    int nranks;
    const unsigned char* nccl_id;   /* 128 bytes from hmg_nccl_unique_id on rank 0, same on all ranks */
    int gather_ref;
} hmg_dist;

/* As hmg_build_hierarchy for one rank of a distributed hierarchy.  lam_host is
 * this rank's owned part of the finest level, [nlayers][20*4^fine_ref/nranks],
 * when gather_ref < fine_ref (else the whole finest level).  Collective: all
 * ranks must call it. */
hmg_status hmg_build_hierarchy_dist(int fine_ref, int coarsest_ref, int nlayers, double thickness,
                                    double w2, const double* lam_host, int device,
                                    const hmg_dist* dist, hmg_hierarchy** out);

/* As hmg_build_hierarchy / hmg_build_hierarchy_dist (dist = NULL: one GPU) with
 * the buoyancy term omega_n = omega_N = (dt/2) N >= 0 of Eq. 5 (
 * DESIGN.md reading R24): eliminating buoyancy scales the vertical velocity
 * mass by 1 + omega_N^2, so the pressure operator's vertical couplings are
 * divided by it (Eq. 8: ((w2*area)*lamf/dz) / (1 + omega_N^2)) and the mixed
 * system (hmg_mixed_*) uses M~2 = M2h (+) (1 + omega_N^2) M2z and the matching
 * lumped mass.  omega_n = 0 is exactly hmg_build_hierarchy.  The matrix-free
 * operator (HMG_OPERATOR=free) supports omega_n = 0 only (HMG_ERR_INVALID_ARG). */
hmg_status hmg_build_hierarchy_ex(int fine_ref, int coarsest_ref, int nlayers, double thickness, double w2,
                                  double omega_n, const double* lam_host, int device, const hmg_dist* dist,
                                  hmg_hierarchy** out);

/* ncclGetUniqueId into id_out[128] (call on rank 0, broadcast the bytes). */
hmg_status hmg_nccl_unique_id(unsigned char* id_out);

/* Host-only query of the partition plan of level `ref` for `rank` (no GPU;
 * used by tests).  Pass NULL arrays to get the sizes first.  Outputs: global
 * offset and count of the owned cells, halo size, number of peers, total
 * send count; halo_gid[n_halo] (global ids, grouped by owner rank, ascending),
 * nbr_local[n_own][3] (local numbering), per peer: rank, send count, receive
 * offset/count (halo slots relative to n_own); send_local (concatenated owned
 * local indices each peer needs, ascending global id). */
hmg_status hmg_partition_plan(int fine_ref, int ref, int rank, int nranks, int64_t* off, int64_t* n_own,
                              int64_t* n_halo, int* npeers, int64_t* send_total, int64_t* halo_gid,
                              int32_t* nbr_local, int32_t* peer_rank, int64_t* send_count,
                              int64_t* recv_offset, int64_t* recv_count, int32_t* send_local);

/* Free all device and host storage of the hierarchy (NULL is a no-op). */
hmg_status hmg_free_hierarchy(hmg_hierarchy* h);

/* Size of level `ref`: number of cells and leading dimension of vectors. */
hmg_status hmg_level_info(const hmg_hierarchy* h, int ref, int64_t* ncells, int64_t* ld);

/* y = H^ x on level `ref` (Eq. 8; "v = H^ u = H^_z u + H^_h u").
 * x, y: device [nlayers][ld].  Row order of reading R5.  x is non-const: on a
 * distributed level the library writes x's halo slots (the neighbours' owned
 * values) before reading them; its owned entries are not modified. */
hmg_status hmg_apply_helmholtz(const hmg_hierarchy* h, int ref, double* x, double* y,
                               void* stream);

/* nsweeps damped line-Jacobi sweeps on level `ref` (Eq. 10 read with Eq. 13,
 * reading R7):  u <- u + omega * T^{-1} (b - H^ u),  T = the column-block
 * (tridiagonal) part of H^ (Eq. 9), solved per column by the Thomas
 * algorithm.  If u_is_zero != 0 the incoming u is taken as zero
 * and the first sweep is u = omega * T^{-1} b (its content is ignored).
 * b, u: device [nlayers][ld]; u is updated in place (ping-pong is internal).
 * A non-positive or non-finite pivot -> HMG_ERR_SINGULAR_COLUMN (this call
 * synchronises `stream` to report it).  The pivots depend on the operator only
 * and hmg_build_hierarchy checks every column of every level once, so a
 * hierarchy that was built without error cannot produce this status here. */
hmg_status hmg_line_smooth(const hmg_hierarchy* h, int ref, const double* b, double* u,
                           int nsweeps, double omega, int u_is_zero, void* stream);

/* b_c = R r_f: 4-child sum restriction from fine_ref to fine_ref-1
 * (reading R8).  r_f: [nlayers][ld_fine], b_c: [nlayers][ld_coarse].
 * Distributed hierarchy: restriction is rank-local; when level fine_ref-1 is
 * replicated (fine_ref-1 <= gather_ref < fine_ref) b_c receives the WHOLE
 * coarse vector on every rank (the coarse all-gather; collective). */
hmg_status hmg_restrict(const hmg_hierarchy* h, int fine_ref, const double* r_f, double* b_c,
                        void* stream);

/* b_c = R (b - H^ u): fused residual + restriction on level fine_ref
 * (residual in the row order of reading R5, then the sum of reading R8).
 * u is non-const for the same reason as x of hmg_apply_helmholtz (halo slots
 * written on a distributed level, owned entries untouched); b_c as for
 * hmg_restrict (whole coarse vector when the coarser level is replicated). */
hmg_status hmg_residual_restrict(const hmg_hierarchy* h, int fine_ref, const double* b,
                                 double* u, double* b_c, void* stream);

/* u_f += P u_c: injection prolongation ("natural embedding"). */
hmg_status hmg_prolong_add(const hmg_hierarchy* h, int fine_ref, const double* u_c, double* u_f,
                           void* stream);

/* z = B b: one V-cycle (Alg. 1 recursively; reading R9) from the finest level
 * with zero initial guess.  b, z: device [nlayers][ld_fine]. */
hmg_status hmg_vcycle(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b, double* z,
                      void* stream);

/* Solve H^ x = b by CG preconditioned with one V-cycle per iteration
 * (reading R10/R12), x0 = 0, stopping when ||r_k||_2 <= rtol ||b||_2 on the
 * recursively updated residual.  b, x: device [nlayers][ld_fine].
 *  iters   number of H^ applications performed
 *  relres  final ||r||/||b||
 * Synchronises `stream` once per iteration (a mapped-memory read of ||r|| -- and,
 * in the first, of ||b||, which one rank sums in the first r update).
 * Returns HMG_ERR_NOT_CONVERGED (x, iters, relres filled) after maxit. */
hmg_status hmg_pcg_solve(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b, double* x,
                         double rtol, int maxit, int* iters, double* relres, void* stream);

/* As hmg_pcg_solve with HOST buffers b_host / x_host of shape
 * [nlayers][ncells_fine] (dense, no padding): copies b in, solves, copies x
 * out; synchronous.  The end-to-end entry point. */
hmg_status hmg_pcg_solve_host(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b_host,
                              double* x_host, double rtol, int maxit, int* iters, double* relres,
                              void* stream);

/* Pipelined end-to-end entry point for a stream of right-hand sides: solves
 * H^ x_i = b_i for i = 0 .. nrhs-1 (HOST buffers b_host[i], x_host[i], each
 * [nlayers][ncells_fine] dense, as hmg_pcg_solve_host), one solve after the
 * other on `stream`, with the host->device copy of b_{i+1} and the
 * device->host copy of x_{i-1} on two internal copy streams overlapping solve
 * i (two device staging pairs, ordered by events).  Each solve is exactly
 * hmg_pcg_solve (same arithmetic, same results).  For the copies to overlap,
 * the host buffers must be page-locked (cudaHostAlloc / cudaHostRegister);
 * pageable buffers give correct results without overlap.  iters[i],
 * relres[i]: per right-hand side.  Synchronous: returns after x_host[nrhs-1]
 * has landed.  Returns HMG_ERR_NOT_CONVERGED if any solve hit maxit (all
 * outputs filled); any other error stops the batch at that solve. */
hmg_status hmg_pcg_solve_host_batch(const hmg_hierarchy* h, const hmg_mg_params* p, int nrhs,
                                    const double* const* b_host, double* const* x_host, double rtol,
                                    int maxit, int* iters, double* relres, void* stream);

/* Residual history of the last hmg_pcg_solve* call on this hierarchy (host,
 * no synchronisation): hist[k] = ||r_k||_2 / ||b||_2 for k = 0 .. iters (the
 * recursively updated residual the stopping test reads; hist[0] = 1, or 0 for
 * b = 0).  *n receives iters + 1; at most cap values are written (hist may be
 * NULL to query n). */
hmg_status hmg_pcg_history(const hmg_hierarchy* h, double* hist, int cap, int* n);

/* Same as hmg_pcg_solve but preconditioned by `nsweeps` line-Jacobi sweeps
 * from zero on the finest level: the paper's single-level method
 * ("two iterations of Block-Jacobi vertical line relaxation"). */
hmg_status hmg_pcg_solve_single_level(const hmg_hierarchy* h, int nsweeps, double omega,
                                      const double* b, double* x, double rtol, int maxit,
                                      int* iters, double* relres, void* stream);

/* Export one level to HOST buffers (tests; synchronous; any pointer may be NULL):
 *  nbr   int32 [ncells][3]     cell across edge (v_j, v_{j+1}) of the cell
 *  geom  double [7][ncells]    area, len_0..2, cd_0..2 (reading R2)
 *  bands double [5][nlayers][ncells]  D, U, H_0, H_1, H_2 (U[k] couples k,k+1)
 *  lam   double [nlayers][ncells]      the level's coefficient */
hmg_status hmg_export_level(const hmg_hierarchy* h, int ref, int32_t* nbr, double* geom,
                            double* bands, double* lam);

/* Diagnostic: which kernels of level `ref` read the edge-deduplicated coupling
 * store (each face coupling stored once per layer instead of once per cell
 * side; built on levels of >= 16M dofs): bit 0 the streamed sweep, bit 1 the
 * streamed apply, bit 2 residual + restriction (then formed by the streamed
 * apply with a restriction epilogue).  Their algorithmic bytes per dof drop
 * by 12 (1.5 instead of 3 couplings); results are bitwise unchanged. */
hmg_status hmg_edge_store(const hmg_hierarchy* h, int ref, int* kernels);

/* Kernel launches issued by the library since the hierarchy was built
 * (diagnostic counter used by the benchmark's gpu_launches claim). */
int64_t hmg_launch_count(const hmg_hierarchy* h);

/* Diagnostics: CUDA-event timing of the library's kernel launches.
 * hmg_profile_begin clears and enables recording (an event pair on the
 * launching stream around every kernel), hmg_profile_end disables it, and
 * hmg_profile_query sums the recorded durations (synchronising on them) for
 * one kernel class on level `ref` (ref < 0: all levels).  Classes:
 * 0 apply, 1 zero-guess sweep, 2 sweep, 3 sweep with fused prolongation,
 * 4 residual+restriction, 5 restriction, 6 prolongation, 7 CG vector kernels,
 * 8 coarse-tail V-cycle (all levels <= the tail level in one launch),
 * 9 operator apply with the CG direction update p = z + beta p fused,
 * 10 the mixed system's kernels (hmg_mixed_*: apply, preconditioner steps,
 * GMRES vector operations; the preconditioner's V-cycle keeps its classes). */
hmg_status hmg_profile_begin(hmg_hierarchy* h);
hmg_status hmg_profile_end(hmg_hierarchy* h);
/* Restrict recording to one kernel class on one level (-1: any); an event pair
 * separates two kernels in the stream, so recording only the kernel being
 * measured leaves the other launches free to overlap (programmatic dependent
 * launch).  Persists until changed; hmg_profile_select(h, -1, -1) records all. */
hmg_status hmg_profile_select(hmg_hierarchy* h, int kernel_class, int ref);
hmg_status hmg_profile_query(const hmg_hierarchy* h, int kernel_class, int ref, int64_t* count, double* total_ms);

/* Diagnostic: for device arrays a, b of length n, writes fast[i] = the
 * shared-reciprocal division the sweep kernel uses and ref[i] = a[i] / b[i]
 * (the compiler's div.rn.f64).  The two must be bitwise equal. */
hmg_status hmg_selftest_div(const double* a, const double* b, double* fast, double* ref, int64_t n,
                            void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-4: the mixed velocity-pressure system around the V-cycle.
 * Eq. 5 with omega_N = 0 at lowest order, on the hierarchy's
 * finest level (single-GPU hierarchies; a distributed one is rejected with
 * HMG_ERR_INVALID_ARG):
 *     A [U; P] = [[M2, -omega D^T], [omega D, M3]] [U; P],   omega = sqrt(w2),
 * U = RT0 normal fluxes through the vertical faces (edge e, layer k; positive
 * from the edge's lower cell to its upper cell) and P1-in-the-vertical fluxes
 * through the interior interfaces (positive upward; u.n = 0 at top and bottom,
 * P:415-418), P = the DG0 pressure; M2 = the consistent velocity mass with
 * weight 1/lam per cell, M3 = diag(vol), D = the net outward flux (DESIGN.md
 * readings R15-R18).  Device vectors, fp64, caller-owned, one contiguous
 * array of ntot doubles:
 *     [0, off_z)        U_h  [nlayers][ldh]      (entries e >= ne are padding)
 *     [off_z, off_p)    U_z  [nlayers-1][ld]     (interface i = row i-1)
 *     [off_p, ntot)     P    [nlayers][ld]       (ld of the finest level)
 * Padding entries of inputs must be zero; outputs keep them zero.  The tables
 * (edge list, RT0 mass rows, lumped inverse) are built on the first call of
 * any hmg_mixed_* function and owned by the hierarchy. */
hmg_status hmg_mixed_layout(const hmg_hierarchy* h, int64_t* ne, int64_t* ldh, int64_t* off_z, int64_t* off_p,
                            int64_t* ntot);
/* Edge table to HOST buffers (tests; either may be NULL): ec int32 [ne][2] the
 * two cells of edge e (lower first), ce int32 [ncells][3] the edge across each
 * neighbour slot.  Edges are numbered by lower cell, then its slot (R16). */
hmg_status hmg_mixed_export_edges(const hmg_hierarchy* h, int32_t* ec, int32_t* ce);
/* y = A x (x, y must not alias). */
hmg_status hmg_mixed_apply(const hmg_hierarchy* h, const double* x, double* y, void* stream);
/* x = B f, the Schur-complement preconditioner of Eq. 6 with the
 * velocity mass replaced by its two-point lumping L (whose Schur complement
 * M3 + omega^2 D L^-1 D^T is exactly this library's H^) and H^-1 by one
 * V-cycle with parameters p (reading R19):
 *     g = f_P - omega D L^-1 f_U,  x_P = V(g),  x_U = L^-1 (f_U + omega D^T x_P).
 * p = NULL: x = f (no preconditioner). */
hmg_status hmg_mixed_precond(const hmg_hierarchy* h, const hmg_mg_params* p, const double* f, double* x,
                             void* stream);
/* Restarted right-preconditioned GMRES(restart) for A X = F from X = 0, the
 * paper's outer solver ("GMRES(k=30) to ||r||/||r_0|| < 1e-5", P:791-796;
 * reading R20): stops when the true residual ||F - A X||_2 <= rtol ||F||_2
 * (checked at the end of each cycle; within a cycle the Givens estimate ends
 * the cycle early).  iters = Arnoldi steps (preconditioner applications
 * excluding the one per cycle that forms X).  restart in [1, 31].
 * gs_passes: classical Gram-Schmidt passes per Arnoldi step -- 1 = CGS (what
 * PETSc's GMRES does by default, so most likely the paper's), 2 = CGS2 (the
 * recommended setting: one pass loses the basis' orthogonality on the
 * anisotropic problems, max|<v_a,v_b> - delta_ab| ~ 1e-1 at ref 5 x 64 C2b
 * against ~1e-12 with two; R20).  Other values: HMG_ERR_INVALID_ARG.
 * Synchronises once per Gram-Schmidt pass (the Hessenberg column).  Returns
 * HMG_ERR_NOT_CONVERGED with X, iters, relres filled after maxit steps. */
hmg_status hmg_mixed_gmres(const hmg_hierarchy* h, const hmg_mg_params* p, const double* F, double* X, double rtol,
                           int restart, int maxit, int gs_passes, int* iters, double* relres, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-3 core: batched per-column banded linear algebra of the
 * next-to-lowest-order discretisation.  There the column operator H^_z of
 * each vertical column is a banded matrix with m = 6 nz rows (DG1: 6 unknowns
 * per prism cell, ordered cell by cell) and bandwidth n_BW = kl + ku + 1 = 27
 * (P:1099-1106), inverted with a precomputed LU factorisation with partial
 * pivoting (LAPACK dgbtrf) and its solve (dgbtrs); the first
 * coarsening step is the p-coarsening DG1 -> DG0 by the natural embedding
 * (P:645-648).  These calls need no hierarchy.  Results are those of LAPACK's
 * algorithms in their operation order (oracle/band_oracle.c), every grid
 * column independent.
 *
 * Batched layouts (device, fp64 unless noted; c = grid column, ld >= ncol a
 * multiple of 32; pointers 16-byte aligned):
 *   ab    [m][2 kl + ku + 1][ld]   LU storage, LAPACK band format per column:
 *                                   A(i, j) at ab[(j*(2kl+ku+1) + kl+ku+i-j)*ld + c]
 *                                   (rows 0..kl-1 of each j: room for U's fill-in)
 *   ipiv  [m][ld] int32             0-based row interchanged with row j
 *   ar    [m][kl + ku + 1][ld]      the paper's row-wise band storage of the
 *                                   product kernel:
 *                                   A(i, j) at ar[(i*(kl+ku+1) + kl+j-i)*ld + c]
 *   vectors [m][ld]; a DG1 vector is [nz][6][ld], a DG0 one [nz][ld].
 * Compiled (kl, ku) pairs: (13, 13) (the NLO operator), (1, 1) (the LO one),
 * (2, 2), (3, 5), (5, 2), (0, 0); others -> HMG_ERR_INVALID_ARG.  m <= 4096. */

/* In-place LU factorisation of every column (dgbtrf; setup, synchronous).  On
 * an exactly zero pivot the factorisation is completed (as LAPACK's info > 0)
 * and HMG_ERR_SINGULAR_COLUMN names the first such grid column; *singular
 * (may be NULL) receives it, or -1. */
hmg_status hmg_band_factor(int64_t ncol, int m, int kl, int ku, double* ab, int64_t ld, int32_t* ipiv,
                           int64_t* singular, void* stream);
/* x = A^-1 b per column from hmg_band_factor's output (dgbtrs, 'N').  b, x
 * must not alias.  Useful bytes per column (Eq. 15):
 * 4 m (3 n_BW + 4). */
hmg_status hmg_band_solve(int64_t ncol, int m, int kl, int ku, const double* ab, int64_t ld,
                          const int32_t* ipiv, const double* b, double* x, void* stream);
/* y = A x per column, A in the row-wise storage ar (Eq. 14's 8 m (n_BW + 2)
 * bytes per column).  y(i) = sum over j in increasing order. */
hmg_status hmg_band_apply(int64_t ncol, int m, int kl, int ku, const double* ar, int64_t ld, const double* x,
                          double* y, void* stream);
/* DG1 -> DG0 restriction (transpose of the natural embedding; reading R21):
 * b0[k][c] = sum_{d=0..5} r1[6k+d][c], summed in d order.  r1 [6 nz][ld],
 * b0 [nz][ld]. */
hmg_status hmg_p_restrict(int64_t ncol, int nz, const double* r1, int64_t ld, double* b0, void* stream);
/* DG0 -> DG1 prolongation-add (natural embedding: a cell constant has every
 * nodal DG1 value equal to it): u1[6k+d][c] += u0[k][c]. */
hmg_status hmg_p_prolong_add(int64_t ncol, int nz, const double* u0, int64_t ld, double* u1, void* stream);

/* Message for the last error on this thread ("" if none). */
const char* hmg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HMG_H */
