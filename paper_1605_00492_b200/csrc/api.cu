// C-ABI of the B200 Helmholtz multigrid library (include/hmg.h): argument
// validation, hierarchy construction, the V-cycle driver (Alg. 1)
// and the PCG driver.  Every step of the path runs in kernels.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <type_traits>
#include <string>

#include "dist.h"
#include "hmg_internal.h"
#include "mesh.h"

using namespace hmg;

namespace {

thread_local std::string g_err;

hmg_status fail(hmg_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

#define HMG_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(e_ == cudaErrorMemoryAllocation ? HMG_ERR_OOM : HMG_ERR_CUDA,          \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

#define HMG_TRY(expr)                      \
    do {                                   \
        hmg_status s_ = (expr);            \
        if (s_ != HMG_OK) return s_;       \
    } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int64_t round_up32(int64_t n) { return (n + 31) & ~int64_t(31); }

std::string& nccl_err_ref();

hmg_status check_launch() {
    if (const char* m = take_launch_error()) return fail(HMG_ERR_CUDA, m);
    if (!nccl_err_ref().empty()) {
        std::string m = nccl_err_ref();
        nccl_err_ref().clear();
        return fail(HMG_ERR_NCCL, m);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(HMG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return HMG_OK;
}

hmg_status check_h(const hmg_hierarchy* h) {
    if (!h) return fail(HMG_ERR_INVALID_ARG, "h: null hierarchy");
    return HMG_OK;
}

const Hierarchy& HH(const hmg_hierarchy* h) { return *reinterpret_cast<const Hierarchy*>(h); }
Hierarchy& HH(hmg_hierarchy* h) { return *reinterpret_cast<Hierarchy*>(h); }

hmg_status check_level(const Hierarchy& H, int ref, const char* name) {
    if (ref < H.coarsest_ref || ref > H.fine_ref)
        return fail(HMG_ERR_INVALID_ARG, std::string(name) + ": level " + std::to_string(ref) +
                                             " outside hierarchy [" + std::to_string(H.coarsest_ref) + ", " +
                                             std::to_string(H.fine_ref) + "]");
    return HMG_OK;
}

hmg_status check_ptr(const void* p, const char* name) {
    if (!p) return fail(HMG_ERR_INVALID_ARG, std::string(name) + ": null pointer");
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
        return fail(HMG_ERR_INVALID_ARG, std::string(name) + ": must be 16-byte aligned");
    return HMG_OK;
}

// host scalar / pointer-array arguments: non-null only
hmg_status check_out(const void* p, const char* name) {
    if (!p) return fail(HMG_ERR_INVALID_ARG, std::string(name) + ": null pointer");
    return HMG_OK;
}

hmg_status check_params(const hmg_mg_params* p) {
    if (!p) return fail(HMG_ERR_INVALID_ARG, "p: null parameters");
    if (p->nu_pre < 0) return fail(HMG_ERR_INVALID_ARG, "p->nu_pre: must be >= 0");
    if (p->nu_post < 0) return fail(HMG_ERR_INVALID_ARG, "p->nu_post: must be >= 0");
    if (p->n_coarse < 1) return fail(HMG_ERR_INVALID_ARG, "p->n_coarse: must be >= 1");
    if (!std::isfinite(p->omega)) return fail(HMG_ERR_INVALID_ARG, "p->omega: must be finite");
    return HMG_OK;
}

// Reads the device singular-pivot flag (synchronises the stream).
hmg_status check_bad(const Hierarchy& H, cudaStream_t s) {
    unsigned long long bad = 0;
    HMG_CUDA(cudaMemcpyAsync(&bad, &H.scal->bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    HMG_CUDA(cudaStreamSynchronize(s));
    if (bad != ~0ull) {
        const unsigned long long reset = ~0ull;
        HMG_CUDA(cudaMemcpy(&H.scal->bad, &reset, sizeof(reset), cudaMemcpyHostToDevice));
        return fail(HMG_ERR_SINGULAR_COLUMN, "singular column: ref " + std::to_string(bad >> 40) + " column " +
                                                 std::to_string(bad & ((1ull << 40) - 1)));
    }
    return HMG_OK;
}

void free_hierarchy(Hierarchy* H) {
    if (!H) return;
    cudaSetDevice(H->device);
    for (auto& L : H->lev) {
        cudaFree(L.nbr); cudaFree(L.geom); cudaFree(L.lam); cudaFree(L.bands);
        cudaFree(L.wa); cudaFree(L.wb); cudaFree(L.b); cudaFree(L.u);
        cudaFree(L.halo_cells); cudaFree(L.halo_count); cudaFree(L.halo_loc);
        cudaFree(L.fden);
        cudaFree(L.small_cells); cudaFree(L.small_count); cudaFree(L.small_loc);
        cudaFree(L.coop_cells); cudaFree(L.coop_count); cudaFree(L.coop_loc);
        cudaFree(L.hedge); cudaFree(L.edge_e0); cudaFree(L.edge_ne); cudaFree(L.edge_hcells);
        cudaFree(L.edge_hcount); cudaFree(L.edge_loc); cudaFree(L.edge_own);
        cudaFree(L.dist.send_idx); cudaFree(L.dist.sendbuf); cudaFree(L.dist.recvbuf);
    }
    cudaFree(H->r); cudaFree(H->z); cudaFree(H->p); cudaFree(H->q); cudaFree(H->p2);
    cudaFree(H->partials); cudaFree(H->scal); cudaFree(H->hb); cudaFree(H->hx);
    cudaFree(H->hb1); cudaFree(H->hx1);
    if (H->xs) cudaStreamDestroy(H->xs);
    if (H->ev_x_go) cudaEventDestroy(H->ev_x_go);
    if (H->ev_x_done) cudaEventDestroy(H->ev_x_done);
    if (H->cs_in) cudaStreamDestroy(H->cs_in);
    if (H->cs_out) cudaStreamDestroy(H->cs_out);
    for (int i = 0; i < 2; ++i)
        for (cudaEvent_t e : {H->ev_in[i], H->ev_solved[i], H->ev_out[i]})
            if (e) cudaEventDestroy(e);
    if (H->scal_host) cudaFreeHost(H->scal_host);
    for (cudaEvent_t e : H->prof.pool) cudaEventDestroy(e);
    cudaFree(H->gbuf_send); cudaFree(H->gbuf_recv);
    mixed_free(H->mix);
    if (H->comm) {
        std::string err;
        if (const Nccl* N = nccl(&err)) N->CommDestroy(H->comm);
    }
    delete H;
}

// -------------------------------------------------------------------------
// Multi-GPU exchange.  NCCL errors are sticky: recorded here and
// reported by the next check_launch().
// -------------------------------------------------------------------------
thread_local std::string g_nccl_err;
std::string& nccl_err_ref() { return g_nccl_err; }

void nccl_check(int r, const char* what) {
    if (r == kNcclSuccess || !g_nccl_err.empty()) return;
    std::string err;
    const Nccl* N = nccl(&err);
    g_nccl_err = std::string(what) + ": " + (N ? N->GetErrorString(r) : err);
}

// Fill the halo slots of vector v on a distributed level from the owners:
// pack my owned cells each peer needs, grouped send/recv, unpack.
void halo_exchange(const Hierarchy& H, const DevLevel& L, double* v, cudaStream_t s) {
    const DistLevel& D = L.dist;
    if (!D.on || D.peer_rank.empty()) return;
    const Nccl* N = nccl(nullptr);
    launch_halo_pack(H, L, v, s);
    const int nz = H.nz;
    nccl_check(N->GroupStart(), "ncclGroupStart");
    for (size_t i = 0; i < D.peer_rank.size(); ++i) {
        if (D.send_cnt[i])
            nccl_check(N->Send(D.sendbuf + D.send_off[i] * nz, (size_t)(D.send_cnt[i] * nz), kNcclFloat64, D.peer_rank[i],
                               H.comm, s), "ncclSend");
        if (D.recv_cnt[i])
            nccl_check(N->Recv(D.recvbuf + D.recv_off[i] * nz, (size_t)(D.recv_cnt[i] * nz), kNcclFloat64, D.peer_rank[i],
                               H.comm, s), "ncclRecv");
    }
    nccl_check(N->GroupEnd(), "ncclGroupEnd");
    launch_halo_unpack(H, L, v, s);
}

// Coarse gather at gather_ref: every rank holds its owned part (global
// numbering) of vector v of the replicated level C; all-gather the rest.
void coarse_gather(const Hierarchy& H, const DevLevel& C, double* v, cudaStream_t s) {
    if (H.nranks == 1 && !H.force_coll) return;
    const int64_t cnt = C.n / H.nranks;
    launch_gather_pack(H, C, v, (int64_t)H.rank * cnt, cnt, s);
    const Nccl* N = nccl(nullptr);
    nccl_check(N->AllGather(H.gbuf_send, H.gbuf_recv, (size_t)(cnt * H.nz), kNcclFloat64, H.comm, s), "ncclAllGather");
    launch_gather_unpack(H, C, v, cnt, s);
}

}  // namespace

void hmg::dist_allreduce_tmp(const Hierarchy& H, cudaStream_t s) {
    const Nccl* N = nccl(nullptr);
    double* t = &H.scal->tmp;
    nccl_check(N->AllReduce(t, t, 1, kNcclFloat64, kNcclSum, H.comm, s), "ncclAllReduce");
}

namespace {

// -------------------------------------------------------------------------
// Sweeps on one level: `count` sweeps from `uin` (nullptr = zero guess), the
// first one adding P uc if uc != nullptr.  Intermediate iterates ping-pong
// through the level's wa/wb, always avoiding the sweep's own input (Jacobi
// semantics: every column must read the OLD neighbour values).  The last
// sweep writes `out` if given (it must not be wa/wb), else wa or wb.
// Returns the buffer holding the result.
// -------------------------------------------------------------------------
double* run_sweeps(const Hierarchy& H, const DevLevel& L, const double* b, double* uin, const double* uc,
                   int count, double* out, double omega, cudaStream_t s) {
    double* cur = uin;
    for (int i = 0; i < count; ++i) {
        double* dst = (i == count - 1 && out) ? out : (cur == L.wa ? L.wb : L.wa);
        if (cur) halo_exchange(H, L, cur, s);      // neighbours' old values (Jacobi)
        const bool last_into_out = i == count - 1 && out;
        if (last_into_out && H.rz_req && L.ref == H.fine_ref && cur && !(i == 0 && uc) && !L.fden &&
            !H.matrix_free && H.use_tc_sweep && sweep_st_supported(H, L)) {
            // the preconditioner's last sweep: <r, z> = <b, u'> accumulated on the fly
            ProfScope ps(H, kKSweep, L.ref, s);
            fin_begin(H, H.rz_op);
            H.rz_parts = launch_sweep_st_dot(H, L, b, cur, dst, omega, s);
            H.rz_req = false;
        } else {
            launch_sweep(H, L, b, cur, i == 0 ? uc : nullptr, dst, omega, s);
        }
        cur = dst;
    }
    return cur;
}

// Alg. 1 recursively (reading R9): out = V_l(b_l) with zero initial guess.
// `out` is never the level's wa/wb (it is the coarse level's u or the caller's z).
// The PCG's deferred x = x + alpha p (pcg_impl): on the side stream xs once
// the stream reaches the V-cycle's coarse part, where HBM is idle and the
// cooperative kernel leaves SMs free; `side` = false runs it on s itself.
// The side stream has low priority and its kernel is enqueued after the
// coarse-part launch, so the (cooperative) coarse kernel gets its SMs first.
void flush_pending_x(const Hierarchy& H, cudaStream_t s, bool side, bool go_recorded = false) {
    if (!H.px.pending) return;
    const DevLevel& F = H.lev[H.fine_ref];
    if (side) {
        if (!go_recorded) cudaEventRecord(H.ev_x_go, s);
        cudaStreamWaitEvent(H.xs, H.ev_x_go, 0);
        // few CTAs only while the update fits the coarse part's duration (C2: 21M dofs,
        // ~300 us); a C4-size update (168M dofs) runs at full width
        const bool trickle = H.x_slow_blocks > 0 && (int64_t)H.nz * F.n <= (32LL << 20);
        launch_update_part(H, F, trickle ? 3 : 2, H.px.first, H.px.x, H.px.p, nullptr, H.xs);
        cudaEventRecord(H.ev_x_done, H.xs);
    } else {
        launch_update_part(H, F, 2, H.px.first, H.px.x, H.px.p, nullptr, s);
    }
    H.px.pending = false;
}

void vcycle_level(const Hierarchy& H, int ref, const hmg_mg_params& p, const double* b, double* out,
                  cudaStream_t s) {
    const DevLevel& L = H.lev[ref];
    if (ref == H.coop_ref && coarse_coop_supported(H)) {   // levels <= coop_ref: one cooperative launch
        if (H.px.pending) cudaEventRecord(H.ev_x_go, s);
        launch_coarse_coop(H, p, b, out, s);
        flush_pending_x(H, s, true, true);
        return;
    }
    if (ref == H.coarsest_ref) {
        flush_pending_x(H, s, true);
        // whole coarsest level in one CTA's shared memory when it fits (ref 0: 20 columns)
        if (H.use_small_sweep && L.n <= kSmallTile && sweep_small_supported(H, L)) {
            ProfScope ps(H, kKCoarseTail, L.ref, s);
            launch_sweep_small(H, L, b, nullptr, nullptr, out, p.omega, p.n_coarse, s);
        } else if (L.fden && L.n <= 128 && coarsest_smem_bytes(H.nz, L.n, (int)((L.n + 31) / 32 * 32)) <= 200 * 1024)
            launch_coarsest(H, L, b, out, p.n_coarse, p.omega, s);
        else
            run_sweeps(H, L, b, nullptr, nullptr, p.n_coarse, out, p.omega, s);
        return;
    }
    const DevLevel& C = H.lev[ref - 1];
    // M1 presmooth from zero: the iterate stays in wa/wb through M2-M3
    double* cur = nullptr;
    if (p.nu_pre > 0) cur = run_sweeps(H, L, b, nullptr, nullptr, p.nu_pre, nullptr, p.omega, s);
    // M2 restrict the residual (b itself when u = 0)
    if (cur) {
        halo_exchange(H, L, cur, s);
        launch_resid_restrict(H, L, b, cur, C.b, s);
    } else {
        launch_restrict(H, L, b, C.b, s);
    }
    if (L.dist.on && !C.dist.on) coarse_gather(H, C, C.b, s);   // distributed -> replicated levels
    // M3 coarse correction
    vcycle_level(H, ref - 1, p, C.b, C.u, s);
    // M4 + M5: prolongation fused into the first postsmoothing sweep (single
    // GPU); on a distributed level the prolonged iterate is formed first and its
    // halo exchanged, because halo cells' parents live on other ranks
    if (!cur) {
        cudaMemsetAsync(L.wa, 0, sizeof(double) * H.nz * L.ld, s);
        cur = L.wa;
    }
    if (p.nu_post > 0 && !L.dist.on) {
        run_sweeps(H, L, b, cur, C.u, p.nu_post, out, p.omega, s);
    } else if (p.nu_post > 0) {
        double* pro = (cur == L.wa) ? L.wb : L.wa;
        launch_prolong_add(H, L, cur, C.u, pro, s);
        run_sweeps(H, L, b, pro, nullptr, p.nu_post, out, p.omega, s);
    } else {
        launch_prolong_add(H, L, cur, C.u, out, s);
    }
}

hmg_status pcg_impl(const Hierarchy& H, const hmg_mg_params* p, int single_sweeps, double single_omega,
                    const double* b, double* x, double rtol, int maxit, int* iters, double* relres,
                    cudaStream_t s) {
    const DevLevel& F = H.lev[H.fine_ref];
    const bool dist = F.dist.on;
    *iters = 0;
    *relres = 0.0;
    auto precond = [&](const double* r, double* z) {
        if (p)
            vcycle_level(H, H.fine_ref, *p, r, z, s);
        else
            run_sweeps(H, F, r, nullptr, nullptr, single_sweeps, z, single_omega, s);
    };
    // x0 = 0, r0 = b: no copies -- the first residual is b itself, and the first
    // x/r update reads b and writes x = 0 + alpha p, r = b - alpha q (the same
    // arithmetic as from x = 0, r = b)
    const double* r0 = b;
    // ||b||: on one rank the first r update sums <b, b> beside <r, r> (fused
    // finalize), so the solve starts without a dot and a host round trip; b = 0
    // is then recognised at the first convergence read (x reset to 0)
    const bool solo = !H.comm || (H.nranks == 1 && !H.force_coll);
    const bool bb_late = solo && maxit > 0;
    double bn = -1.0;
    H.res_hist.clear();
    if (!bb_late) {
        fin_begin(H, kFinBB);
        launch_dot(H, F, r0, r0, s);
        launch_finalize(H, kFinBB, s);
        HMG_TRY(check_launch());
        HMG_CUDA(cudaStreamSynchronize(s));
        bn = std::sqrt(H.scal_host->bb);
        H.res_hist.assign(1, bn == 0.0 ? 0.0 : 1.0);
        if (bn == 0.0 || maxit == 0) {            // x = x0 = 0 (and r = b: relres 1 when b != 0)
            HMG_CUDA(cudaMemset2DAsync(x, sizeof(double) * F.ld, 0, sizeof(double) * F.n, H.nz, s));
            if (bn == 0.0) return HMG_OK;
            *relres = 1.0;
            return fail(HMG_ERR_NOT_CONVERGED, "not converged after 0 iterations (relres 1)");
        }
    }
    // <r, z> after each preconditioner application: fused into its last sweep
    // when that is a streamed fine-level sweep (a fixed-order per-CTA sum, like
    // the separate dot kernel's -- PCG parity is the iteration count)
    auto precond_dot = [&](const double* r, double* z, int op) {
        H.rz_req = H.fuse_rz;
        H.rz_parts = 0;
        H.rz_op = op;
        precond(r, z);
        H.rz_req = false;
        if (H.rz_parts > 0) {
            finalize_parts(H, H.rz_parts, op, s);
        } else {
            fin_begin(H, op);
            launch_dot(H, F, r, z, s);
            launch_finalize(H, op, s);
        }
    };
    precond_dot(r0, H.z, kFinRhoInit);
    // z, p_old and p_new rotate through {z, p, p2}, so that p_1 = z_1 needs no
    // copy and p = z + beta p_old is formed inside q = H^ p.  Multi-GPU: the halo
    // of z is exchanged, and the halo slots of p_new are formed by the same
    // addition from the halos of z and p_old (k_halo_pupdate).
    double* pc = H.z;                              // current search direction
    double* zb = H.z;                              // buffer holding the current z
    // x = x + alpha p is needed only at the end: with defer_x it leaves the
    // critical path (r = r - alpha q and <r, r> stay on s), runs on the side
    // stream under the next V-cycle's coarse part, and s waits for it before
    // the next apply (which overwrites alpha and, an iteration later, p).
    bool x_inflight = false;
    auto join_x = [&]() {
        if (x_inflight) cudaStreamWaitEvent(s, H.ev_x_done, 0);
        x_inflight = false;
    };
    H.px.pending = false;
    for (int it = 1; it <= maxit; ++it) {
        join_x();
        if (it == 1) {
            if (dist) halo_exchange(H, F, pc, s);
            launch_apply_dot(H, F, pc, H.q, s);    // q = H^ p, alpha = rho / <p, q>
        } else {                                   // p = z + beta p fused into q = H^ p
            double* pn = (pc != H.p2 && zb != H.p2) ? H.p2 : ((pc != H.p && zb != H.p) ? H.p : H.z);
            if (dist) {
                halo_exchange(H, F, zb, s);
                launch_halo_pupdate(H, F, zb, pc, pn, s);
            }
            launch_apply_pupdate_dot(H, F, zb, pc, pn, H.q, s);
            pc = pn;
        }
        fin_begin(H, it == 1 && bb_late ? kFinRRBB : kFinRR);
        if (H.defer_x) {
            launch_update_part(H, F, 1, it == 1, x, pc, b, s);   // r = r - alpha q (b - alpha q), partial <r, r>
            H.px.pending = true;
            H.px.first = it == 1;
            H.px.x = x;
            H.px.p = pc;
        } else if (it == 1) {
            launch_update_xr_first(H, F, x, pc, b, s);   // x = 0 + alpha p, r = b - alpha q, partial <r, r>
        } else {
            launch_update_xr(H, F, x, pc, s);      // x += alpha p, r -= alpha q, partial <r, r>
        }
        launch_finalize(H, kFinRR, s);
        {
            // an error leaves no deferred x update behind (nor a side stream the
            // caller's stream does not wait for)
            hmg_status st = check_launch();
            const cudaError_t e = cudaStreamSynchronize(s);
            if (st != HMG_OK || e != cudaSuccess) {
                H.px.pending = false;
                join_x();
                if (st != HMG_OK) return st;
                return fail(HMG_ERR_CUDA, std::string("cudaStreamSynchronize: ") + cudaGetErrorString(e));
            }
        }
        if (H.scal_host->bad != ~0ull) {
            H.px.pending = false;
            return check_bad(H, s);
        }
        if (bn < 0.0) {                            // the first read: ||b|| (bb_late)
            bn = std::sqrt(H.scal_host->bb);
            H.res_hist.assign(1, bn == 0.0 ? 0.0 : 1.0);
            if (bn == 0.0) {                       // b = 0: x = x0 = 0 (the iteration's scalars were 0/0)
                H.px.pending = false;
                HMG_CUDA(cudaMemset2DAsync(x, sizeof(double) * F.ld, 0, sizeof(double) * F.n, H.nz, s));
                HMG_CUDA(cudaStreamSynchronize(s));
                *iters = 0;
                *relres = 0.0;
                return HMG_OK;
            }
        }
        const double rn = std::sqrt(H.scal_host->rr);
        *iters = it;
        *relres = rn / bn;
        H.res_hist.push_back(rn / bn);
        if (rn <= rtol * bn) {
            flush_pending_x(H, s, false);          // the last x update, in stream order
            HMG_TRY(check_launch());
            return HMG_OK;
        }
        zb = (pc != H.z) ? H.z : H.p;              // a buffer that is not p
        x_inflight = H.px.pending;                 // launched on xs inside the V-cycle (or below)
        precond_dot(H.r, zb, kFinRZ);              // beta = rho' / rho, rho = rho' (p updated in the next apply)
        if (H.px.pending) {                        // preconditioner without a coarse part
            flush_pending_x(H, s, false);
            x_inflight = false;
        }
    }
    join_x();
    return fail(HMG_ERR_NOT_CONVERGED, "not converged after " + std::to_string(maxit) +
                                           " iterations (relres " + std::to_string(*relres) + ")");
}


// ---------------------------------------------------------------------------
// Hierarchy construction (single GPU, or one rank of a distributed hierarchy).
// ---------------------------------------------------------------------------
hmg_status build_impl(int fine_ref, int coarsest_ref, int nlayers, double thickness, double w2, double omega_n,
                      const double* lam_host, int device, const hmg_dist* dist, hmg_hierarchy** out) {
    g_err.clear();
    if (!out) return fail(HMG_ERR_INVALID_ARG, "out: null pointer");
    *out = nullptr;
    if (fine_ref < 0 || fine_ref > kMaxRef)
        return fail(HMG_ERR_INVALID_ARG, "fine_ref: must be in [0, 10], got " + std::to_string(fine_ref));
    if (coarsest_ref < 0 || coarsest_ref > fine_ref)
        return fail(HMG_ERR_INVALID_ARG, "coarsest_ref: must be in [0, fine_ref], got " + std::to_string(coarsest_ref));
    if (nlayers < 1 || nlayers > kMaxLayers)
        return fail(HMG_ERR_INVALID_ARG, "nlayers: must be in [1, 256], got " + std::to_string(nlayers));
    if (!(thickness > 0) || !std::isfinite(thickness)) return fail(HMG_ERR_INVALID_ARG, "thickness: must be > 0 and finite");
    if (!(w2 >= 0) || !std::isfinite(w2)) return fail(HMG_ERR_INVALID_ARG, "w2: must be >= 0 and finite");
    if (!(omega_n >= 0) || !std::isfinite(omega_n))
        return fail(HMG_ERR_INVALID_ARG, "omega_n: must be >= 0 and finite");
    if (!lam_host) return fail(HMG_ERR_INVALID_ARG, "lam_host: null pointer");
    int rank = 0, nranks = 1, gather_ref = fine_ref;
    if (dist) {
        rank = dist->rank;
        nranks = dist->nranks;
        gather_ref = dist->gather_ref;
        if (nranks < 1 || 320 % nranks != 0) return fail(HMG_ERR_INVALID_ARG, "dist->nranks: must divide 320");
        if (rank < 0 || rank >= nranks) return fail(HMG_ERR_INVALID_ARG, "dist->rank: must be in [0, nranks)");
        if (!dist->nccl_id) return fail(HMG_ERR_INVALID_ARG, "dist->nccl_id: null pointer");
        if (gather_ref < std::max(2, coarsest_ref) || gather_ref > fine_ref)
            return fail(HMG_ERR_INVALID_ARG, "dist->gather_ref: must be in [max(2, coarsest_ref), fine_ref]");
        if (nranks > 1 && gather_ref >= fine_ref)   // every level replicated: nothing to distribute
            return fail(HMG_ERR_INVALID_ARG, "dist->gather_ref: must be < fine_ref when nranks > 1");
    }
    // lam_host: the finest level, [nlayers][20*4^fine_ref] (single GPU) or this
    // rank's owned cells [nlayers][20*4^fine_ref/nranks] (distributed, when
    // gather_ref < fine_ref) -- see include/hmg.h
    const int64_t nfine = 20 * (int64_t(1) << (2 * fine_ref));
    const bool dist_fine = dist && gather_ref < fine_ref;
    const int64_t nlam = dist_fine ? nfine / nranks : nfine;
    double lam_min = HUGE_VAL, lam_max = 0.0;
    for (int64_t i = 0; i < nlam * nlayers; ++i) {
        if (!(lam_host[i] > 0) || !std::isfinite(lam_host[i]))
            return fail(HMG_ERR_INVALID_ARG, "lam_host: entry " + std::to_string(i) + " is not finite and > 0");
        lam_min = std::min(lam_min, lam_host[i]);
        lam_max = std::max(lam_max, lam_host[i]);
    }
    int ndev = 0;
    HMG_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(HMG_ERR_INVALID_ARG, "device: no CUDA device " + std::to_string(device));
    HMG_CUDA(cudaSetDevice(device));

    Hierarchy* H = new (std::nothrow) Hierarchy();
    if (!H) return fail(HMG_ERR_OOM, "host allocation");
    H->device = device;
    H->fine_ref = fine_ref;
    H->coarsest_ref = coarsest_ref;
    H->nz = nlayers;
    H->thickness = thickness;
    H->w2 = w2;
    H->dz = thickness / nlayers;
    H->sn = 1.0 + omega_n * omega_n;
    H->rank = rank;
    H->nranks = nranks;
    H->gather_ref = dist ? gather_ref : -1;
    // Test knobs (the only environment switches; tests/ use each one): route a
    // one-rank hierarchy through every collective, the matrix-free operator
    // (NEXT-2), the deferred CG x update and its CTA count, the threshold of
    // the edge-deduplicated coupling store, and HMG_COOP_REF below.
    if (const char* e = std::getenv("HMG_FORCE_COLLECTIVES")) H->force_coll = dist && std::string(e) == "1";
    if (const char* e = std::getenv("HMG_OPERATOR")) H->matrix_free = std::string(e) == "free";
    if (H->matrix_free && H->sn != 1.0) {
        delete H;
        return fail(HMG_ERR_INVALID_ARG, "omega_n: the matrix-free operator (HMG_OPERATOR=free) needs omega_n = 0");
    }
    if (const char* e = std::getenv("HMG_DEFER_X")) H->defer_x = std::string(e) != "0";
    if (const char* e = std::getenv("HMG_X_BLOCKS")) H->x_slow_blocks = std::atoi(e);
    if (const char* e = std::getenv("HMG_EDGE_MIN_DOFS")) H->edge_min_dofs = std::atoll(e);
    {
        // Cooperative coarse tail (coarse_coop.cu): by default every level of at
        // most kCoopMaxCells cells runs in one cooperative launch -- those levels
        // are latency-bound (a sweep is a 2 x nz-step dependency chain, ~4 us,
        // against ~3 us per dependent kernel launch).  HMG_COOP_REF=r overrides
        // (-1: off).  It never spans distributed levels.
        int coop = coarsest_ref;
        const int ctw = coarse_coop_tile_width(nlayers);   // narrower tiles for deep columns
        const int64_t coop_max = kCoopMaxCells * (ctw > 0 ? ctw : kSmallTile) / kSmallTile;
        while (coop < fine_ref && 20LL * (1LL << (2 * (coop + 1))) <= coop_max) ++coop;
        if (const char* e = std::getenv("HMG_COOP_REF")) coop = std::atoi(e);
        H->coop_ref = coop < 0 ? -1 : std::min(std::max(coop, coarsest_ref), dist ? gather_ref : fine_ref);
    }
    if (H->use_tc_sweep && !tensor_maps_available()) {
        delete H;
        return fail(HMG_ERR_CUDA, "cuTensorMapEncodeTiled not available from the CUDA driver");
    }
    auto cleanup = [&](hmg_status s2) { free_hierarchy(H); return s2; };
#define BCUDA(call)                                                                         \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return cleanup(fail(e_ == cudaErrorMemoryAllocation ? HMG_ERR_OOM : HMG_ERR_CUDA, \
                                std::string(#call) + ": " + cudaGetErrorString(e_)));      \
    } while (0)
    if (dist) {
        std::string err;
        const Nccl* N = nccl(&err);
        if (!N) return cleanup(fail(HMG_ERR_NCCL, err));
        NcclUniqueId id;
        std::memcpy(id.internal, dist->nccl_id, sizeof(id.internal));
        const int r = N->CommInitRank(&H->comm, nranks, id, rank);
        if (r != kNcclSuccess) return cleanup(fail(HMG_ERR_NCCL, std::string("ncclCommInitRank: ") + N->GetErrorString(r)));
    }

    std::vector<HostLevel> host;
    try {
        host = build_icosahedral_levels(fine_ref);
    } catch (const std::exception& e) {
        return cleanup(fail(HMG_ERR_INVALID_ARG, std::string("mesh: ") + e.what()));
    }
    // Distributed: all levels' coefficients on the host (4-child means, reading
    // R3, same formula), because halo cells need their neighbours' values.
    std::vector<std::vector<double>> lam_levels;
    if (dist) {
        lam_levels.resize(fine_ref + 1);
        lam_levels[fine_ref].assign(lam_host, lam_host + nlam * nlayers);
        if (dist_fine) {
            // the fine level arrives distributed: gather it (host staging through the device)
            const int64_t per = nfine / nranks;
            std::vector<double> full((size_t)nfine * nlayers);
            double *dsend = nullptr, *drecv = nullptr;
            BCUDA(cudaMalloc(&dsend, sizeof(double) * per * nlayers));
            BCUDA(cudaMalloc(&drecv, sizeof(double) * nfine * nlayers));
            BCUDA(cudaMemcpy(dsend, lam_host, sizeof(double) * per * nlayers, cudaMemcpyHostToDevice));
            std::string err;
            const Nccl* N = nccl(&err);
            const int r = N->AllGather(dsend, drecv, (size_t)per * nlayers, kNcclFloat64, H->comm, nullptr);
            if (r != kNcclSuccess) return cleanup(fail(HMG_ERR_NCCL, std::string("ncclAllGather: ") + N->GetErrorString(r)));
            BCUDA(cudaDeviceSynchronize());
            std::vector<double> stage((size_t)nfine * nlayers);
            BCUDA(cudaMemcpy(stage.data(), drecv, sizeof(double) * nfine * nlayers, cudaMemcpyDeviceToHost));
            cudaFree(dsend);
            cudaFree(drecv);
            for (int q = 0; q < nranks; ++q)            // [q][nz][per] -> [nz][nfine]
                for (int k = 0; k < nlayers; ++k)
                    std::memcpy(&full[(size_t)k * nfine + (size_t)q * per], &stage[((size_t)q * nlayers + k) * per],
                                sizeof(double) * per);
            lam_levels[fine_ref] = std::move(full);
        }
        for (int r = fine_ref - 1; r >= coarsest_ref; --r) {
            const int64_t nf = host[r + 1].n, nc = host[r].n;
            lam_levels[r].resize((size_t)nc * nlayers);
            for (int k = 0; k < nlayers; ++k)
                for (int64_t p = 0; p < nc; ++p) {
                    const double* l = &lam_levels[r + 1][(size_t)k * nf + 4 * p];
                    lam_levels[r][(size_t)k * nc + p] = 0.25 * (((l[0] + l[1]) + l[2]) + l[3]);
                }
        }
    }
    H->lev.resize(fine_ref + 1);
    cudaStream_t s = nullptr;
    for (int r = coarsest_ref; r <= fine_ref; ++r) {
        DevLevel& L = H->lev[r];
        const HostLevel& HL = host[r];
        L.ref = r;
        const bool distributed = dist && r > gather_ref;
        LevelPlan plan;
        if (distributed) plan = plan_level(r, HL.nbr, rank, nranks);
        const int64_t off = distributed ? plan.off : 0;
        L.n = distributed ? plan.n_own : HL.n;
        const int64_t nh = distributed ? plan.n_halo() : 0;
        L.ld = round_up32(L.n + nh);
        const std::vector<int32_t>& nbl = distributed ? plan.nbr_local : HL.nbr;
        const size_t vb = sizeof(double) * nlayers * L.ld;
        // SoA neighbour table and geometry of the owned cells; padding points at cell 0 / is zero
        std::vector<int32_t> nbr(3 * L.ld, 0);
        std::vector<double> geom(7 * L.ld, 0.0);
        for (int64_t c = 0; c < L.n; ++c) {
            const int64_t g = off + c;
            geom[c] = HL.area[g];
            for (int j = 0; j < 3; ++j) {
                nbr[j * L.ld + c] = nbl[c * 3 + j];
                geom[(1 + j) * L.ld + c] = HL.len[g * 3 + j];
                geom[(4 + j) * L.ld + c] = HL.cd[g * 3 + j];
            }
        }
        BCUDA(cudaMalloc(&L.nbr, sizeof(int32_t) * 3 * L.ld));
        BCUDA(cudaMalloc(&L.geom, sizeof(double) * 7 * L.ld));
        BCUDA(cudaMalloc(&L.lam, vb));
        BCUDA(cudaMalloc(&L.bands, 5 * vb));
        BCUDA(cudaMalloc(&L.wa, vb));
        BCUDA(cudaMalloc(&L.wb, vb));
        BCUDA(cudaMemset(L.lam, 0, vb));
        BCUDA(cudaMemset(L.bands, 0, 5 * vb));
        BCUDA(cudaMemset(L.wa, 0, vb));
        BCUDA(cudaMemset(L.wb, 0, vb));
        if (r < fine_ref) {
            BCUDA(cudaMalloc(&L.b, vb));
            BCUDA(cudaMalloc(&L.u, vb));
            BCUDA(cudaMemset(L.b, 0, vb));
            BCUDA(cudaMemset(L.u, 0, vb));
        }
        BCUDA(cudaMemcpy(L.nbr, nbr.data(), sizeof(int32_t) * 3 * L.ld, cudaMemcpyHostToDevice));
        BCUDA(cudaMemcpy(L.geom, geom.data(), sizeof(double) * 7 * L.ld, cudaMemcpyHostToDevice));
        if (!dist) {
            // Matrix-free couplings without the per-quotient fast-path test
            // (mf_ops.cuh): prove every numerator, divisor and quotient of this
            // level within [2^-900, 2^900].  Coarse coefficients are means of
            // fine ones, so the fine range [lam_min, lam_max] bounds every level.
            double amin = HUGE_VAL, amax = 0, lmn = HUGE_VAL, lmx = 0, cmn = HUGE_VAL, cmx = 0;
            for (int64_t g = 0; g < HL.n; ++g) {
                amin = std::min(amin, HL.area[g]);
                amax = std::max(amax, HL.area[g]);
                for (int j = 0; j < 3; ++j) {
                    lmn = std::min(lmn, HL.len[g * 3 + j]);
                    lmx = std::max(lmx, HL.len[g * 3 + j]);
                    cmn = std::min(cmn, HL.cd[g * 3 + j]);
                    cmx = std::max(cmx, HL.cd[g * 3 + j]);
                }
            }
            auto in = [](double v) { return v >= 0x1p-900 && v <= 0x1p900; };
            const double nv0 = w2 * amin * lam_min, nv1 = w2 * amax * lam_max;
            const double dz = H->dz;
            const double nh0 = w2 * lmn * dz * lam_min, nh1 = w2 * lmx * dz * lam_max;
            L.mf_safe = w2 == 0.0 ||
                        (in(dz) && in(cmn) && in(cmx) && in(nv0) && in(nv1) && in(nh0) && in(nh1) && in(nv0 / dz) &&
                         in(nv1 / dz) && in(nh0 / cmx) && in(nh1 / cmn));
        }
        if (dist) {      // coefficients: owned + halo cells from the host copy
            std::vector<double> lam((size_t)nlayers * L.ld, 1.0);
            const std::vector<double>& G = lam_levels[r];
            for (int k = 0; k < nlayers; ++k) {
                for (int64_t c = 0; c < L.n; ++c) lam[(size_t)k * L.ld + c] = G[(size_t)k * HL.n + off + c];
                for (int64_t h = 0; h < nh; ++h) lam[(size_t)k * L.ld + L.n + h] = G[(size_t)k * HL.n + plan.halo_gid[h]];
            }
            BCUDA(cudaMemcpy(L.lam, lam.data(), vb, cudaMemcpyHostToDevice));
        }
        if (distributed) {
            DistLevel& D = L.dist;
            D.on = true;
            D.off = off;
            D.n_halo = nh;
            std::vector<int32_t> sidx;
            for (const PeerPlan& q : plan.peers) {
                D.peer_rank.push_back(q.rank);
                D.send_off.push_back((int64_t)sidx.size());
                D.send_cnt.push_back((int64_t)q.send_local.size());
                D.recv_off.push_back(q.recv_offset);
                D.recv_cnt.push_back(q.recv_count);
                sidx.insert(sidx.end(), q.send_local.begin(), q.send_local.end());
            }
            D.send_total = (int64_t)sidx.size();
            if (D.send_total) {
                BCUDA(cudaMalloc(&D.send_idx, sizeof(int32_t) * sidx.size()));
                BCUDA(cudaMemcpy(D.send_idx, sidx.data(), sizeof(int32_t) * sidx.size(), cudaMemcpyHostToDevice));
                BCUDA(cudaMalloc(&D.sendbuf, sizeof(double) * D.send_total * nlayers));
            }
            if (nh) BCUDA(cudaMalloc(&D.recvbuf, sizeof(double) * nh * nlayers));
            // coarser level replicated: its vectors use global numbering
            D.coff = (r - 1 <= gather_ref) ? off / 4 : 0;
        }
        // tile halos: 128-cell tiles of the streamed sweep (sweep_tc.cu) and
        // 32-cell tiles of the small-level sweep (sweep_small.cu)
        auto build_halo = [&](int tile, int hmax, int32_t** d_cells, int32_t** d_count, uint32_t** d_loc) -> hmg_status {
            const int64_t ntiles = (L.n + tile - 1) / tile;
            std::vector<int32_t> hcells(ntiles * hmax, 0), hcount(ntiles, 0);
            std::vector<uint32_t> loc(L.ld, 0);
            for (int64_t t = 0; t < ntiles; ++t) {
                const int64_t a = t * tile, e = std::min<int64_t>(L.n, a + tile);
                std::vector<int32_t> outs;
                for (int64_t c = a; c < e; ++c)
                    for (int j = 0; j < 3; ++j) {
                        const int32_t o = nbl[c * 3 + j];
                        if (o < a || o >= e) outs.push_back(o);
                    }
                std::sort(outs.begin(), outs.end());
                outs.erase(std::unique(outs.begin(), outs.end()), outs.end());
                if ((int)outs.size() > hmax) return HMG_OK;        // table not usable: kernel not selected
                hcount[t] = (int32_t)outs.size();
                std::copy(outs.begin(), outs.end(), hcells.begin() + t * hmax);
                for (int64_t c = a; c < e; ++c) {
                    uint32_t packed = 0;
                    for (int j = 0; j < 3; ++j) {
                        const int32_t o = nbl[c * 3 + j];
                        uint32_t slot;
                        if (o >= a && o < e)
                            slot = (uint32_t)(o - a);
                        else
                            slot = tile + (uint32_t)(std::lower_bound(outs.begin(), outs.end(), o) - outs.begin());
                        packed |= slot << (8 * j);
                    }
                    loc[c] = packed;
                }
            }
            HMG_CUDA(cudaMalloc(d_cells, sizeof(int32_t) * hcells.size()));
            HMG_CUDA(cudaMalloc(d_count, sizeof(int32_t) * hcount.size()));
            HMG_CUDA(cudaMalloc(d_loc, sizeof(uint32_t) * loc.size()));
            HMG_CUDA(cudaMemcpy(*d_cells, hcells.data(), sizeof(int32_t) * hcells.size(), cudaMemcpyHostToDevice));
            HMG_CUDA(cudaMemcpy(*d_count, hcount.data(), sizeof(int32_t) * hcount.size(), cudaMemcpyHostToDevice));
            HMG_CUDA(cudaMemcpy(*d_loc, loc.data(), sizeof(uint32_t) * loc.size(), cudaMemcpyHostToDevice));
            return HMG_OK;
        };
        {
            hmg_status hs = build_halo(kSweepTile, kHaloMax, &L.halo_cells, &L.halo_count, &L.halo_loc);
            if (hs != HMG_OK) return cleanup(hs);
            L.halo.cells = L.halo_cells;
            L.halo.count = L.halo_count;
            L.halo.loc = L.halo_loc;
            if (L.n <= kFactMaxCells) {
                hs = build_halo(kSmallTile, kSmallHaloMax, &L.small_cells, &L.small_count, &L.small_loc);
                if (hs != HMG_OK) return cleanup(hs);
                L.small.cells = L.small_cells;
                L.small.count = L.small_count;
                L.small.loc = L.small_loc;
            }
            // edge-deduplicated couplings for the streamed sweep (levels without
            // precomputed Thomas factors, i.e. the ones k_sweep_st serves)
            // only where the streamed kernels are bound by HBM bandwidth (>= 16M dofs
            // on the level); on smaller levels they are bound by the consumers' per-layer
            // work and the extra copies cost more than the bytes saved (measured at ref 6)
            if (H->edge_h && L.n > H->fact_max_cells && L.halo.loc && L.n * nlayers >= H->edge_min_dofs) {
                const int64_t n = L.n, ntl = (n + kSweepTile - 1) / kSweepTile;
                std::vector<int64_t> eown(n + 1, 0);
                for (int64_t c = 0; c < n; ++c) {
                    int cnt = 0;
                    for (int j = 0; j < 3; ++j) cnt += nbl[c * 3 + j] > c;
                    eown[c + 1] = eown[c] + cnt;
                }
                const int64_t nE = eown[n], ldE = round_up32(nE);
                std::vector<int32_t> eid(3 * n), own(2 * ldE, 0);
                for (int64_t c = 0; c < n; ++c) {
                    int64_t q = eown[c];
                    for (int j = 0; j < 3; ++j) {
                        const int32_t o = nbl[c * 3 + j];
                        if (o > c) {
                            eid[3 * c + j] = (int32_t)q;
                            own[q] = (int32_t)c;
                            own[ldE + q] = j;
                            ++q;
                        }
                    }
                }
                for (int64_t c = 0; c < n; ++c)
                    for (int j = 0; j < 3; ++j) {
                        const int32_t o = nbl[c * 3 + j];
                        if (o < c) {                     // owned by o (< c, so owned, not a halo slot)
                            int jo = 0;
                            while (jo < 3 && nbl[o * 3 + jo] != (int32_t)c) ++jo;
                            int64_t q = eown[o];
                            for (int i = 0; i < jo; ++i) q += nbl[o * 3 + i] > o;
                            eid[3 * c + j] = (int32_t)q;
                        }
                    }
                std::vector<int32_t> e0(ntl), nel(ntl), hc(ntl * kEdgeHalo, 0), hn(ntl, 0);
                std::vector<uint32_t> eloc(L.ld, 0);
                bool ok = true;
                for (int64_t t = 0; t < ntl && ok; ++t) {
                    const int64_t a = t * kSweepTile, e = std::min<int64_t>(n, a + kSweepTile);
                    const int64_t lo = eown[a] & ~int64_t(1), hi = (eown[e] + 1) & ~int64_t(1);
                    if (hi - lo > kEdgeRange) ok = false;
                    e0[t] = (int32_t)lo;
                    nel[t] = (int32_t)(hi - lo);
                    for (int64_t c = a; c < e && ok; ++c) {
                        uint32_t packed = 0;
                        for (int j = 0; j < 3; ++j) {
                            const int32_t id = eid[3 * c + j];
                            uint32_t off;
                            if (id >= eown[a] && id < eown[e]) {
                                off = (uint32_t)(id - lo);
                            } else {
                                if (hn[t] >= kEdgeHalo) { ok = false; break; }
                                hc[t * kEdgeHalo + hn[t]] = id;
                                off = (uint32_t)(kEdgeRange + hn[t]);
                                ++hn[t];
                            }
                            packed |= off << (8 * j);
                        }
                        eloc[c] = packed;
                    }
                }
                if (ok) {
                    auto up = [&](auto** dst, const auto& src) -> bool {
                        using T = typename std::decay_t<decltype(src)>::value_type;
                        return cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * src.size()) == cudaSuccess &&
                               cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice) ==
                                   cudaSuccess;
                    };
                    if (!(up(&L.edge_e0, e0) && up(&L.edge_ne, nel) && up(&L.edge_hcells, hc) &&
                          up(&L.edge_hcount, hn) && up(&L.edge_loc, eloc) && up(&L.edge_own, own)))
                        return cleanup(fail(HMG_ERR_OOM, "edge tables: device allocation failed"));
                    BCUDA(cudaMalloc(&L.hedge, sizeof(double) * nlayers * ldE));
                    BCUDA(cudaMemset(L.hedge, 0, sizeof(double) * nlayers * ldE));
                    L.edge.H = L.hedge;
                    L.edge.ldE = ldE;
                    L.edge.e0 = L.edge_e0;
                    L.edge.ne = L.edge_ne;
                    L.edge.hcells = L.edge_hcells;
                    L.edge.hcount = L.edge_hcount;
                    L.edge.loc = L.edge_loc;
                    L.edge_count = nE;
                }
            }
            const int ctw = coarse_coop_tile_width(nlayers);
            if (r <= H->coop_ref && ctw == kSmallTile) {
                L.coop_halo = L.small;
            } else if (r <= H->coop_ref && ctw > 0) {
                hs = build_halo(ctw, kSmallHaloMax, &L.coop_cells, &L.coop_count, &L.coop_loc);
                if (hs != HMG_OK) return cleanup(hs);
                L.coop_halo.cells = L.coop_cells;
                L.coop_halo.count = L.coop_count;
                L.coop_halo.loc = L.coop_loc;
            }
        }
    }
    host.clear();
    DevLevel& F = H->lev[fine_ref];
    if (!dist) {
        // fine coefficients (dense host rows -> padded device rows), coarse by 4-child means
        BCUDA(cudaMemcpy2D(F.lam, sizeof(double) * F.ld, lam_host, sizeof(double) * F.n, sizeof(double) * F.n, nlayers,
                           cudaMemcpyHostToDevice));
        for (int r = fine_ref - 1; r >= coarsest_ref; --r) launch_coarsen_lam(*H, H->lev[r + 1], H->lev[r], s);
    }
    for (int r = coarsest_ref; r <= fine_ref; ++r) {
        launch_assemble(*H, H->lev[r], s);
        if (H->lev[r].hedge) launch_edge_h(*H, H->lev[r], H->lev[r].edge_count, s);
    }
    // PCG workspace
    const size_t fb = sizeof(double) * nlayers * F.ld;
    for (double** v : {&H->r, &H->z, &H->p, &H->q, &H->p2}) {
        BCUDA(cudaMalloc(v, fb));
        BCUDA(cudaMemset(*v, 0, fb));
    }
    H->npartials = 2 * partials_needed(F.n, nlayers) + 148 * 8 + 64;   // x 2: the first r update's <r, r> and <b, b>
    BCUDA(cudaMalloc(&H->partials, sizeof(double) * H->npartials));
    {
        int lo = 0, hi = 0;
        BCUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));   // lo: the least urgent
        BCUDA(cudaStreamCreateWithPriority(&H->xs, cudaStreamNonBlocking, lo));
    }
    BCUDA(cudaEventCreateWithFlags(&H->ev_x_go, cudaEventDisableTiming));
    BCUDA(cudaEventCreateWithFlags(&H->ev_x_done, cudaEventDisableTiming));
    BCUDA(cudaMalloc(&H->scal, sizeof(PcgScalars)));
    BCUDA(cudaHostAlloc(&H->scal_host, sizeof(PcgScalars), cudaHostAllocMapped));
    BCUDA(cudaHostGetDevicePointer(&H->scal_pub, H->scal_host, 0));
    PcgScalars init{};
    init.bad = ~0ull;
    BCUDA(cudaMemcpy(H->scal, &init, sizeof(init), cudaMemcpyHostToDevice));
    if (dist && gather_ref < fine_ref) {      // coarse-gather staging at gather_ref
        const DevLevel& C = H->lev[gather_ref];
        const int64_t cnt = C.n / nranks;
        BCUDA(cudaMalloc(&H->gbuf_send, sizeof(double) * cnt * nlayers));
        BCUDA(cudaMalloc(&H->gbuf_recv, sizeof(double) * C.n * nlayers));
    }
    // Thomas factors (matrix-only; computed once) for the coarse-tail levels and
    // for every level too small to fill the GPU (latency-bound sweeps)
    for (int r = coarsest_ref; r <= fine_ref; ++r) {
        DevLevel& L = H->lev[r];
        if (!(r <= H->coop_ref || L.n <= H->fact_max_cells)) continue;
        const size_t vb = sizeof(double) * nlayers * L.ld;
        BCUDA(cudaMalloc(&L.fden, 3 * vb));          // [3][nz][ld]: den, y, g (one TMA box)
        L.fy = L.fden + (size_t)nlayers * L.ld;
        L.fg = L.fy + (size_t)nlayers * L.ld;
        launch_factor(*H, L, s);
    }
    {
        // every other level: pivots checked once, g_k fast-path exactness recorded
        unsigned int* gslow = nullptr;
        BCUDA(cudaMalloc(&gslow, sizeof(unsigned int) * (fine_ref + 1)));
        BCUDA(cudaMemset(gslow, 0, sizeof(unsigned int) * (fine_ref + 1)));
        for (int r = coarsest_ref; r <= fine_ref; ++r)
            if (!H->lev[r].fden) launch_pivot_check(*H, H->lev[r], gslow + r, s);
        std::vector<unsigned int> gs(fine_ref + 1, 1u);
        BCUDA(cudaMemcpy(gs.data(), gslow, sizeof(unsigned int) * (fine_ref + 1), cudaMemcpyDeviceToHost));
        cudaFree(gslow);
        for (int r = coarsest_ref; r <= fine_ref; ++r)
            H->lev[r].g_safe = !H->lev[r].fden && gs[r] == 0 && H->check_skip;
    }
    BCUDA(cudaGetLastError());
    BCUDA(cudaDeviceSynchronize());
    {
        unsigned long long bad = 0;
        BCUDA(cudaMemcpy(&bad, &H->scal->bad, sizeof(bad), cudaMemcpyDeviceToHost));
        if (bad != ~0ull)
            return cleanup(fail(HMG_ERR_SINGULAR_COLUMN, "singular column: ref " + std::to_string(bad >> 40) +
                                                             " column " + std::to_string(bad & ((1ull << 40) - 1))));
    }
#undef BCUDA
    *out = reinterpret_cast<hmg_hierarchy*>(H);
    return HMG_OK;
}

// NEXT-4 (mixed.cu): restarted right-preconditioned GMRES(m) on the mixed
// system (reading R20), the oracle's ora_mixed_gmres step for step: classical
// Gram-Schmidt applied gs_passes times (2 = CGS2, the default) against one w, Givens rotations and the small triangular solve
// on the host, every vector operation in mixed.cu's kernels.  Dot products
// are deterministic block trees (the oracle's are sequential): parity is the
// iteration count.
hmg_status mixed_gmres_impl(const Hierarchy& H, const hmg_mg_params* p, const double* F, double* X, double rtol,
                            int m, int maxit, int gs_passes, int* iters, double* relres, cudaStream_t s) {
    MixedSystem& M = *H.mix;
    const int64_t N = M.ntot;
    if (M.m < m) {
        cudaFree(M.V); cudaFree(M.w); cudaFree(M.z); cudaFree(M.t);
        M.V = M.w = M.z = M.t = nullptr;
        M.m = 0;
        HMG_CUDA(cudaMalloc(&M.V, sizeof(double) * N * (m + 1)));
        HMG_CUDA(cudaMalloc(&M.w, sizeof(double) * N));
        HMG_CUDA(cudaMalloc(&M.z, sizeof(double) * N));
        HMG_CUDA(cudaMalloc(&M.t, sizeof(double) * N));
        M.m = m;
    }
    // padding entries of every work vector stay zero
    HMG_CUDA(cudaMemsetAsync(M.V, 0, sizeof(double) * N * (M.m + 1), s));
    HMG_CUDA(cudaMemsetAsync(M.z, 0, sizeof(double) * N, s));
    HMG_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * N, s));
    HMG_CUDA(cudaMemcpyAsync(M.t, F, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    F = M.t;                       // library copy: 16-byte aligned for the vector kernels
    *iters = 0;
    *relres = 0.0;
    auto fetch = [&](int nv) -> hmg_status {
        HMG_CUDA(cudaMemcpyAsync(M.dots_host, M.dots, sizeof(double) * nv, cudaMemcpyDeviceToHost, s));
        HMG_TRY(check_launch());
        HMG_CUDA(cudaStreamSynchronize(s));
        return HMG_OK;
    };
    auto norm = [&](const double* a, double* out) -> hmg_status {
        mixed_dots(H, a, nullptr, 0, 2, s);
        HMG_TRY(fetch(1));
        *out = std::sqrt(M.dots_host[0]);
        return HMG_OK;
    };
    double fn = 0.0;
    HMG_TRY(norm(F, &fn));
    if (fn == 0.0) return HMG_OK;
    HMG_CUDA(cudaMemcpyAsync(M.w, F, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    std::vector<double> Hm((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), yv(m);
    std::vector<const double*> vp(m + 1);
    for (int i = 0; i <= m; ++i) vp[i] = M.V + (int64_t)i * N;
    double beta = fn;
    int total = 0;
    while (total < maxit) {
        mixed_vec(H, 0, M.w, nullptr, beta, M.V, s);          // v_0 = r / beta
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int j;
        for (j = 0; j < m && total < maxit; ++j) {
            mixed_precond(H, p, vp[j], M.z, s);                // w = A M^-1 v_j
            launch_mixed_apply(H, M.z, M.w, s);
            for (int pass = 0; pass < gs_passes; ++pass) {     // CGS (1) or CGS2 (2, the default)
                mixed_dots(H, M.w, vp.data(), j + 1, 1, s);    // c_i = <v_i, w>, i <= j
                HMG_TRY(fetch(j + 1));
                for (int i = 0; i <= j; ++i) {
                    yv[i] = M.dots_host[i];
                    Hm[(size_t)i * m + j] = pass == 0 ? yv[i] : Hm[(size_t)i * m + j] + yv[i];
                }
                mixed_update(H, M.w, M.w, vp.data(), yv.data(), j + 1, false, s);
            }
            double hn = 0.0;
            HMG_TRY(norm(M.w, &hn));
            Hm[(size_t)(j + 1) * m + j] = hn;
            mixed_vec(H, 0, M.w, nullptr, hn, const_cast<double*>(vp[j + 1]), s);
            for (int i = 0; i < j; ++i) {
                const double a = Hm[(size_t)i * m + j], b = Hm[(size_t)(i + 1) * m + j];
                Hm[(size_t)i * m + j] = cs[i] * a + sn[i] * b;
                Hm[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
            }
            const double a = Hm[(size_t)j * m + j], b = Hm[(size_t)(j + 1) * m + j];
            const double rr = std::sqrt(a * a + b * b);
            cs[j] = a / rr;
            sn[j] = b / rr;
            Hm[(size_t)j * m + j] = rr;
            Hm[(size_t)(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++total;
            if (std::fabs(g[j + 1]) <= rtol * fn) {
                ++j;
                break;
            }
        }
        for (int i = j - 1; i >= 0; --i) {                    // y = H^-1 g
            double sm = g[i];
            for (int l = i + 1; l < j; ++l) sm = sm - Hm[(size_t)i * m + l] * yv[l];
            yv[i] = sm / Hm[(size_t)i * m + i];
        }
        mixed_update(H, nullptr, M.w, vp.data(), yv.data(), j, true, s);    // w = V y
        mixed_precond(H, p, M.w, M.z, s);                      // x += M^-1 (V y)
        mixed_vec(H, 2, M.z, nullptr, 0.0, X, s);
        launch_mixed_apply(H, X, M.z, s);                      // r = F - A x
        mixed_vec(H, 1, F, M.z, 0.0, M.w, s);
        HMG_TRY(norm(M.w, &beta));
        *iters = total;
        *relres = beta / fn;
        if (beta <= rtol * fn) return HMG_OK;
    }
    return fail(HMG_ERR_NOT_CONVERGED, "GMRES not converged after " + std::to_string(maxit) + " iterations (relres " +
                                           std::to_string(*relres) + ")");
}

hmg_status ensure_mixed(const Hierarchy& H) {
    if (H.mix) return HMG_OK;
    const std::string e = mixed_setup(H);
    if (!e.empty()) return fail(e.find("single-GPU") != std::string::npos ? HMG_ERR_INVALID_ARG : HMG_ERR_CUDA, e);
    return check_launch();
}

}  // namespace

void hmg::vcycle_fine(const Hierarchy& H, const hmg_mg_params& p, const double* b, double* out, cudaStream_t s) {
    vcycle_level(H, H.fine_ref, p, b, out, s);
}

extern "C" {

const char* hmg_last_error(void) { return g_err.c_str(); }

hmg_status hmg_build_hierarchy(int fine_ref, int coarsest_ref, int nlayers, double thickness, double w2,
                               const double* lam_host, int device, hmg_hierarchy** out) {
    return build_impl(fine_ref, coarsest_ref, nlayers, thickness, w2, 0.0, lam_host, device, nullptr, out);
}

hmg_status hmg_build_hierarchy_ex(int fine_ref, int coarsest_ref, int nlayers, double thickness, double w2,
                                  double omega_n, const double* lam_host, int device, const hmg_dist* dist,
                                  hmg_hierarchy** out) {
    return build_impl(fine_ref, coarsest_ref, nlayers, thickness, w2, omega_n, lam_host, device, dist, out);
}

hmg_status hmg_build_hierarchy_dist(int fine_ref, int coarsest_ref, int nlayers, double thickness, double w2,
                                    const double* lam_host, int device, const hmg_dist* dist, hmg_hierarchy** out) {
    if (!dist) return fail(HMG_ERR_INVALID_ARG, "dist: null pointer");
    return build_impl(fine_ref, coarsest_ref, nlayers, thickness, w2, 0.0, lam_host, device, dist, out);
}

hmg_status hmg_nccl_unique_id(unsigned char* id_out) {
    if (!id_out) return fail(HMG_ERR_INVALID_ARG, "id_out: null pointer");
    std::string err;
    const Nccl* N = nccl(&err);
    if (!N) return fail(HMG_ERR_NCCL, err);
    NcclUniqueId id;
    const int r = N->GetUniqueId(&id);
    if (r != kNcclSuccess) return fail(HMG_ERR_NCCL, std::string("ncclGetUniqueId: ") + N->GetErrorString(r));
    std::memcpy(id_out, id.internal, sizeof(id.internal));
    return HMG_OK;
}

hmg_status hmg_partition_plan(int fine_ref, int ref, int rank, int nranks, int64_t* off, int64_t* n_own,
                              int64_t* n_halo, int* npeers, int64_t* send_total, int64_t* halo_gid,
                              int32_t* nbr_local, int32_t* peer_rank, int64_t* send_count, int64_t* recv_offset,
                              int64_t* recv_count, int32_t* send_local) {
    g_err.clear();
    if (fine_ref < 2 || fine_ref > kMaxRef) return fail(HMG_ERR_INVALID_ARG, "fine_ref: must be in [2, 10]");
    if (ref < 2 || ref > fine_ref) return fail(HMG_ERR_INVALID_ARG, "ref: must be in [2, fine_ref]");
    if (nranks < 1 || 320 % nranks != 0) return fail(HMG_ERR_INVALID_ARG, "nranks: must divide 320");
    if (rank < 0 || rank >= nranks) return fail(HMG_ERR_INVALID_ARG, "rank: must be in [0, nranks)");
    std::vector<HostLevel> host = build_icosahedral_levels(ref);
    LevelPlan P = plan_level(ref, host[ref].nbr, rank, nranks);
    if (off) *off = P.off;
    if (n_own) *n_own = P.n_own;
    if (n_halo) *n_halo = P.n_halo();
    if (npeers) *npeers = (int)P.peers.size();
    int64_t tot = 0;
    for (const PeerPlan& q : P.peers) tot += (int64_t)q.send_local.size();
    if (send_total) *send_total = tot;
    if (halo_gid) std::copy(P.halo_gid.begin(), P.halo_gid.end(), halo_gid);
    if (nbr_local) std::copy(P.nbr_local.begin(), P.nbr_local.end(), nbr_local);
    int64_t pos = 0;
    for (size_t i = 0; i < P.peers.size(); ++i) {
        const PeerPlan& q = P.peers[i];
        if (peer_rank) peer_rank[i] = q.rank;
        if (send_count) send_count[i] = (int64_t)q.send_local.size();
        if (recv_offset) recv_offset[i] = q.recv_offset;
        if (recv_count) recv_count[i] = q.recv_count;
        if (send_local) std::copy(q.send_local.begin(), q.send_local.end(), send_local + pos);
        pos += (int64_t)q.send_local.size();
    }
    return HMG_OK;
}

hmg_status hmg_free_hierarchy(hmg_hierarchy* h) {
    free_hierarchy(reinterpret_cast<Hierarchy*>(h));
    return HMG_OK;
}

hmg_status hmg_level_info(const hmg_hierarchy* h, int ref, int64_t* ncells, int64_t* ld) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    if (ref < 0 || ref > H.fine_ref) return fail(HMG_ERR_INVALID_ARG, "ref: outside [0, fine_ref]");
    if (ref >= H.coarsest_ref) {
        if (ncells) *ncells = H.lev[ref].n;
        if (ld) *ld = H.lev[ref].ld;
        return HMG_OK;
    }
    const int64_t n = 20 * (int64_t(1) << (2 * ref));
    if (ncells) *ncells = n;
    if (ld) *ld = round_up32(n);
    return HMG_OK;
}

hmg_status hmg_apply_helmholtz(const hmg_hierarchy* h, int ref, double* x, double* y, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, ref, "ref"));
    HMG_TRY(check_ptr(x, "x"));
    HMG_TRY(check_ptr(y, "y"));
    if (x == y) return fail(HMG_ERR_INVALID_ARG, "y: must not alias x");
    halo_exchange(H, H.lev[ref], x, S(stream));
    launch_apply(H, H.lev[ref], x, y, S(stream));
    return check_launch();
}

hmg_status hmg_line_smooth(const hmg_hierarchy* h, int ref, const double* b, double* u, int nsweeps, double omega,
                           int u_is_zero, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, ref, "ref"));
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(u, "u"));
    if (nsweeps < 0) return fail(HMG_ERR_INVALID_ARG, "nsweeps: must be >= 0");
    if (!std::isfinite(omega)) return fail(HMG_ERR_INVALID_ARG, "omega: must be finite");
    if (b == u) return fail(HMG_ERR_INVALID_ARG, "u: must not alias b");
    if (nsweeps == 0) {
        if (u_is_zero)
            HMG_CUDA(cudaMemset2DAsync(u, sizeof(double) * H.lev[ref].ld, 0, sizeof(double) * H.lev[ref].n, H.nz,
                                       S(stream)));
        return HMG_OK;
    }
    const DevLevel& L = H.lev[ref];
    if (u_is_zero) {
        run_sweeps(H, L, b, nullptr, nullptr, nsweeps, u, omega, S(stream));
    } else {
        // Jacobi semantics need the old iterate intact: sweep out of place, copy back
        const double* res = run_sweeps(H, L, b, u, nullptr, nsweeps, nullptr, omega, S(stream));
        HMG_CUDA(cudaMemcpy2DAsync(u, sizeof(double) * L.ld, res, sizeof(double) * L.ld, sizeof(double) * L.n, H.nz,
                                   cudaMemcpyDeviceToDevice, S(stream)));
    }
    HMG_TRY(check_launch());
    return check_bad(H, S(stream));
}

hmg_status hmg_restrict(const hmg_hierarchy* h, int fine_ref, const double* r_f, double* b_c, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, fine_ref, "fine_ref"));
    if (fine_ref == H.coarsest_ref) return fail(HMG_ERR_INVALID_ARG, "fine_ref: no coarser level in hierarchy");
    HMG_TRY(check_ptr(r_f, "r_f"));
    HMG_TRY(check_ptr(b_c, "b_c"));
    const DevLevel& L = H.lev[fine_ref];
    const DevLevel& C = H.lev[fine_ref - 1];
    launch_restrict(H, L, r_f, b_c, S(stream));
    if (L.dist.on && !C.dist.on) coarse_gather(H, C, b_c, S(stream));   // replicated coarse level: whole vector
    return check_launch();
}

hmg_status hmg_residual_restrict(const hmg_hierarchy* h, int fine_ref, const double* b, double* u, double* b_c,
                                 void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, fine_ref, "fine_ref"));
    if (fine_ref == H.coarsest_ref) return fail(HMG_ERR_INVALID_ARG, "fine_ref: no coarser level in hierarchy");
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(u, "u"));
    HMG_TRY(check_ptr(b_c, "b_c"));
    const DevLevel& L = H.lev[fine_ref];
    const DevLevel& C = H.lev[fine_ref - 1];
    halo_exchange(H, L, u, S(stream));             // neighbours' values of u (halo slots are library scratch)
    launch_resid_restrict(H, L, b, u, b_c, S(stream));
    if (L.dist.on && !C.dist.on) coarse_gather(H, C, b_c, S(stream));   // replicated coarse level: whole vector
    return check_launch();
}

hmg_status hmg_prolong_add(const hmg_hierarchy* h, int fine_ref, const double* u_c, double* u_f, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, fine_ref, "fine_ref"));
    if (fine_ref == H.coarsest_ref) return fail(HMG_ERR_INVALID_ARG, "fine_ref: no coarser level in hierarchy");
    HMG_TRY(check_ptr(u_c, "u_c"));
    HMG_TRY(check_ptr(u_f, "u_f"));
    launch_prolong_add(H, H.lev[fine_ref], u_f, u_c, u_f, S(stream));
    return check_launch();
}

hmg_status hmg_vcycle(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b, double* z, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_params(p));
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(z, "z"));
    if (b == z) return fail(HMG_ERR_INVALID_ARG, "z: must not alias b");
    vcycle_level(H, H.fine_ref, *p, b, z, S(stream));
    return check_launch();
}

hmg_status hmg_pcg_solve(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b, double* x, double rtol,
                         int maxit, int* iters, double* relres, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_params(p));
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(x, "x"));
    HMG_TRY(check_out(iters, "iters"));
    HMG_TRY(check_out(relres, "relres"));
    if (b == x) return fail(HMG_ERR_INVALID_ARG, "x: must not alias b");
    if (!(rtol >= 0)) return fail(HMG_ERR_INVALID_ARG, "rtol: must be >= 0");
    if (maxit < 0) return fail(HMG_ERR_INVALID_ARG, "maxit: must be >= 0");
    return pcg_impl(H, p, 0, 0.0, b, x, rtol, maxit, iters, relres, S(stream));
}

hmg_status hmg_pcg_solve_single_level(const hmg_hierarchy* h, int nsweeps, double omega, const double* b, double* x,
                                      double rtol, int maxit, int* iters, double* relres, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    if (nsweeps < 1) return fail(HMG_ERR_INVALID_ARG, "nsweeps: must be >= 1");
    if (!std::isfinite(omega)) return fail(HMG_ERR_INVALID_ARG, "omega: must be finite");
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(x, "x"));
    HMG_TRY(check_out(iters, "iters"));
    HMG_TRY(check_out(relres, "relres"));
    if (b == x) return fail(HMG_ERR_INVALID_ARG, "x: must not alias b");
    if (!(rtol >= 0)) return fail(HMG_ERR_INVALID_ARG, "rtol: must be >= 0");
    if (maxit < 0) return fail(HMG_ERR_INVALID_ARG, "maxit: must be >= 0");
    return pcg_impl(H, nullptr, nsweeps, omega, b, x, rtol, maxit, iters, relres, S(stream));
}

hmg_status hmg_pcg_solve_host(const hmg_hierarchy* h, const hmg_mg_params* p, const double* b_host, double* x_host,
                              double rtol, int maxit, int* iters, double* relres, void* stream) {
    HMG_TRY(check_h(h));
    Hierarchy& H = const_cast<Hierarchy&>(HH(h));
    HMG_TRY(check_out(b_host, "b_host"));
    HMG_TRY(check_out(x_host, "x_host"));
    const DevLevel& F = H.lev[H.fine_ref];
    const size_t vb = sizeof(double) * H.nz * F.ld;
    if (!H.hb) {
        HMG_CUDA(cudaMalloc(&H.hb, vb));
        HMG_CUDA(cudaMalloc(&H.hx, vb));
    }
    cudaStream_t s = S(stream);
    HMG_CUDA(cudaMemcpy2DAsync(H.hb, sizeof(double) * F.ld, b_host, sizeof(double) * F.n, sizeof(double) * F.n, H.nz,
                               cudaMemcpyHostToDevice, s));
    hmg_status st = hmg_pcg_solve(h, p, H.hb, H.hx, rtol, maxit, iters, relres, stream);
    if (st != HMG_OK && st != HMG_ERR_NOT_CONVERGED) return st;
    std::string msg = g_err;
    HMG_CUDA(cudaMemcpy2DAsync(x_host, sizeof(double) * F.n, H.hx, sizeof(double) * F.ld, sizeof(double) * F.n, H.nz,
                               cudaMemcpyDeviceToHost, s));
    HMG_CUDA(cudaStreamSynchronize(s));
    g_err = msg;
    return st;
}

hmg_status hmg_pcg_solve_host_batch(const hmg_hierarchy* h, const hmg_mg_params* p, int nrhs,
                                    const double* const* b_host, double* const* x_host, double rtol, int maxit,
                                    int* iters, double* relres, void* stream) {
    HMG_TRY(check_h(h));
    Hierarchy& H = const_cast<Hierarchy&>(HH(h));
    if (nrhs < 0) return fail(HMG_ERR_INVALID_ARG, "nrhs: must be >= 0");
    if (nrhs == 0) return HMG_OK;
    HMG_TRY(check_out(b_host, "b_host"));
    HMG_TRY(check_out(x_host, "x_host"));
    HMG_TRY(check_out(iters, "iters"));
    HMG_TRY(check_out(relres, "relres"));
    for (int i = 0; i < nrhs; ++i) {
        if (!b_host[i]) return fail(HMG_ERR_INVALID_ARG, "b_host[" + std::to_string(i) + "]: null pointer");
        if (!x_host[i]) return fail(HMG_ERR_INVALID_ARG, "x_host[" + std::to_string(i) + "]: null pointer");
    }
    HMG_CUDA(cudaSetDevice(H.device));
    const DevLevel& F = H.lev[H.fine_ref];
    const size_t vb = sizeof(double) * H.nz * F.ld;
    if (!H.hb) {
        HMG_CUDA(cudaMalloc(&H.hb, vb));
        HMG_CUDA(cudaMalloc(&H.hx, vb));
    }
    if (!H.hb1) {
        HMG_CUDA(cudaMalloc(&H.hb1, vb));
        HMG_CUDA(cudaMalloc(&H.hx1, vb));
        HMG_CUDA(cudaStreamCreateWithFlags(&H.cs_in, cudaStreamNonBlocking));
        HMG_CUDA(cudaStreamCreateWithFlags(&H.cs_out, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            HMG_CUDA(cudaEventCreateWithFlags(&H.ev_in[i], cudaEventDisableTiming));
            HMG_CUDA(cudaEventCreateWithFlags(&H.ev_solved[i], cudaEventDisableTiming));
            HMG_CUDA(cudaEventCreateWithFlags(&H.ev_out[i], cudaEventDisableTiming));
        }
    }
    double* const dB[2] = {H.hb, H.hb1};
    double* const dX[2] = {H.hx, H.hx1};
    cudaStream_t s = S(stream);
    const size_t hp = sizeof(double) * F.n, dp = sizeof(double) * F.ld;
    // Solve i runs on `stream` from dB[i % 2] into dX[i % 2]; the copy of b_{i+1}
    // in (cs_in) and of x_{i-1} out (cs_out) overlap it.  Buffer reuse is
    // ordered by events: b_{i+1} lands in the buffer solve i-1 read, after that
    // solve; solve i writes the x buffer whose copy-out (x_{i-2}) it waits for.
    HMG_CUDA(cudaEventRecord(H.ev_solved[1], s));   // the calling stream's prior work (buffers may be in use)
    HMG_CUDA(cudaStreamWaitEvent(H.cs_in, H.ev_solved[1], 0));
    HMG_CUDA(cudaMemcpy2DAsync(dB[0], dp, b_host[0], hp, hp, H.nz, cudaMemcpyHostToDevice, H.cs_in));
    HMG_CUDA(cudaEventRecord(H.ev_in[0], H.cs_in));
    hmg_status worst = HMG_OK;
    std::string msg;
    for (int i = 0; i < nrhs; ++i) {
        const int c = i & 1, o = c ^ 1;
        if (i + 1 < nrhs) {
            if (i >= 1) HMG_CUDA(cudaStreamWaitEvent(H.cs_in, H.ev_solved[o], 0));
            HMG_CUDA(cudaMemcpy2DAsync(dB[o], dp, b_host[i + 1], hp, hp, H.nz, cudaMemcpyHostToDevice, H.cs_in));
            HMG_CUDA(cudaEventRecord(H.ev_in[o], H.cs_in));
        }
        HMG_CUDA(cudaStreamWaitEvent(s, H.ev_in[c], 0));
        if (i >= 2) HMG_CUDA(cudaStreamWaitEvent(s, H.ev_out[c], 0));
        int it = 0;
        double rr = 0.0;
        const hmg_status st = hmg_pcg_solve(h, p, dB[c], dX[c], rtol, maxit, &it, &rr, stream);
        iters[i] = it;
        relres[i] = rr;
        if (st != HMG_OK && st != HMG_ERR_NOT_CONVERGED) {
            cudaStreamSynchronize(H.cs_in);
            cudaStreamSynchronize(H.cs_out);
            return st;
        }
        if (st != HMG_OK && worst == HMG_OK) {
            worst = st;
            msg = g_err;
        }
        HMG_CUDA(cudaEventRecord(H.ev_solved[c], s));
        HMG_CUDA(cudaStreamWaitEvent(H.cs_out, H.ev_solved[c], 0));
        HMG_CUDA(cudaMemcpy2DAsync(x_host[i], hp, dX[c], dp, hp, H.nz, cudaMemcpyDeviceToHost, H.cs_out));
        HMG_CUDA(cudaEventRecord(H.ev_out[c], H.cs_out));
    }
    HMG_CUDA(cudaStreamSynchronize(H.cs_out));
    HMG_CUDA(cudaStreamSynchronize(H.cs_in));
    // the caller's stream is ordered after the last copy-out
    HMG_CUDA(cudaStreamWaitEvent(s, H.ev_out[(nrhs - 1) & 1], 0));
    g_err = msg;
    return worst;
}

hmg_status hmg_pcg_history(const hmg_hierarchy* h, double* hist, int cap, int* n) {
    HMG_TRY(check_h(h));
    HMG_TRY(check_out(n, "n"));
    if (cap < 0) return fail(HMG_ERR_INVALID_ARG, "cap: must be >= 0");
    const std::vector<double>& v = HH(h).res_hist;
    *n = (int)v.size();
    if (hist)
        for (int i = 0; i < cap && i < (int)v.size(); ++i) hist[i] = v[i];
    return HMG_OK;
}

hmg_status hmg_export_level(const hmg_hierarchy* h, int ref, int32_t* nbr, double* geom, double* bands, double* lam) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, ref, "ref"));
    const DevLevel& L = H.lev[ref];
    HMG_CUDA(cudaSetDevice(H.device));
    HMG_CUDA(cudaDeviceSynchronize());
    if (nbr) {
        std::vector<int32_t> t(3 * L.ld);
        HMG_CUDA(cudaMemcpy(t.data(), L.nbr, sizeof(int32_t) * 3 * L.ld, cudaMemcpyDeviceToHost));
        for (int64_t c = 0; c < L.n; ++c)
            for (int j = 0; j < 3; ++j) nbr[c * 3 + j] = t[j * L.ld + c];
    }
    if (geom)
        HMG_CUDA(cudaMemcpy2D(geom, sizeof(double) * L.n, L.geom, sizeof(double) * L.ld, sizeof(double) * L.n, 7,
                              cudaMemcpyDeviceToHost));
    if (bands)
        HMG_CUDA(cudaMemcpy2D(bands, sizeof(double) * L.n, L.bands, sizeof(double) * L.ld, sizeof(double) * L.n,
                              5 * H.nz, cudaMemcpyDeviceToHost));
    if (lam)
        HMG_CUDA(cudaMemcpy2D(lam, sizeof(double) * L.n, L.lam, sizeof(double) * L.ld, sizeof(double) * L.n, H.nz,
                              cudaMemcpyDeviceToHost));
    return HMG_OK;
}

int64_t hmg_launch_count(const hmg_hierarchy* h) { return h ? HH(h).launches : -1; }

hmg_status hmg_edge_store(const hmg_hierarchy* h, int ref, int* kernels) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_level(H, ref, "ref"));
    HMG_TRY(check_out(kernels, "kernels"));
    const DevLevel& L = H.lev[ref];
    *kernels = 0;
    if (L.edge.H) {
        if (sweep_edge_store(H, L)) *kernels |= 1;
        *kernels |= 2;
        if (resid_st_supported(H, L)) *kernels |= 4;
    }
    return HMG_OK;
}

hmg_status hmg_profile_begin(hmg_hierarchy* h) {
    HMG_TRY(check_h(h));
    Profiler& P = HH(h).prof;
    P.on = true;
    P.used = 0;
    P.cls.clear();
    P.ref.clear();
    return HMG_OK;
}

hmg_status hmg_profile_select(hmg_hierarchy* h, int kernel_class, int ref) {
    HMG_TRY(check_h(h));
    if (kernel_class >= kKNumClasses) return fail(HMG_ERR_INVALID_ARG, "kernel_class: unknown");
    Profiler& P = HH(h).prof;
    P.only_cls = kernel_class < 0 ? -1 : kernel_class;
    P.only_ref = ref < 0 ? -1 : ref;
    return HMG_OK;
}

hmg_status hmg_profile_end(hmg_hierarchy* h) {
    HMG_TRY(check_h(h));
    HH(h).prof.on = false;
    return HMG_OK;
}

hmg_status hmg_profile_query(const hmg_hierarchy* h, int kernel_class, int ref, int64_t* count, double* total_ms) {
    HMG_TRY(check_h(h));
    HMG_TRY(check_ptr(count, "count"));
    HMG_TRY(check_ptr(total_ms, "total_ms"));
    if (kernel_class < 0 || kernel_class >= kKNumClasses) return fail(HMG_ERR_INVALID_ARG, "kernel_class: unknown");
    const Profiler& P = HH(h).prof;
    *count = 0;
    *total_ms = 0.0;
    for (size_t i = 0; i < P.cls.size(); ++i) {
        if (P.cls[i] != kernel_class || (ref >= 0 && P.ref[i] != ref)) continue;
        float ms = 0.f;
        HMG_CUDA(cudaEventSynchronize(P.pool[2 * i + 1]));
        HMG_CUDA(cudaEventElapsedTime(&ms, P.pool[2 * i], P.pool[2 * i + 1]));
        *count += 1;
        *total_ms += ms;
    }
    return HMG_OK;
}

hmg_status hmg_selftest_div(const double* a, const double* b, double* fast, double* ref, int64_t n, void* stream) {
    HMG_TRY(check_ptr(a, "a"));
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(fast, "fast"));
    HMG_TRY(check_ptr(ref, "ref"));
    if (n < 0) return fail(HMG_ERR_INVALID_ARG, "n: must be >= 0");
    if (n == 0) return HMG_OK;
    launch_selftest_div(n, a, b, fast, ref, S(stream));
    return check_launch();
}

hmg_status hmg_mixed_layout(const hmg_hierarchy* h, int64_t* ne, int64_t* ldh, int64_t* off_z, int64_t* off_p,
                            int64_t* ntot) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(ensure_mixed(H));
    const MixedSystem& M = *H.mix;
    if (ne) *ne = M.ne;
    if (ldh) *ldh = M.ldh;
    if (off_z) *off_z = M.off_z;
    if (off_p) *off_p = M.off_p;
    if (ntot) *ntot = M.ntot;
    return HMG_OK;
}

hmg_status hmg_mixed_export_edges(const hmg_hierarchy* h, int32_t* ec, int32_t* ce) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(ensure_mixed(H));
    const MixedSystem& M = *H.mix;
    const DevLevel& L = H.lev[H.fine_ref];
    if (ec) {
        std::vector<int32_t> a(M.ne), b(M.ne);
        HMG_CUDA(cudaMemcpy(a.data(), M.eca, sizeof(int32_t) * M.ne, cudaMemcpyDeviceToHost));
        HMG_CUDA(cudaMemcpy(b.data(), M.ecb, sizeof(int32_t) * M.ne, cudaMemcpyDeviceToHost));
        for (int64_t e = 0; e < M.ne; ++e) {
            ec[2 * e] = a[e];
            ec[2 * e + 1] = b[e];
        }
    }
    if (ce) {
        std::vector<int32_t> t(3 * L.ld);
        HMG_CUDA(cudaMemcpy(t.data(), M.ce, sizeof(int32_t) * 3 * L.ld, cudaMemcpyDeviceToHost));
        for (int64_t c = 0; c < L.n; ++c)
            for (int j = 0; j < 3; ++j) ce[3 * c + j] = t[j * L.ld + c];
    }
    return HMG_OK;
}

hmg_status hmg_mixed_apply(const hmg_hierarchy* h, const double* x, double* y, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    HMG_TRY(check_ptr(x, "x"));
    HMG_TRY(check_ptr(y, "y"));
    if (x == y) return fail(HMG_ERR_INVALID_ARG, "y: must not alias x");
    HMG_TRY(ensure_mixed(H));
    launch_mixed_apply(H, x, y, S(stream));
    return check_launch();
}

hmg_status hmg_mixed_precond(const hmg_hierarchy* h, const hmg_mg_params* p, const double* f, double* x,
                             void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    if (p) HMG_TRY(check_params(p));
    HMG_TRY(check_ptr(f, "f"));
    HMG_TRY(check_ptr(x, "x"));
    if (f == x) return fail(HMG_ERR_INVALID_ARG, "x: must not alias f");
    HMG_TRY(ensure_mixed(H));
    mixed_precond(H, p, f, x, S(stream));
    return check_launch();
}

hmg_status hmg_mixed_gmres(const hmg_hierarchy* h, const hmg_mg_params* p, const double* F, double* X, double rtol,
                           int restart, int maxit, int gs_passes, int* iters, double* relres, void* stream) {
    HMG_TRY(check_h(h));
    const Hierarchy& H = HH(h);
    if (p) HMG_TRY(check_params(p));
    HMG_TRY(check_ptr(F, "F"));
    HMG_TRY(check_ptr(X, "X"));
    HMG_TRY(check_out(iters, "iters"));
    HMG_TRY(check_out(relres, "relres"));
    if (F == X) return fail(HMG_ERR_INVALID_ARG, "X: must not alias F");
    if (!(rtol >= 0)) return fail(HMG_ERR_INVALID_ARG, "rtol: must be >= 0");
    if (restart < 1 || restart > mixed_lin_max() - 1)
        return fail(HMG_ERR_INVALID_ARG, "restart: must be in [1, " + std::to_string(mixed_lin_max() - 1) + "]");
    if (maxit < 0) return fail(HMG_ERR_INVALID_ARG, "maxit: must be >= 0");
    if (gs_passes < 1 || gs_passes > 2) return fail(HMG_ERR_INVALID_ARG, "gs_passes: must be 1 (CGS) or 2 (CGS2)");
    HMG_TRY(ensure_mixed(H));
    return mixed_gmres_impl(H, p, F, X, rtol, restart, maxit, gs_passes, iters, relres, S(stream));
}

// ---------------------------------------------------------------------------
// NEXT-3 core: batched per-column banded algebra (band.cu; include/hmg.h)
// ---------------------------------------------------------------------------
static hmg_status check_band(int64_t ncol, int m, int kl, int ku, int64_t ld) {
    if (ncol < 0) return fail(HMG_ERR_INVALID_ARG, "ncol: must be >= 0");
    if (m < 1 || m > 4096) return fail(HMG_ERR_INVALID_ARG, "m: must be in [1, 4096]");
    if (!band_shape_supported(kl, ku))
        return fail(HMG_ERR_INVALID_ARG, "kl, ku: (" + std::to_string(kl) + ", " + std::to_string(ku) +
                                             ") not compiled; supported: (13,13) (1,1) (2,2) (3,5) (5,2) (0,0)");
    if (ld < ncol || ld % 32 != 0) return fail(HMG_ERR_INVALID_ARG, "ld: must be >= ncol and a multiple of 32");
    if ((int64_t)m * (2 * kl + ku + 1) > (int64_t)1 << 31) return fail(HMG_ERR_INVALID_ARG, "m: band too large");
    return HMG_OK;
}

hmg_status hmg_band_factor(int64_t ncol, int m, int kl, int ku, double* ab, int64_t ld, int32_t* ipiv,
                           int64_t* singular, void* stream) {
    g_err.clear();
    HMG_TRY(check_band(ncol, m, kl, ku, ld));
    HMG_TRY(check_ptr(ab, "ab"));
    HMG_TRY(check_ptr(ipiv, "ipiv"));
    if (singular) *singular = -1;
    if (ncol == 0) return HMG_OK;
    unsigned long long* bad = nullptr;
    HMG_CUDA(cudaMalloc(&bad, sizeof(*bad)));
    const unsigned long long none = ~0ull;
    HMG_CUDA(cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, S(stream)));
    launch_band_factor(ncol, m, kl, ku, ab, ld, ipiv, bad, S(stream));
    hmg_status st = check_launch();
    unsigned long long got = none;
    if (st == HMG_OK) {
        cudaError_t e = cudaMemcpyAsync(&got, bad, sizeof(got), cudaMemcpyDeviceToHost, S(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
        if (e != cudaSuccess) st = fail(HMG_ERR_CUDA, std::string("hmg_band_factor: ") + cudaGetErrorString(e));
    }
    cudaFree(bad);
    if (st != HMG_OK) return st;
    if (got != none) {
        const int64_t col = (int64_t)(got >> 24), row = (int64_t)(got & ((1ull << 24) - 1));
        if (singular) *singular = col;
        return fail(HMG_ERR_SINGULAR_COLUMN, "singular column: column " + std::to_string(col) + " (U(" +
                                                 std::to_string(row) + ", " + std::to_string(row) + ") = 0)");
    }
    return HMG_OK;
}

hmg_status hmg_band_solve(int64_t ncol, int m, int kl, int ku, const double* ab, int64_t ld, const int32_t* ipiv,
                          const double* b, double* x, void* stream) {
    g_err.clear();
    HMG_TRY(check_band(ncol, m, kl, ku, ld));
    HMG_TRY(check_ptr(ab, "ab"));
    HMG_TRY(check_ptr(ipiv, "ipiv"));
    HMG_TRY(check_ptr(b, "b"));
    HMG_TRY(check_ptr(x, "x"));
    if (b == x) return fail(HMG_ERR_INVALID_ARG, "x: must not alias b");
    if (ncol == 0) return HMG_OK;
    try {
        launch_band_solve(ncol, m, kl, ku, ab, ld, ipiv, b, x, S(stream));
    } catch (const std::exception& e) {
        return fail(HMG_ERR_CUDA, std::string("hmg_band_solve: ") + e.what());
    }
    return check_launch();
}

hmg_status hmg_band_apply(int64_t ncol, int m, int kl, int ku, const double* ar, int64_t ld, const double* x, double* y,
                          void* stream) {
    g_err.clear();
    HMG_TRY(check_band(ncol, m, kl, ku, ld));
    HMG_TRY(check_ptr(ar, "ar"));
    HMG_TRY(check_ptr(x, "x"));
    HMG_TRY(check_ptr(y, "y"));
    if (x == y) return fail(HMG_ERR_INVALID_ARG, "y: must not alias x");
    if (ncol == 0) return HMG_OK;
    try {
        launch_band_apply(ncol, m, kl, ku, ar, ld, x, y, S(stream));
    } catch (const std::exception& e) {
        return fail(HMG_ERR_CUDA, std::string("hmg_band_apply: ") + e.what());
    }
    return check_launch();
}

hmg_status hmg_p_restrict(int64_t ncol, int nz, const double* r1, int64_t ld, double* b0, void* stream) {
    g_err.clear();
    if (ncol < 0) return fail(HMG_ERR_INVALID_ARG, "ncol: must be >= 0");
    if (nz < 1 || nz > 65535) return fail(HMG_ERR_INVALID_ARG, "nz: must be in [1, 65535]");
    if (ld < ncol) return fail(HMG_ERR_INVALID_ARG, "ld: must be >= ncol");
    HMG_TRY(check_ptr(r1, "r1"));
    HMG_TRY(check_ptr(b0, "b0"));
    if (ncol == 0) return HMG_OK;
    launch_p_restrict(ncol, nz, r1, ld, b0, S(stream));
    return check_launch();
}

hmg_status hmg_p_prolong_add(int64_t ncol, int nz, const double* u0, int64_t ld, double* u1, void* stream) {
    g_err.clear();
    if (ncol < 0) return fail(HMG_ERR_INVALID_ARG, "ncol: must be >= 0");
    if (nz < 1 || nz > 65535) return fail(HMG_ERR_INVALID_ARG, "nz: must be in [1, 65535]");
    if (ld < ncol) return fail(HMG_ERR_INVALID_ARG, "ld: must be >= ncol");
    HMG_TRY(check_ptr(u0, "u0"));
    HMG_TRY(check_ptr(u1, "u1"));
    if (ncol == 0) return HMG_OK;
    launch_p_prolong_add(ncol, nz, u0, ld, u1, S(stream));
    return check_launch();
}

}  // extern "C"
