// Coarse tail of the V-cycle in ONE kernel launch (SURVEY 7 "coarse levels
// are latency-bound", B8): every level ref <= tail_ref of Alg. 1,
// i.e. presmoothing, residual restriction, the coarsest level's n_coarse
// sweeps (BASELINE.json: 20) and the postsmoothing with the fused
// prolongation, runs inside a single CTA with __syncthreads between the
// dependent steps instead of ~40 kernel launches.  The paper saw the same
// coarse-level inefficiency on CPUs.
//
// Arithmetic is identical to the per-level kernels (readings R5-R9, same
// operation order, no contraction).  The Thomas pivots den_k, their refined
// reciprocals y_k and the multipliers g_k depend only on the matrix, so they
// are computed once at setup (k_factor, same formulas as the sweeps) and read
// here: the per-layer dependency chain of a sweep shrinks to the z recurrence.
// The column state z_k lives in shared memory.  Everything the tail touches
// (<= 1 MB at tail_ref 2) stays in L1/L2.
#include <cfloat>

#include <cooperative_groups.h>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {
namespace {

__device__ __forceinline__ bool pivot_ok(double den) { return den > 0.0 && den <= DBL_MAX; }

// ---------------------------------------------------------------------------
// Setup: Thomas factors per column (reading R6 order).
// ---------------------------------------------------------------------------
__global__ void k_factor(LevelView L, double* __restrict__ den_out, double* __restrict__ y_out,
                         double* __restrict__ g_out, int ref, unsigned long long* __restrict__ bad) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= L.n) return;
    const int64_t ld = L.ld;
    const int nz = L.nz;
    double den = L.D[c];
    bool ok = pivot_ok(den);
    for (int k = 0; k < nz; ++k) {
        const int64_t i = k * ld + c;
        const double y = div_recip(den);
        den_out[i] = den;
        y_out[i] = y;
        if (k < nz - 1) {
            const double Uk = L.U[i];
            bool slow = false;
            double g = div_fast(Uk, den, y, slow);
            if (slow) g = Uk / den;
            g_out[i] = g;
            den = L.D[i + ld] - Uk * g;
            ok = ok && pivot_ok(den);
        } else {
            g_out[i] = 0.0;
        }
    }
    if (!ok) atomicMin(bad, ((unsigned long long)ref << 40) | (unsigned long long)c);
}

// Setup, levels without stored factors: the Thomas pivots of every column
// (the sweeps' own operations: den_k, div_recip, g_k by the fast path) are
// checked once -- they depend on the matrix only -- and it is recorded whether
// any multiplier g_k = U_k / den_k left the fast path's exact range.  If none
// did, the sweeps on this level skip both per-layer tests (DevLevel::g_safe).
__global__ void k_pivot_check(LevelView L, int ref, unsigned long long* __restrict__ bad,
                              unsigned int* __restrict__ gslow) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= L.n) return;
    const int64_t ld = L.ld;
    const int nz = L.nz;
    double den = L.D[c];
    bool ok = true, slow = false;
    for (int k = 0; k < nz; ++k) {
        ok = ok && pivot_ok(den);
        if (k == nz - 1) break;
        const int64_t i = k * ld + c;
        const double Uk = L.U[i];
        const double y = div_recip(den);
        bool sl = false;
        double g = div_fast(Uk, den, y, sl);
        if (sl) g = Uk / den;
        slow = slow || sl;
        den = L.D[i + ld] - Uk * g;
    }
    if (!ok) atomicMin(bad, ((unsigned long long)ref << 40) | (unsigned long long)c);
    if (slow) atomicOr(gslow, 1u);
}

// u value of cell `cell` at row offset `row` (with the fused prolongation)
__device__ __forceinline__ double uval(const double* __restrict__ u, const double* __restrict__ uc, int64_t row,
                                       int64_t rowc, int64_t cell) {
    double v = u[row + cell];
    if (uc) v = v + uc[rowc + (cell >> 2)];
    return v;
}

// One damped line-Jacobi sweep of column c: uout = uin(+P uc) + omega T^{-1}(b - H^(uin + P uc));
// uin == nullptr: zero guess.  The z_k of the column live in shared memory
// zs[k * stride]; loops are unrolled so that the (independent) loads of
// several layers are in flight together -- the tail is latency-bound.
__device__ void sweep_col(const TailLevel& T, int nz, const double* __restrict__ b, const double* __restrict__ uin,
                          const double* __restrict__ uc, double* __restrict__ uout, double omega, int64_t c,
                          double* __restrict__ zs, int stride) {
    const LevelView& L = T.V;
    const int64_t ld = L.ld, ldc = T.ldc;
    const double* __restrict__ den_p = T.den;
    const double* __restrict__ y_p = T.y;
    const double* __restrict__ g_p = T.g;
    double um = 0.0, uk = 0.0, Um = 0.0, zprev = 0.0;
    int32_t n0 = 0, n1 = 0, n2 = 0;
    if (uin) {
        n0 = L.nbr[c];
        n1 = L.nbr[ld + c];
        n2 = L.nbr[2 * ld + c];
        uk = uval(uin, uc, 0, 0, c);
    }
#pragma unroll 8
    for (int k = 0; k < nz; ++k) {
        const int64_t row = k * ld, i = row + c, rowc = k * ldc;
        const double Dk = L.D[i];
        const double Uk = L.U[i];
        double r, up = 0.0;
        if (!uin) {
            r = b[i];
        } else {
            if (k < nz - 1) up = uval(uin, uc, row + ld, rowc + ldc, c);
            double acc = Dk * uk;
            if (k > 0) acc = acc + Um * um;
            if (k < nz - 1) acc = acc + Uk * up;
            acc = acc + L.H0[i] * uval(uin, uc, row, rowc, n0);
            acc = acc + L.H1[i] * uval(uin, uc, row, rowc, n1);
            acc = acc + L.H2[i] * uval(uin, uc, row, rowc, n2);
            r = b[i] - acc;
        }
        const double den = den_p[i];
        const double num = (k == 0) ? r : r - Um * zprev;
        bool slow = false;
        double z = div_fast_z(num, den, y_p[i], slow);
        if (slow) z = num / den;
        zs[k * stride] = z;
        zprev = z;
        um = uk;
        uk = up;
        Um = Uk;
    }
    double dl = 0.0;
#pragma unroll 8
    for (int k = nz - 1; k >= 0; --k) {
        const int64_t i = k * ld + c;
        const double zk = zs[k * stride];
        dl = (k == nz - 1) ? zk : zk - g_p[i] * dl;
        uout[i] = uin ? uval(uin, uc, k * ld, k * ldc, c) + omega * dl : omega * dl;
    }
}

// Coarse cell p: b_c[k][p] = ((r0 + r1) + r2) + r3 over its 4 children, r = b - H^ u
// (u == nullptr: r = b, plain restriction).
__device__ void resid_restrict_cell(const TailLevel& F, int nz, const double* b, const double* u, double* bc,
                                    int64_t ldc, int64_t p) {
    const LevelView& L = F.V;
    const int64_t ld = L.ld;
    for (int k = 0; k < nz; ++k) {
        double r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t c = 4 * p + q, i = k * ld + c;
            if (!u) {
                r[q] = b[i];
                continue;
            }
            double acc = L.D[i] * u[i];
            if (k > 0) acc = acc + L.U[i - ld] * u[i - ld];
            if (k < nz - 1) acc = acc + L.U[i] * u[i + ld];
            acc = acc + L.H0[i] * u[k * ld + L.nbr[c]];
            acc = acc + L.H1[i] * u[k * ld + L.nbr[ld + c]];
            acc = acc + L.H2[i] * u[k * ld + L.nbr[2 * ld + c]];
            r[q] = b[i] - acc;
        }
        bc[k * ldc + p] = ((r[0] + r[1]) + r[2]) + r[3];
    }
}

// Block-wide or grid-wide barrier between the dependent steps of the tail.
template <bool GRID>
__device__ __forceinline__ void tail_sync() {
    if (GRID)
        cooperative_groups::this_grid().sync();
    else
        __syncthreads();
}

// GRID = false: one CTA runs every step (__syncthreads between them).
// GRID = true: a cooperative launch of several CTAs; columns are dealt out
// over all threads of the grid and the dependent steps are separated by grid
// barriers (~1 us each on B200, against ~3 us per dependent kernel launch);
// the coarsest level's sweeps run in CTA 0 alone when its columns fit there.
template <bool GRID>
__global__ void __launch_bounds__(GRID ? 128 : 512, 1) k_coarse_tail(TailParams P) {
    extern __shared__ double zsm[];          // [nz][blockDim]: Thomas z of each thread's current column
    const int nz = P.nz;
    const int zstride = blockDim.x;
    const int64_t t = GRID ? (int64_t)blockIdx.x * blockDim.x + threadIdx.x : threadIdx.x;
    const int64_t T = GRID ? (int64_t)gridDim.x * blockDim.x : blockDim.x;
    double* zs = zsm + threadIdx.x;
    const double w = P.omega;
    const double* cur[kMaxRef + 1];          // presmoothed iterate per level
    // ---- down leg: presmooth, restrict the residual ----
    for (int l = P.top; l > P.coarsest; --l) {
        const TailLevel& L = P.lev[l];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        const double* c_in = nullptr;
        double* dst = L.wa;
        for (int s = 0; s < P.nu_pre; ++s) {
            dst = (c_in == L.wa) ? L.wb : L.wa;
            for (int64_t c = t; c < L.V.n; c += T) sweep_col(L, nz, bl, c_in, nullptr, dst, w, c, zs, zstride);
            tail_sync<GRID>();
            c_in = dst;
        }
        cur[l] = c_in;
        const TailLevel& C = P.lev[l - 1];
        for (int64_t p = t; p < C.V.n; p += T) resid_restrict_cell(L, nz, bl, c_in, C.b, C.V.ld, p);
        tail_sync<GRID>();
    }
    // ---- coarsest level: n_coarse sweeps from zero, result in its u ----
    {
        const int l = P.coarsest;
        const TailLevel& L = P.lev[l];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        double* out = (l == P.top) ? P.out_top : L.u;
        const double* c_in = nullptr;
        const bool one_cta = GRID && L.V.n <= (int64_t)blockDim.x;   // CTA 0 alone, block barriers
        if (!one_cta || blockIdx.x == 0) {
            const int64_t tt = one_cta ? threadIdx.x : t, TT = one_cta ? blockDim.x : T;
            for (int s = 0; s < P.n_coarse; ++s) {
                double* dst = (s == P.n_coarse - 1) ? out : ((c_in == L.wa) ? L.wb : L.wa);
                for (int64_t c = tt; c < L.V.n; c += TT) sweep_col(L, nz, bl, c_in, nullptr, dst, w, c, zs, zstride);
                if (one_cta)
                    __syncthreads();
                else
                    tail_sync<GRID>();
                c_in = dst;
            }
        }
        if (one_cta) tail_sync<GRID>();
    }
    // ---- up leg: prolongation fused into the first postsmoothing sweep ----
    for (int l = P.coarsest + 1; l <= P.top; ++l) {
        const TailLevel& L = P.lev[l];
        const TailLevel& C = P.lev[l - 1];
        const double* bl = (l == P.top) ? P.b_top : L.b;
        double* out = (l == P.top) ? P.out_top : L.u;
        const double* c_in = cur[l];
        if (!c_in) {                          // nu_pre = 0: the presmoothed iterate is zero
            for (int64_t i = t; i < (int64_t)nz * L.V.ld; i += T) L.wa[i] = 0.0;
            tail_sync<GRID>();
            c_in = L.wa;
        }
        if (P.nu_post == 0) {
            for (int64_t c = t; c < L.V.n; c += T)
                for (int k = 0; k < nz; ++k)
                    out[k * L.V.ld + c] = c_in[k * L.V.ld + c] + C.u[k * C.V.ld + (c >> 2)];
            tail_sync<GRID>();
            continue;
        }
        for (int s = 0; s < P.nu_post; ++s) {
            double* dst = (s == P.nu_post - 1) ? out : ((c_in == L.wa) ? L.wb : L.wa);
            TailLevel Lc = L;
            Lc.ldc = C.V.ld;
            for (int64_t c = t; c < L.V.n; c += T)
                sweep_col(Lc, nz, bl, c_in, s == 0 ? C.u : nullptr, dst, w, c, zs, zstride);
            tail_sync<GRID>();
            c_in = dst;
        }
    }
}

}  // namespace

void launch_pivot_check(const Hierarchy& H, const DevLevel& L, unsigned int* gslow, cudaStream_t s) {
    k_pivot_check<<<(unsigned)((L.n + 127) / 128), 128, 0, s>>>(L.view(H.nz), L.ref, &H.scal->bad, gslow);
    ++H.launches;
}

void launch_factor(const Hierarchy& H, const DevLevel& L, cudaStream_t s) {
    k_factor<<<(unsigned)((L.n + 127) / 128), 128, 0, s>>>(L.view(H.nz), L.fden, L.fy, L.fg, L.ref, &H.scal->bad);
    ++H.launches;
}

void launch_coarse_tail(const Hierarchy& H, const hmg_mg_params& p, const double* b_top, double* out_top,
                        cudaStream_t s) {
    TailParams P;
    P.nz = H.nz;
    P.top = H.tail_ref;
    P.coarsest = H.coarsest_ref;
    P.nu_pre = p.nu_pre;
    P.nu_post = p.nu_post;
    P.n_coarse = p.n_coarse;
    P.omega = p.omega;
    P.b_top = b_top;
    P.out_top = out_top;
    for (int r = H.coarsest_ref; r <= H.tail_ref; ++r) {
        const DevLevel& L = H.lev[r];
        TailLevel& T = P.lev[r];
        T.V = L.view(H.nz);
        T.wa = L.wa;
        T.wb = L.wb;
        T.b = L.b;
        T.u = L.u;
        T.den = L.fden;
        T.y = L.fy;
        T.g = L.fg;
        T.ldc = 0;
    }
    const int64_t n = H.lev[H.tail_ref].n;
    ProfScope ps(H, kKCoarseTail, H.tail_ref, s);
    if (H.tail_grid) {
        // cooperative launch: blocks of tail_threads columns, as many as the
        // top level needs, all co-resident (cooperative launch guarantees it)
        const int threads = H.tail_threads;
        const size_t smem = sizeof(double) * H.nz * threads;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_coarse_tail<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr = true;
        }
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_tail<true>, threads, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
        int64_t grid = (n + threads - 1) / threads;
        const int64_t cap = (int64_t)(per_sm < 1 ? 1 : per_sm) * sms;
        if (grid > cap) grid = cap;
        void* args[] = {&P};
        cudaLaunchCooperativeKernel((const void*)k_coarse_tail<true>, dim3((unsigned)grid), dim3(threads), args, smem,
                                    s);
        ++H.launches;
        return;
    }
    int threads = (int)((n + 31) / 32 * 32);
    if (threads > 512) threads = 512;
    const int cap = (int)((200 * 1024) / (sizeof(double) * H.nz)) / 32 * 32;   // z slots in shared memory
    if (threads > cap) threads = cap < 32 ? 32 : cap;
    const size_t smem = sizeof(double) * H.nz * threads;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_coarse_tail<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    k_coarse_tail<false><<<1, threads, smem, s>>>(P);
    ++H.launches;
}

}  // namespace hmg

// ===========================================================================
// Coarsest-level solve: n_coarse sweeps from zero (Alg. 1 M3 at the bottom of
// the recursion) for a level small enough to live in one CTA's
// shared memory (ref 0: 20 columns).  Operands (bands, precomputed pivots,
// the right-hand side) are loaded once; the sweeps then run entirely from
// shared memory with __syncthreads between them.  Same arithmetic and
// operation order as every other sweep.
// ===========================================================================
namespace hmg {
namespace {

constexpr int kCoarsestArrays = 9;   // D, U, H0, H1, H2, b, den, y, g
#ifdef HMG_TIMING
__device__ long long g_cs_timing[64];
#define CSTAMP(i) do { if (threadIdx.x == 0) g_cs_timing[i] = clock64(); } while (0)
#else
#define CSTAMP(i) do {} while (0)
#endif

__global__ void __launch_bounds__(128, 1)
    k_coarsest(LevelView L, const double* __restrict__ fden, const double* __restrict__ fy,
               const double* __restrict__ fg, const double* __restrict__ bvec, double* __restrict__ out, int n_coarse,
               double omega) {
    extern __shared__ double sm[];
    const int nz = L.nz, n = (int)L.n;
    const int64_t ld = L.ld;
    const int t = threadIdx.x, T = blockDim.x;
    const int plane = nz * n;                        // one array, compact [nz][n]
    double* A = sm;                                  // [9][nz][n]
    double* ua = A + kCoarsestArrays * plane;        // ping-pong iterates [nz][n]
    double* ub = ua + plane;
    double* zs = ub + plane;                         // [nz][T] Thomas z of each thread's column
    int* nb = reinterpret_cast<int*>(zs + nz * T);   // [3][n]
    const double* src[kCoarsestArrays] = {L.D, L.U, L.H0, L.H1, L.H2, bvec, fden, fy, fg};
    // all operand loads in flight at once (asynchronous 8-byte copies), one wait
    for (int a = 0; a < kCoarsestArrays; ++a)
        for (int k = 0; k < nz; ++k)
            for (int c = t; c < n; c += T) ptx::cp_async8(&A[a * plane + k * n + c], &src[a][(int64_t)k * ld + c]);
    for (int j = 0; j < 3; ++j)
        for (int c = t; c < n; c += T) nb[j * n + c] = L.nbr[(int64_t)j * ld + c];
    CSTAMP(0);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    CSTAMP(1);
    const double* __restrict__ D = A;
    const double* __restrict__ U = A + plane;
    const double* __restrict__ H0 = A + 2 * plane;
    const double* __restrict__ H1 = A + 3 * plane;
    const double* __restrict__ H2 = A + 4 * plane;
    const double* __restrict__ b = A + 5 * plane;
    const double* __restrict__ den = A + 6 * plane;
    const double* __restrict__ y = A + 7 * plane;
    const double* __restrict__ g = A + 8 * plane;
    const double* cur = nullptr;
    double* __restrict__ z = zs + t;
    for (int s = 0; s < n_coarse; ++s) {
        double* __restrict__ dst = (cur == ua) ? ub : ua;
        const double* __restrict__ cu = cur;
        for (int c = t; c < n; c += T) {
            const int n0 = nb[c], n1 = nb[n + c], n2 = nb[2 * n + c];
            // pass 1: residual of every layer (independent across layers -> ILP)
            auto residuals = [&]() {
#pragma unroll 8
                for (int k = 0; k < nz; ++k) {
                    const int i = k * n + c, row = k * n;
                    double r;
                    if (!cu) {
                        r = b[i];
                    } else {
                        const double uk = cu[i];
                        double acc = D[i] * uk;
                        if (k > 0) acc = acc + U[i - n] * cu[i - n];
                        if (k < nz - 1) acc = acc + U[i] * cu[i + n];
                        acc = acc + H0[i] * cu[row + n0];
                        acc = acc + H1[i] * cu[row + n1];
                        acc = acc + H2[i] * cu[row + n2];
                        r = b[i] - acc;
                    }
                    z[k * T] = r;
                }
            };
            residuals();
            // pass 2: forward elimination z_k = (r_k - U_{k-1} z_{k-1}) / den_k
            bool slow = false;
            double zprev = 0.0;
#pragma unroll 8
            for (int k = 0; k < nz; ++k) {
                const int i = k * n + c;
                const double r = z[k * T];
                const double num = (k == 0) ? r : r - U[i - n] * zprev;
                const double zk = div_fast_z(num, den[i], y[i], slow);
                z[k * T] = zk;
                zprev = zk;
            }
            if (slow) {                              // rare (e.g. zero numerator): redo with '/'
                residuals();
                zprev = 0.0;
                for (int k = 0; k < nz; ++k) {
                    const int i = k * n + c;
                    const double r = z[k * T];
                    const double num = (k == 0) ? r : r - U[i - n] * zprev;
                    const double zk = num / den[i];
                    z[k * T] = zk;
                    zprev = zk;
                }
            }
            if (s < 8) CSTAMP(3 + 3 * s);
            double dl = 0.0;
#pragma unroll 8
            for (int k = nz - 1; k >= 0; --k) {
                const int i = k * n + c;
                const double zk = z[k * T];
                dl = (k == nz - 1) ? zk : zk - g[i] * dl;
                dst[i] = cu ? cu[i] + omega * dl : omega * dl;
            }
        }
        if (s < 8) CSTAMP(4 + 3 * s);
        __syncthreads();
        cur = dst;
    }
    for (int k = 0; k < nz; ++k)
        for (int c = t; c < n; c += T) out[(int64_t)k * ld + c] = cur[k * n + c];
}

}  // namespace

#ifdef HMG_TIMING
extern "C" void hmg_debug_cs_timing(long long* out) { cudaMemcpyFromSymbol(out, g_cs_timing, sizeof(long long) * 64); }
#endif

size_t coarsest_smem_bytes(int nz, int64_t n, int threads) {
    return sizeof(double) * ((size_t)(kCoarsestArrays + 2) * nz * n + (size_t)nz * threads) + sizeof(int) * 3 * n;
}

void launch_coarsest(const Hierarchy& H, const DevLevel& L, const double* b, double* out, int n_coarse, double omega,
                     cudaStream_t s) {
    const int threads = (int)((L.n + 31) / 32 * 32);
    const size_t smem = coarsest_smem_bytes(H.nz, L.n, threads);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    ProfScope ps(H, kKCoarseTail, L.ref, s);
    k_coarsest<<<1, threads, smem, s>>>(L.view(H.nz), L.fden, L.fy, L.fg, b, out, n_coarse, omega);
    ++H.launches;
}

}  // namespace hmg
