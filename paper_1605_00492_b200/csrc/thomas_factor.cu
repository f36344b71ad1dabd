// Thomas factors and the coarsest-level solve.
//  * k_factor: the pivots den_k, their refined reciprocals y_k and the
//    multipliers g_k of every column (reading R6 order; they depend on the
//    matrix only), computed once at setup for the latency-bound levels, whose
//    sweeps then run only the z recurrence.
//  * k_pivot_check: the same pivots checked once on every other level (a bad
//    pivot is reported by hmg_build_hierarchy).
//  * k_coarsest: the coarsest level's n_coarse sweeps from zero (
//    BASELINE.json: 20) in one CTA's shared memory.
#include <cfloat>

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

}  // namespace

void launch_pivot_check(const Hierarchy& H, const DevLevel& L, unsigned int* gslow, cudaStream_t s) {
    k_pivot_check<<<(unsigned)((L.n + 127) / 128), 128, 0, s>>>(L.view(H.nz), L.ref, &H.scal->bad, gslow);
    ++H.launches;
}

void launch_factor(const Hierarchy& H, const DevLevel& L, cudaStream_t s) {
    k_factor<<<(unsigned)((L.n + 127) / 128), 128, 0, s>>>(L.view(H.nz), L.fden, L.fy, L.fg, L.ref, &H.scal->bad);
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
