// NEXT-3 core: batched per-column banded linear algebra of the
// next-to-lowest-order (NLO) discretisation -- the column operator H^_z of
// every vertical column is a banded matrix with m = 6 nz rows (6 DG1 unknowns
// per cell) and bandwidth n_BW = kl + ku + 1 = 27, inverted by a
// precomputed LU factorisation with partial pivoting (LAPACK dgbtrf) and the
// matching solve (dgbtrs); the paper's banded product kernel
// (P:752-762); and the p-coarsening DG1 <-> DG0 by the natural embedding
// (P:645-648).  Arithmetic follows oracle/band_oracle.c's order (LAPACK's),
// no contraction (-fmad=false), so results are bitwise the oracle's.
//
// B200 layout: every array is batched over the grid columns c (thread = grid
// column, a warp reads 32 consecutive columns = one coalesced 256-byte row):
//   LU factors  ab  [m][ldab][ld]   ldab = 2 kl + ku + 1, A(i, j) at
//                                   ab[(j * ldab + kl + ku + i - j) * ld + c]
//   pivots      ipiv [m][ld] int32  (0-based row interchanged with row j)
//   row storage ar  [m][bw][ld]     bw = kl + ku + 1, A(i, j) at
//                                   ar[(i * bw + kl + j - i) * ld + c]
//   vectors     [m][ld]             (a DG1 vector: [nz][6][ld])
//
// The solve is HBM-bound (Eq. 15: 4 m (3 n_BW + 4) bytes per column -- the
// kl multipliers and ipiv in the forward pass, the kl + ku + 1 rows of U in
// the backward pass, b in, x out): 32-column tiles, one producer warp
// streaming each elimination step's band rows (2-D TMA box) and pivot row
// (bulk copy) through a ring of mbarrier-guarded shared-memory stages, one
// consumer warp running the substitutions with the active part of the vector
// in registers (a sliding window of kl + 1 / kl + ku + 1 values).  The forward
// result y lives in x (L2) between the two passes and comes back through a
// register prefetch queue.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);

namespace {

constexpr int kBandCols = 32;      // grid columns per tile (one consumer warp)
constexpr int kBandThreads = 64;   // consumer warp + producer warp
constexpr int kYQ = 8;             // backward prefetch distance of y (steps)

// ---------------------------------------------------------------------------
// Factorisation: dgbtf2 per grid column, in place in global memory (setup).
// ---------------------------------------------------------------------------
template <int KL, int KU>
__global__ void __launch_bounds__(128) k_gbtrf(int64_t ncol, int m, double* __restrict__ ab, int64_t ld,
                                               int32_t* __restrict__ ipiv, unsigned long long* __restrict__ bad) {
    constexpr int KV = KL + KU, LDAB = 2 * KL + KU + 1;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    auto A = [&](int r, int j) -> double& { return ab[((int64_t)j * LDAB + r) * ld + c]; };
    for (int j = KU + 1; j < KV && j < m; ++j)
        for (int i = KV - j; i < KL; ++i) A(i, j) = 0.0;
    int ju = 0;
    bool singular = false;
    int first = 0;
    for (int j = 0; j < m; ++j) {
        if (j + KV < m) {
#pragma unroll
            for (int i = 0; i < KL; ++i) A(i, j + KV) = 0.0;
        }
        const int km = KL < m - 1 - j ? KL : m - 1 - j;
        double col[KL + 1];
#pragma unroll
        for (int i = 0; i <= KL; ++i) col[i] = (i <= km) ? A(KV + i, j) : 0.0;
        int jp = 0;
        double vmax = fabs(col[0]);
#pragma unroll
        for (int i = 1; i <= KL; ++i)
            if (i <= km && fabs(col[i]) > vmax) {
                vmax = fabs(col[i]);
                jp = i;
            }
        ipiv[(int64_t)j * ld + c] = j + jp;
        double piv = col[0];
#pragma unroll
        for (int i = 1; i <= KL; ++i)
            if (i == jp) piv = col[i];
        if (piv != 0.0) {
            const int jlast = j + KU + jp < m - 1 ? j + KU + jp : m - 1;
            if (jlast > ju) ju = jlast;
            if (jp != 0) {
                for (int cc = j; cc <= ju; ++cc) {
                    double& a = A(KV + jp - (cc - j), cc);
                    double& b = A(KV - (cc - j), cc);
                    const double t = a;
                    a = b;
                    b = t;
                }
                // the column's own entries in registers follow the swap
                const double t0 = col[0];
#pragma unroll
                for (int i = 1; i <= KL; ++i)
                    if (i == jp) col[i] = t0;
                col[0] = piv;
            }
            if (km > 0) {
                const double rp = 1.0 / col[0];
#pragma unroll
                for (int i = 1; i <= KL; ++i)
                    if (i <= km) {
                        col[i] = col[i] * rp;
                        A(KV + i, j) = col[i];
                    }
                for (int cc = j + 1; cc <= ju; ++cc) {
                    const double ujc = A(KV - (cc - j), cc);
                    if (ujc == 0.0) continue;
                    const double temp = -ujc;
#pragma unroll
                    for (int i = 1; i <= KL; ++i)
                        if (i <= km) {
                            double& a = A(KV + i - (cc - j), cc);
                            a = a + col[i] * temp;
                        }
                }
            }
        } else if (!singular) {
            singular = true;
            first = j;
        }
    }
    if (singular) atomicMin(bad, ((unsigned long long)c << 24) | (unsigned long long)first);
}

// ---------------------------------------------------------------------------
// Solve: dgbtrs ('N', one right-hand side), TMA-streamed.
// ---------------------------------------------------------------------------
struct BandSolveMaps {
    CUtensorMap fwd;   // ab rows, box kBandCols x max(KL, 1)
    CUtensorMap bwd;   // ab rows, box kBandCols x (KV + 1)
    CUtensorMap b;     // right-hand side [m][ld], box kBandCols x 1 (rows >= m zero-filled)
};

template <int KL, int KU>
struct SolveStage {
    static constexpr int KV = KL + KU;
    static constexpr int ROWS = KV + 1 > KL + 2 ? KV + 1 : KL + 2;   // bwd rows / fwd rows + b row
    static constexpr int KLB = KL > 0 ? KL : 1;                      // fwd box rows
    static constexpr int BYTES = ROWS * kBandCols * 8 + kBandCols * 4;
};

template <int KL, int KU>
__global__ void __launch_bounds__(kBandThreads, 1)
    k_gbtrs(const __grid_constant__ BandSolveMaps maps, const double* __restrict__ bvec,
            const int32_t* __restrict__ ipiv, double* __restrict__ x, int64_t ncol, int m, int64_t ld, int S) {
    using St = SolveStage<KL, KU>;
    constexpr int KV = KL + KU, LDAB = 2 * KL + KU + 1;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    unsigned char* stages = smem + 128 * ((16 * S + 127) / 128);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * kBandCols;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int nstages = 2 * m;
    if (warp == 1) {   // producer
        if (lane == 0) {
            for (int k = 0; k < nstages; ++k) {
                const int s = k % S;
                if (k >= S) ptx::mbar_wait(&empty[s], ((k / S) - 1) & 1);
                unsigned char* st = stages + (size_t)s * St::BYTES;
                if (k < m) {
                    const int j = k;
                    ptx::mbar_arrive_expect_tx(&full[s], (St::KLB + 1) * kBandCols * 8 + kBandCols * 4);
                    ptx::tma_load_2d(st, &maps.fwd, (int)c0, j * LDAB + KV + 1, &full[s]);
                    ptx::tma_load_2d(st + St::KLB * kBandCols * 8, &maps.b, (int)c0, j + KL + 1, &full[s]);
                    ptx::bulk_g2s(st + St::ROWS * kBandCols * 8, ipiv + (int64_t)j * ld + c0, kBandCols * 4, &full[s]);
                } else {
                    const int j = nstages - 1 - k;
                    ptx::mbar_arrive_expect_tx(&full[s], (KV + 1) * kBandCols * 8);
                    ptx::tma_load_2d(st, &maps.bwd, (int)c0, j * LDAB, &full[s]);
                }
            }
        }
        return;
    }
    // consumer warp: lane = grid column c0 + lane
    const int64_t c = c0 + lane;
    const bool live = c < ncol;
    // ---- forward: row interchanges and L multipliers, y into x ----
    double w[KL + 1];
#pragma unroll
    for (int q = 0; q <= KL; ++q) w[q] = (q < m) ? bvec[(int64_t)q * ld + c] : 0.0;
    for (int j = 0; j < m; ++j) {
        const int s = j % S;
        ptx::mbar_wait(&full[s], (j / S) & 1);
        const double* st = reinterpret_cast<const double*>(stages + (size_t)s * St::BYTES);
        const int32_t* pv = reinterpret_cast<const int32_t*>(st + St::ROWS * kBandCols);
        if (KL > 0 && j < m - 1) {
            const int lm = KL < m - 1 - j ? KL : m - 1 - j;
            const int p = pv[lane] - j;
            const double old0 = w[0];
            double new0 = old0;
#pragma unroll
            for (int q = 1; q <= KL; ++q) {
                const bool hit = p == q;
                const double wq = w[q];
                new0 = hit ? wq : new0;
                w[q] = hit ? old0 : wq;
            }
            w[0] = new0;
            if (new0 != 0.0) {
                const double temp = -new0;
#pragma unroll
                for (int i = 1; i <= KL; ++i)
                    if (i <= lm) w[i] = w[i] + st[(i - 1) * kBandCols + lane] * temp;
            }
        }
        const double incoming = st[St::KLB * kBandCols + lane];   // b row j + KL + 1 (0 past the end)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        if (live) x[(int64_t)j * ld + c] = w[0];
#pragma unroll
        for (int q = 0; q < KL; ++q) w[q] = w[q + 1];
        w[KL] = incoming;
    }
    // ---- backward: U (kl + ku super-diagonals), column-oriented (dtbsv) ----
    double u[KV + 1];   // u[KV] = x(j), u[KV - i] = x(j - i)
#pragma unroll
    for (int q = 0; q <= KV; ++q) {
        const int idx = m - 1 - KV + q;
        u[q] = idx >= 0 ? x[(int64_t)idx * ld + c] : 0.0;
    }
    double yq[kYQ];   // y(j - KV - 1 - d) prefetched kYQ steps ahead
#pragma unroll
    for (int d = 0; d < kYQ; ++d) {
        const int idx = m - 1 - KV - 1 - d;
        yq[d] = idx >= 0 ? x[(int64_t)idx * ld + c] : 0.0;
    }
    for (int t0 = 0; t0 < m; t0 += kYQ) {
#pragma unroll
        for (int d = 0; d < kYQ; ++d) {
            const int t = t0 + d;
            if (t < m) {
                const int j = m - 1 - t;
                const int k = m + t;
                const int s = k % S;
                ptx::mbar_wait(&full[s], (k / S) & 1);
                const double* st = reinterpret_cast<const double*>(stages + (size_t)s * St::BYTES);
                if (u[KV] != 0.0) {
                    u[KV] = u[KV] / st[KV * kBandCols + lane];
                    const double temp = u[KV];
#pragma unroll
                    for (int i = 1; i <= KV; ++i)
                        if (j - i >= 0) u[KV - i] = u[KV - i] - temp * st[(KV - i) * kBandCols + lane];
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
                if (live) x[(int64_t)j * ld + c] = u[KV];
#pragma unroll
                for (int q = KV; q > 0; --q) u[q] = u[q - 1];
                u[0] = yq[d];
                const int idx = j - KV - 1 - kYQ;
                yq[d] = idx >= 0 ? x[(int64_t)idx * ld + c] : 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Product y = A x, the paper's row-wise band kernel, TMA-streamed.
// ---------------------------------------------------------------------------
struct BandApplyMaps {
    CUtensorMap a;   // ar rows [m * bw][ld], box kBandCols x bw
    CUtensorMap x;   // x [m][ld], box kBandCols x 1
};

template <int KL, int KU>
__global__ void __launch_bounds__(kBandThreads, 1)
    k_gbmv(const __grid_constant__ BandApplyMaps maps, const double* __restrict__ xin, double* __restrict__ y,
           int64_t ncol, int m, int64_t ld, int S) {
    constexpr int BW = KL + KU + 1;
    constexpr int BYTES = (BW + 1) * kBandCols * 8;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    unsigned char* stages = smem + 128 * ((16 * S + 127) / 128);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * kBandCols;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == 1) {
        if (lane == 0) {
            for (int i = 0; i < m; ++i) {
                const int s = i % S;
                if (i >= S) ptx::mbar_wait(&empty[s], ((i / S) - 1) & 1);
                unsigned char* st = stages + (size_t)s * BYTES;
                ptx::mbar_arrive_expect_tx(&full[s], BYTES);
                ptx::tma_load_2d(st, &maps.a, (int)c0, i * BW, &full[s]);
                ptx::tma_load_2d(st + BW * kBandCols * 8, &maps.x, (int)c0, i + KU + 1, &full[s]);
            }
        }
        return;
    }
    const int64_t c = c0 + lane;
    double w[BW];   // w[q] = x(i - KL + q)
#pragma unroll
    for (int q = 0; q < BW; ++q) {
        const int j = q - KL;
        w[q] = (j >= 0 && j < m) ? xin[(int64_t)j * ld + c] : 0.0;
    }
    for (int i = 0; i < m; ++i) {
        const int s = i % S;
        ptx::mbar_wait(&full[s], (i / S) & 1);
        const double* st = reinterpret_cast<const double*>(stages + (size_t)s * BYTES);
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < BW; ++q) {
            const int j = i - KL + q;
            if (j >= 0 && j < m) acc = acc + st[q * kBandCols + lane] * w[q];
        }
        const double incoming = st[BW * kBandCols + lane];   // x(i + KU + 1)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        if (c < ncol) y[(int64_t)i * ld + c] = acc;
#pragma unroll
        for (int q = 0; q < BW - 1; ++q) w[q] = w[q + 1];
        w[BW - 1] = incoming;
    }
}

// ---------------------------------------------------------------------------
// p-coarsening DG1 <-> DG0 (natural embedding; reading R21).
// ---------------------------------------------------------------------------
__global__ void k_p_restrict(int64_t ncol, int nz, const double* __restrict__ r1, int64_t ld, double* __restrict__ b0) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c >= ncol) return;
    const double* r = r1 + (int64_t)6 * k * ld + c;
    b0[(int64_t)k * ld + c] = ((((r[0] + r[ld]) + r[2 * ld]) + r[3 * ld]) + r[4 * ld]) + r[5 * ld];
}

__global__ void k_p_prolong_add(int64_t ncol, int nz, const double* __restrict__ u0, int64_t ld, double* __restrict__ u1) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (c >= ncol) return;
    const double v = u0[(int64_t)k * ld + c];
    double* u = u1 + (int64_t)6 * k * ld + c;
#pragma unroll
    for (int d = 0; d < 6; ++d) u[d * ld] = u[d * ld] + v;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int stages_for(int bytes_per_stage) {
    // two CTAs per SM: ~100 KB of ring each
    int S = (100 * 1024) / bytes_per_stage;
    return S < 4 ? 4 : (S > 32 ? 32 : S);
}

size_t smem_for(int S, int bytes_per_stage) { return 128 * ((16 * S + 127) / 128) + (size_t)S * bytes_per_stage; }

template <int KL, int KU>
void factor_t(int64_t ncol, int m, double* ab, int64_t ld, int32_t* ipiv, unsigned long long* bad, cudaStream_t s) {
    k_gbtrf<KL, KU><<<(unsigned)((ncol + 127) / 128), 128, 0, s>>>(ncol, m, ab, ld, ipiv, bad);
}

template <int KL, int KU>
void solve_t(int64_t ncol, int m, const double* ab, int64_t ld, const int32_t* ipiv, const double* b, double* x,
             cudaStream_t s) {
    using St = SolveStage<KL, KU>;
    constexpr int KV = KL + KU, LDAB = 2 * KL + KU + 1;
    BandSolveMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    maps.fwd = make_tensor_map(ab, ld, (int64_t)m * LDAB, kBandCols, St::KLB, 1);
    maps.bwd = make_tensor_map(ab, ld, (int64_t)m * LDAB, kBandCols, KV + 1, 1);
    maps.b = make_tensor_map(b, ld, m, kBandCols, 1, 1);
    const int S = stages_for(St::BYTES);
    const size_t smem = smem_for(S, St::BYTES);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gbtrs<KL, KU>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    k_gbtrs<KL, KU><<<(unsigned)((ncol + kBandCols - 1) / kBandCols), kBandThreads, smem, s>>>(maps, b, ipiv, x, ncol,
                                                                                             m, ld, S);
}

template <int KL, int KU>
void apply_t(int64_t ncol, int m, const double* ar, int64_t ld, const double* x, double* y, cudaStream_t s) {
    constexpr int BW = KL + KU + 1;
    constexpr int BYTES = (BW + 1) * kBandCols * 8;
    BandApplyMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    maps.a = make_tensor_map(ar, ld, (int64_t)m * BW, kBandCols, BW, 1);
    maps.x = make_tensor_map(x, ld, m, kBandCols, 1, 1);
    const int S = stages_for(BYTES);
    const size_t smem = smem_for(S, BYTES);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gbmv<KL, KU>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    k_gbmv<KL, KU><<<(unsigned)((ncol + kBandCols - 1) / kBandCols), kBandThreads, smem, s>>>(maps, x, y, ncol, m, ld,
                                                                                            S);
}

// The (kl, ku) pairs compiled: the NLO column operator (13, 13),
// the LO one (1, 1), and small shapes the tests use.
#define HMG_BAND_SHAPES(X) X(13, 13) X(1, 1) X(2, 2) X(3, 5) X(5, 2) X(0, 0)

}  // namespace

bool band_shape_supported(int kl, int ku) {
#define X(a, b) if (kl == a && ku == b) return true;
    HMG_BAND_SHAPES(X)
#undef X
    return false;
}

void launch_band_factor(int64_t ncol, int m, int kl, int ku, double* ab, int64_t ld, int32_t* ipiv,
                        unsigned long long* bad, cudaStream_t s) {
#define X(a, b) if (kl == a && ku == b) return factor_t<a, b>(ncol, m, ab, ld, ipiv, bad, s);
    HMG_BAND_SHAPES(X)
#undef X
}

void launch_band_solve(int64_t ncol, int m, int kl, int ku, const double* ab, int64_t ld, const int32_t* ipiv,
                       const double* b, double* x, cudaStream_t s) {
#define X(a, bb) if (kl == a && ku == bb) return solve_t<a, bb>(ncol, m, ab, ld, ipiv, b, x, s);
    HMG_BAND_SHAPES(X)
#undef X
}

void launch_band_apply(int64_t ncol, int m, int kl, int ku, const double* ar, int64_t ld, const double* x, double* y,
                       cudaStream_t s) {
#define X(a, b) if (kl == a && ku == b) return apply_t<a, b>(ncol, m, ar, ld, x, y, s);
    HMG_BAND_SHAPES(X)
#undef X
}

void launch_p_restrict(int64_t ncol, int nz, const double* r1, int64_t ld, double* b0, cudaStream_t s) {
    k_p_restrict<<<dim3((unsigned)((ncol + 255) / 256), (unsigned)nz), 256, 0, s>>>(ncol, nz, r1, ld, b0);
}

void launch_p_prolong_add(int64_t ncol, int nz, const double* u0, int64_t ld, double* u1, cudaStream_t s) {
    k_p_prolong_add<<<dim3((unsigned)((ncol + 255) / 256), (unsigned)nz), 256, 0, s>>>(ncol, nz, u0, ld, u1);
}

}  // namespace hmg
