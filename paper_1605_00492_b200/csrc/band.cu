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
// the backward pass, b in, x out): 128-column tiles, one producer warp
// streaming several elimination steps' band rows (3-D TMA boxes, evict-first)
// and pivot / b rows through a ring of mbarrier-guarded shared-memory stages,
// four consumer warps (thread = grid column) running the substitutions with
// the active part of the vector in registers (a sliding window of kl + 1 /
// kl + ku + 1 values).  The forward result y lives in x (L2) between the two
// passes and comes back through a register prefetch queue.  The product
// streams its row-wise band the same way (32-column tiles).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "hmg_internal.h"
#include "sm100_ptx.cuh"

namespace hmg {

CUtensorMap make_tensor_map(const double* base, int64_t ld, int64_t rows, int box_x, int G, int planes);

namespace {

constexpr int kBandCols = 32;      // grid columns per tile (one consumer warp)
constexpr int kBandThreads = 64;   // consumer warp + producer warp
constexpr int kYQ = 16;            // backward prefetch distance of y (steps)

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
// Solve: dgbtrs ('N', one right-hand side), TMA-streamed.  A stage carries G
// consecutive elimination steps: forward, a 3-D box of the kl multiplier rows
// of G matrix columns, the G b rows entering the window and the G pivot rows;
// backward, a 3-D box of the kl + ku + 1 rows of U of G matrix columns.
// ---------------------------------------------------------------------------
struct BandSolveMaps {
    CUtensorMap fwd;   // ab as {ld, ldab, m}, box {COLS, max(kl, 1), GF}
    CUtensorMap bwd;   // ab as {ld, ldab, m}, box {COLS, kl + ku + 1, GB}
    CUtensorMap b;     // b as {ld, m}, box {COLS, GF} (rows >= m zero-filled)
    CUtensorMap piv;   // ipiv as {ld, m} int32, box {COLS, GF}
};

template <int KL, int KU, int NW, int BUDGET_KB = 100>
struct SolveCfg {
    static constexpr int KV = KL + KU;
    static constexpr int COLS = 32 * NW;
    static constexpr int KLB = KL > 0 ? KL : 1;
    static constexpr int GB = 2;                                          // backward steps per stage
    static constexpr int BWD_BYTES = GB * (KV + 1) * COLS * 8;
    static constexpr int GF = (BWD_BYTES / ((KLB + 1) * COLS * 8 + COLS * 4)) > 0
                                  ? (BWD_BYTES / ((KLB + 1) * COLS * 8 + COLS * 4)) : 1;   // forward steps per stage
    static constexpr int FWD_L = GF * KLB * COLS * 8;                    // multiplier rows
    static constexpr int FWD_B = GF * COLS * 8;                          // b rows
    static constexpr int FWD_P = GF * COLS * 4;                          // pivot rows
    static constexpr int FWD_BYTES = FWD_L + FWD_B + FWD_P;
    static constexpr int RAW = BWD_BYTES > FWD_BYTES ? BWD_BYTES : FWD_BYTES;
    static constexpr int BYTES = (RAW + 127) / 128 * 128;
    static constexpr int S0 = (BUDGET_KB * 1024) / BYTES;                 // ring stages within the budget
    static constexpr int S = S0 < 3 ? 3 : (S0 > 24 ? 24 : S0);
    static constexpr int HDR = 128 * ((16 * S + 127) / 128);              // mbarriers
    static constexpr size_t SMEM = HDR + (size_t)S * BYTES;
};

template <int KL, int KU, int NW, int BUDGET_KB>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_gbtrs(const __grid_constant__ BandSolveMaps maps, const double* __restrict__ bvec, double* __restrict__ x,
            int64_t ncol, int m, int64_t ld) {
    using C = SolveCfg<KL, KU, NW, BUDGET_KB>;
    constexpr int KV = C::KV, COLS = C::COLS, S = C::S, GF = C::GF, GB = C::GB;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    unsigned char* stages = smem + C::HDR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * COLS;
    const int nf = (m + GF - 1) / GF, nb = (m + GB - 1) / GB;   // forward / backward stages
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], NW);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == NW) {   // producer
        if (lane == 0) {
            // the factors are read once: evict them first, so that y (written by
            // the forward pass, read back by the backward pass) stays in L2
            const uint64_t pol = ptx::policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            for (int k = 0; k < nf + nb; ++k) {
                if (k >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
                unsigned char* st = stages + (size_t)s * C::BYTES;
                if (k < nf) {
                    const int j0 = k * GF;
                    ptx::mbar_arrive_expect_tx(&full[s], C::FWD_BYTES);
                    ptx::tma_load_3d_hint(st, &maps.fwd, (int)c0, KV + 1, j0, &full[s], pol);
                    ptx::tma_load_2d_hint(st + C::FWD_L, &maps.b, (int)c0, j0 + KL + 1, &full[s], pol);
                    ptx::tma_load_2d_hint(st + C::FWD_L + C::FWD_B, &maps.piv, (int)c0, j0, &full[s], pol);
                } else {
                    // backward stage q covers steps j = jtop - GB + 1 .. jtop (box starts at the lower one)
                    const int q = k - nf;
                    const int jtop = m - 1 - q * GB;
                    ptx::mbar_arrive_expect_tx(&full[s], C::BWD_BYTES);
                    ptx::tma_load_3d_hint(st, &maps.bwd, (int)c0, 0, jtop - GB + 1, &full[s], pol);
                }
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    // consumer warps: thread = grid column c0 + 32 warp + lane
    const int col = warp * 32 + lane;
    const int64_t c = c0 + col;
    const bool live = c < ncol;
    // reads of lanes past the last column (a partial tile; c may exceed ld) use
    // the last column instead: results of those lanes are never stored
    const int64_t cr = live ? c : ncol - 1;
    int s = 0;
    uint32_t ph = 0;
    // ---- forward: row interchanges and L multipliers, y into x ----
    double w[KL + 1];
#pragma unroll
    for (int q = 0; q <= KL; ++q) w[q] = (q < m) ? bvec[(int64_t)q * ld + cr] : 0.0;
    for (int k = 0; k < nf; ++k) {
        ptx::mbar_wait(&full[s], ph);
        const unsigned char* st = stages + (size_t)s * C::BYTES;
        const double* Ls = reinterpret_cast<const double*>(st);
        const double* bs = reinterpret_cast<const double*>(st + C::FWD_L);
        const int32_t* ps = reinterpret_cast<const int32_t*>(st + C::FWD_L + C::FWD_B);
        double yv[GF];
        double inc[GF];
        int pv[GF];
#pragma unroll
        for (int g = 0; g < GF; ++g) {
            inc[g] = bs[g * COLS + col];
            pv[g] = ps[g * COLS + col];
        }
#pragma unroll
        for (int g = 0; g < GF; ++g) {
            const int j = k * GF + g;
            if (KL > 0 && j < m - 1) {
                const int lm = KL < m - 1 - j ? KL : m - 1 - j;
                const int p = pv[g] - j;
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
                        if (i <= lm) w[i] = w[i] + Ls[(g * C::KLB + i - 1) * COLS + col] * temp;
                }
            }
            yv[g] = w[0];
#pragma unroll
            for (int q = 0; q < KL; ++q) w[q] = w[q + 1];
            w[KL] = inc[g];   // b row j + KL + 1 (0 past the end)
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        if (++s == S) {
            s = 0;
            ph ^= 1;
        }
        if (live) {
#pragma unroll
            for (int g = 0; g < GF; ++g)
                if (k * GF + g < m) x[(int64_t)(k * GF + g) * ld + c] = yv[g];
        }
    }
    // ---- backward: U (kl + ku super-diagonals), column-oriented (dtbsv) ----
    double u[KV + 1];   // u[KV] = x(j), u[KV - i] = x(j - i)
#pragma unroll
    for (int q = 0; q <= KV; ++q) {
        const int idx = m - 1 - KV + q;
        u[q] = idx >= 0 ? x[(int64_t)idx * ld + cr] : 0.0;
    }
    constexpr int YQ = 2 * GB * ((kYQ + 2 * GB - 1) / (2 * GB));   // prefetch distance, a multiple of GB
    double yq[YQ];      // y(j - KV - 1 - d), d steps ahead
#pragma unroll
    for (int d = 0; d < YQ; ++d) {
        const int idx = m - 1 - KV - 1 - d;
        yq[d] = idx >= 0 ? x[(int64_t)idx * ld + cr] : 0.0;
    }
    for (int q0 = 0; q0 < nb; q0 += YQ / GB) {
#pragma unroll
        for (int qq = 0; qq < YQ / GB; ++qq) {
            const int q = q0 + qq;
            if (q < nb) {
                ptx::mbar_wait(&full[s], ph);
                const double* Us = reinterpret_cast<const double*>(stages + (size_t)s * C::BYTES);
                const int jtop = m - 1 - q * GB;
                double xo[GB];
#pragma unroll
                for (int g = 0; g < GB; ++g) {
                    const int j = jtop - g;   // this step's column; plane GB - 1 - g of the box
                    const double* Uj = Us + (GB - 1 - g) * (KV + 1) * COLS;
                    if (j >= 0) {
                        if (u[KV] != 0.0) {
                            u[KV] = u[KV] / Uj[KV * COLS + col];
                            const double temp = u[KV];
#pragma unroll
                            for (int i = 1; i <= KV; ++i)
                                if (j - i >= 0) u[KV - i] = u[KV - i] - temp * Uj[(KV - i) * COLS + col];
                        }
                    }
                    xo[g] = u[KV];
#pragma unroll
                    for (int r = KV; r > 0; --r) u[r] = u[r - 1];
                    const int d = qq * GB + g;
                    u[0] = yq[d];
                    const int idx = j - KV - 1 - YQ;
                    yq[d] = idx >= 0 ? x[(int64_t)idx * ld + cr] : 0.0;
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
                if (live) {
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (jtop - g >= 0) x[(int64_t)(jtop - g) * ld + c] = xo[g];
                }
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
    const int64_t cr = c < ncol ? c : ncol - 1;   // partial tile: read a valid column, never store
    double w[BW];   // w[q] = x(i - KL + q)
#pragma unroll
    for (int q = 0; q < BW; ++q) {
        const int j = q - KL;
        w[q] = (j >= 0 && j < m) ? xin[(int64_t)j * ld + cr] : 0.0;
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

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Tensor map over a row-major array of `rank` dims (dims[0] fastest), box
// `box`; out-of-range box elements are zero-filled.
CUtensorMap encode(CUtensorMapDataType dt, int esize, int rank, const void* base, const uint64_t* dims,
                   const uint32_t* box) {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeFn) nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], e[5];
    uint64_t stride = (uint64_t)esize;
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = 1;
        if (i > 0) st[i - 1] = stride;
        stride *= dims[i];
    }
    const CUresult r = fn(&m, dt, (cuuint32_t)rank, const_cast<void*>(base), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
    return m;
}

template <int KL, int KU, int NW, int BUD>
void solve_cfg(int64_t ncol, int m, const double* ab, int64_t ld, const int32_t* ipiv, const double* b, double* x,
               cudaStream_t s) {
    using C = SolveCfg<KL, KU, NW, BUD>;
    constexpr int LDAB = 2 * KL + KU + 1;
    BandSolveMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    {
        const uint64_t dims[3] = {(uint64_t)ld, (uint64_t)LDAB, (uint64_t)m};
        const uint32_t boxf[3] = {(uint32_t)C::COLS, (uint32_t)C::KLB, (uint32_t)C::GF};
        const uint32_t boxb[3] = {(uint32_t)C::COLS, (uint32_t)(C::KV + 1), (uint32_t)C::GB};
        maps.fwd = encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 3, ab, dims, boxf);
        maps.bwd = encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 3, ab, dims, boxb);
        const uint64_t vd[2] = {(uint64_t)ld, (uint64_t)m};
        const uint32_t vb[2] = {(uint32_t)C::COLS, (uint32_t)C::GF};
        maps.b = encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, b, vd, vb);
        maps.piv = encode(CU_TENSOR_MAP_DATA_TYPE_INT32, 4, 2, ipiv, vd, vb);
    }
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gbtrs<KL, KU, NW, BUD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    k_gbtrs<KL, KU, NW, BUD><<<(unsigned)((ncol + C::COLS - 1) / C::COLS), 32 * (NW + 1), C::SMEM, s>>>(maps, b, x,
                                                                                                     ncol, m, ld);
}

// 128 grid columns per CTA (four consumer warps; 1 KB box rows), one CTA per
// SM with a 3-stage ring of 55 KB stages: measured best at the NLO size
// (tools/gpu_runs/r02f.sh: 32-column tiles with 2 / 3 CTAs per SM 4.1 / 5.1
// TB/s, 64-column 5.1, 128-column 5.53 TB/s; the factors stream with an
// evict-first L2 policy so that y stays in L2 between the two passes).
template <int KL, int KU>
void solve_t(int64_t ncol, int m, const double* ab, int64_t ld, const int32_t* ipiv, const double* b, double* x,
             cudaStream_t s) {
    solve_cfg<KL, KU, 4, 200>(ncol, m, ab, ld, ipiv, b, x, s);
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
