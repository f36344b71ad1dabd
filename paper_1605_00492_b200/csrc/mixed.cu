// NEXT-4: the mixed velocity-pressure system around the
// V-cycle -- Eq. 5 with omega_N = 0, the Schur-complement
// preconditioner of Eq. 6 with a lumped velocity mass, and the
// vector kernels of restarted GMRES.  Readings R15-R20 of
// DESIGN.md; the host driver (hmg_mixed_gmres) is in api.cu.
//
// Unknowns, one device vector [U_h | U_z | P] (reading R15):
//   U_h [nz][ldh]   normal flux through the vertical face of edge e in layer
//                   k, positive from cell a to cell b (a < b), ldh = ne
//                   rounded up to 32;
//   U_z [nz-1][ld]  flux through interface i = 1..nz-1 of column c (row
//                   i-1), positive upward (u.n = 0 at top and bottom);
//   P   [nz][ld]    pressure, the layout of every other fine-level vector,
//                   so the preconditioner's V-cycle reads and writes it in
//                   place.  Padding entries are zero and stay zero.
// A = [[M2, -omega D^T], [omega D, M3]], omega = sqrt(w2).
//
// Every kernel follows the operation order of oracle/hmg_oracle.c's mixed_*
// functions (written independently from the same readings), so applies and
// preconditioner applications are bitwise the oracle's.  They are thread-per-
// edge or thread-per-column kernels walking the layers: HBM-bound streams
// (U rows, lam, P) plus same-row neighbour gathers served by L2.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "hmg_internal.h"
#include "mesh.h"
#include "sm100_ptx.cuh"

namespace hmg {

namespace {

constexpr int kMixBlock = 128;

struct MixView {
    int nz;
    int64_t n, ld, ne, ldh, off_z, off_p;
    double dz, om;
    double sn;                          // 1 + omega_N^2 (reading R24)
    const int32_t* __restrict__ eca;    // [ldh] lower cell a
    const int32_t* __restrict__ ecb;    // [ldh] upper cell b
    const int32_t* __restrict__ ee;     // [6][ldh] edges of a's slots 0..2, then b's
    const double* __restrict__ eg;      // [6][ldh] RT0 mass row of the edge in a, then in b
    const int32_t* __restrict__ ce;     // [3][ld] edge across each slot
    const double* __restrict__ cs;      // [3][ld] +1 if the edge's flux leaves the cell
    const double* __restrict__ lam;     // [nz][ld]
    const double* __restrict__ area;    // [ld] (row 0 of geom)
    const double* __restrict__ IL;      // [off_p]: lumped inverse of every velocity dof
};

MixView view(const Hierarchy& H) {
    const MixedSystem& M = *H.mix;
    const DevLevel& L = H.lev[H.fine_ref];
    MixView v;
    v.nz = H.nz;
    v.n = L.n;
    v.ld = L.ld;
    v.ne = M.ne;
    v.ldh = M.ldh;
    v.off_z = M.off_z;
    v.off_p = M.off_p;
    v.dz = H.dz;
    v.om = M.omega;
    v.sn = H.sn;
    v.eca = M.eca;
    v.ecb = M.ecb;
    v.ee = M.ee;
    v.eg = M.eg;
    v.ce = M.ce;
    v.cs = M.cs;
    v.lam = L.lam;
    v.area = L.geom;
    v.IL = M.IL;
    return v;
}

unsigned nblk(int64_t n) { return (unsigned)((n + kMixBlock - 1) / kMixBlock); }

// Lumped inverse (reading R19): IL_h[k][e] = ((len dz) lamf) / cd (len, cd of
// the edge as seen from a), IL_z[i-1][c] = (area lamf) / dz, lamf = 0.5 (lam_a + lam_b).
__global__ void k_mixed_il(MixView V, const double* __restrict__ geom, const int32_t* __restrict__ esa,
                           double* __restrict__ IL) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < V.ne) {
        const int64_t a = V.eca[t], b = V.ecb[t];
        const int j = esa[t];
        const double len = geom[(1 + j) * V.ld + a], cd = geom[(4 + j) * V.ld + a];
        for (int k = 0; k < V.nz; ++k) {
            const double lamf = 0.5 * (V.lam[k * V.ld + a] + V.lam[k * V.ld + b]);
            IL[k * V.ldh + t] = ((len * V.dz) * lamf) / cd;
        }
    }
    if (t < V.n) {
        const double ar = V.area[t];
        for (int i = 1; i <= V.nz - 1; ++i) {
            const double lamf = 0.5 * (V.lam[(i - 1) * V.ld + t] + V.lam[i * V.ld + t]);
            IL[V.off_z + (i - 1) * V.ld + t] = ((ar * lamf) / V.dz) / V.sn;   // lumping of M~2z (R24)
        }
    }
}

// y_h = M2h U_h - omega (P_a - P_b) per (edge, layer) (reading R18):
// t_s = ((g0 U[E0] + g1 U[E1]) + g2 U[E2]), m_s = t_s / (dz lam_s), y = (m_a + m_b) - omega (P_a - P_b)
__global__ void __launch_bounds__(kMixBlock, 8) k_mixed_apply_h(MixView V, const double* __restrict__ x,
                                                                double* __restrict__ y) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= V.ne) return;
    const int64_t a = V.eca[e], b = V.ecb[e];
    int32_t E[6];
    double g[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        E[q] = V.ee[q * V.ldh + e];
        g[q] = V.eg[q * V.ldh + e];
    }
    const double* P = x + V.off_p;
#pragma unroll 1
    for (int k = 0; k < V.nz; ++k) {
        const double* Ur = x + k * V.ldh;
        double ta = g[0] * Ur[E[0]];
        ta = ta + g[1] * Ur[E[1]];
        ta = ta + g[2] * Ur[E[2]];
        double tb = g[3] * Ur[E[3]];
        tb = tb + g[4] * Ur[E[4]];
        tb = tb + g[5] * Ur[E[5]];
        const double ma = ta / (V.dz * V.lam[k * V.ld + a]);
        const double mb = tb / (V.dz * V.lam[k * V.ld + b]);
        const double th = P[k * V.ld + a] - P[k * V.ld + b];
        y[k * V.ldh + e] = (ma + mb) - V.om * th;
    }
}

// y_z = M2z U_z - omega (P_{i-1} - P_i) per (column, interface) and
// y_p = omega (D U) + vol P per (column, layer); one thread per column.
__global__ void __launch_bounds__(kMixBlock) k_mixed_apply_zp(MixView V, const double* __restrict__ x,
                                                              double* __restrict__ y) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= V.n) return;
    const double ar = V.area[c], dz = V.dz;
    const double* W = x + V.off_z + c;
    const double* P = x + V.off_p + c;
    const double* lam = V.lam + c;
    const int nz = V.nz;
    const int64_t ld = V.ld;
#pragma unroll 4
    for (int i = 1; i <= nz - 1; ++i) {
        const double slo = ar * lam[(i - 1) * ld];
        const double shi = ar * lam[i * ld];
        const double dg = ((dz / 3.0) / slo) + ((dz / 3.0) / shi);
        double v = dg * W[(i - 1) * ld];
        if (i - 1 >= 1) v = v + ((dz / 6.0) / slo) * W[(i - 2) * ld];
        if (i + 1 <= nz - 1) v = v + ((dz / 6.0) / shi) * W[i * ld];
        v = v * V.sn;                                  // M~2z = (1 + omega_N^2) M2z (Eq. 5)
        y[V.off_z + (i - 1) * ld + c] = v - V.om * (P[(i - 1) * ld] - P[i * ld]);
    }
    const int32_t E0 = V.ce[c], E1 = V.ce[ld + c], E2 = V.ce[2 * ld + c];
    const double s0 = V.cs[c], s1 = V.cs[ld + c], s2 = V.cs[2 * ld + c];
    const double vol = ar * dz;
#pragma unroll 4
    for (int k = 0; k < nz; ++k) {
        const double* Ur = x + k * V.ldh;
        double d = s0 * Ur[E0];
        d = d + s1 * Ur[E1];
        d = d + s2 * Ur[E2];
        if (k + 1 <= nz - 1) d = d + W[k * ld];
        if (k >= 1) d = d - W[(k - 1) * ld];
        y[V.off_p + k * ld + c] = V.om * d + vol * P[k * ld];
    }
}

// Preconditioner step 1: g = f_p - omega D (L^-1 f_u), per (column, layer).
__global__ void __launch_bounds__(kMixBlock) k_mixed_pre_p(MixView V, const double* __restrict__ f,
                                                           double* __restrict__ g) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= V.n) return;
    const int64_t ld = V.ld;
    const int32_t E0 = V.ce[c], E1 = V.ce[ld + c], E2 = V.ce[2 * ld + c];
    const double s0 = V.cs[c], s1 = V.cs[ld + c], s2 = V.cs[2 * ld + c];
    const int nz = V.nz;
#pragma unroll 4
    for (int k = 0; k < nz; ++k) {
        const int64_t r = k * V.ldh;
        double d = s0 * (f[r + E0] * V.IL[r + E0]);
        d = d + s1 * (f[r + E1] * V.IL[r + E1]);
        d = d + s2 * (f[r + E2] * V.IL[r + E2]);
        if (k + 1 <= nz - 1) {
            const int64_t q = V.off_z + k * ld + c;
            d = d + f[q] * V.IL[q];
        }
        if (k >= 1) {
            const int64_t q = V.off_z + (k - 1) * ld + c;
            d = d - f[q] * V.IL[q];
        }
        g[k * ld + c] = f[V.off_p + k * ld + c] - V.om * d;
    }
}

// Preconditioner step 3: x_u = L^-1 (f_u + omega D^T x_p); x_p is already in x.
__global__ void __launch_bounds__(kMixBlock) k_mixed_pre_u(MixView V, const double* __restrict__ f,
                                                           double* __restrict__ x) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double* xp = x + V.off_p;
    const int64_t t = t0 < V.ne ? t0 : t0 - V.ne;   // threads [0, ne): edges; [ne, ne + n): columns
    if (t0 < V.ne) {
        const int64_t a = V.eca[t], b = V.ecb[t];
#pragma unroll 4
        for (int k = 0; k < V.nz; ++k) {
            const int64_t q = k * V.ldh + t;
            x[q] = (f[q] + V.om * (xp[k * V.ld + a] - xp[k * V.ld + b])) * V.IL[q];
        }
    }
    if (t0 >= V.ne && t < V.n) {
#pragma unroll 4
        for (int i = 1; i <= V.nz - 1; ++i) {
            const int64_t q = V.off_z + (i - 1) * V.ld + t;
            x[q] = (f[q] + V.om * (xp[(i - 1) * V.ld + t] - xp[i * V.ld + t])) * V.IL[q];
        }
    }
}

// ---- flat vector kernels of GMRES (padding entries are zero) ----
// Every GMRES work vector is library-allocated (16-byte aligned, ntot even),
// so the kernels stream double2.  Dots: groups of G basis vectors against one
// w, each thread keeping 2 double2 of every vector in flight; per-block
// partial sums in a fixed order (per-thread strided order, warp shuffle tree,
// warps in order), then one warp per sum (k_gs_final), so results are
// deterministic.  Updates w_out = w_in - c_0 v_0 - c_1 v_1 ... apply the terms
// in order i (the oracle's per-entry order), G vectors per pass.
constexpr int kDotBlock = 256;
constexpr int kLinMax = 32;
constexpr int kGroup = 8;
struct GsArgs {
    const double2* v[kGroup];
    double c[kGroup];
};

template <int G, bool SELF>
__global__ void __launch_bounds__(kDotBlock) k_dots(GsArgs A, const double2* __restrict__ w, int64_t N2,
                                                    double* __restrict__ part) {
    constexpr int NS = SELF ? 1 : G;
    __shared__ double red[NS][kDotBlock / 32];
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    const int64_t span = (int64_t)gridDim.x * kDotBlock * 2;
    for (int64_t q0 = (int64_t)blockIdx.x * kDotBlock * 2 + threadIdx.x; q0 < N2; q0 += span) {
        const int64_t q1 = q0 + kDotBlock;
        const bool h1 = q1 < N2;
        const double2 w0 = w[q0];
        const double2 w1 = h1 ? w[q1] : make_double2(0.0, 0.0);
        if (SELF) {
            acc[0] = acc[0] + w0.x * w0.x;
            acc[0] = acc[0] + w0.y * w0.y;
            acc[0] = acc[0] + w1.x * w1.x;
            acc[0] = acc[0] + w1.y * w1.y;
        } else {
            double2 x0[G], x1[G];
#pragma unroll
            for (int i = 0; i < G; ++i) {
                x0[i] = A.v[i][q0];
                x1[i] = h1 ? A.v[i][q1] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int i = 0; i < G; ++i) {
                acc[i] = acc[i] + x0[i].x * w0.x;
                acc[i] = acc[i] + x0[i].y * w0.y;
                acc[i] = acc[i] + x1[i].x * w1.x;
                acc[i] = acc[i] + x1[i].y * w1.y;
            }
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        double t = acc[i];
        for (int off = 16; off > 0; off >>= 1) t = t + __shfl_down_sync(0xffffffffu, t, off);
        if (lane == 0) red[i][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x < NS) {
        double t = 0.0;
        for (int wi = 0; wi < kDotBlock / 32; ++wi) t = t + red[threadIdx.x][wi];
        part[threadIdx.x * gridDim.x + blockIdx.x] = t;
    }
}

// out[i] (+)= sum over blocks of part[i][.]: one warp per sum, lanes take blocks
// lane, lane + 32, ... in order, then a fixed shuffle tree
__global__ void k_gs_final(const double* __restrict__ part, int nblocks, double* __restrict__ out) {
    const int i = blockIdx.x, lane = threadIdx.x;
    double t = 0.0;
    for (int b = lane; b < nblocks; b += 32) t = t + part[i * nblocks + b];
    for (int off = 16; off > 0; off >>= 1) t = t + __shfl_down_sync(0xffffffffu, t, off);
    if (lane == 0) out[i] = t;
}

// w_out = w_in -/+ sum_{i < G} c_i v_i (ADD with w_in == nullptr: 0 + ...)
template <int G, bool ADD>
__global__ void __launch_bounds__(kDotBlock) k_upd(GsArgs A, const double2* win, double2* wout, int64_t N2) {
    const int64_t stride = (int64_t)gridDim.x * kDotBlock;
    for (int64_t q = (int64_t)blockIdx.x * kDotBlock + threadIdx.x; q < N2; q += stride) {
        double2 x[G];
#pragma unroll
        for (int i = 0; i < G; ++i) x[i] = A.v[i][q];
        double2 t = win ? win[q] : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < G; ++i) {
            if (ADD) {
                t.x = t.x + A.c[i] * x[i].x;
                t.y = t.y + A.c[i] * x[i].y;
            } else {
                t.x = t.x - A.c[i] * x[i].x;
                t.y = t.y - A.c[i] * x[i].y;
            }
        }
        wout[q] = t;
    }
}

// y = x / s for library vectors (double2; shared-reciprocal IEEE division,
// exact '/' redo where the fast path is not valid)
__global__ void __launch_bounds__(kDotBlock) k_scale2(const double2* __restrict__ x, double s, double2* __restrict__ y,
                                                      int64_t N2) {
    const int64_t stride = (int64_t)gridDim.x * kDotBlock;
    const double ys = div_recip(s);
    for (int64_t q = (int64_t)blockIdx.x * kDotBlock + threadIdx.x; q < N2; q += stride) {
        const double2 a = x[q];
        bool slow = false;
        double2 r;
        r.x = div_fast_z(a.x, s, ys, slow);
        r.y = div_fast_z(a.y, s, ys, slow);
        if (slow) {
            r.x = a.x / s;
            r.y = a.y / s;
        }
        y[q] = r;
    }
}

// 1: y = x - b   2: y = y + x   (scalar: y may be a caller's unaligned vector)
template <int OP>
__global__ void k_vec(const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ y, int64_t N) {
    const int64_t stride = (int64_t)gridDim.x * kDotBlock;
    for (int64_t q = (int64_t)blockIdx.x * kDotBlock + threadIdx.x; q < N; q += stride) {
        if (OP == 1) y[q] = x[q] - b[q];
        if (OP == 2) y[q] = y[q] + x[q];
    }
}

unsigned flat_grid(const Hierarchy& H) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H.device);
    return (unsigned)(4 * sms);
}

}  // namespace

void mixed_free(MixedSystem* M) {
    if (!M) return;
    cudaFree(M->eca); cudaFree(M->ecb); cudaFree(M->esa); cudaFree(M->ee); cudaFree(M->eg);
    cudaFree(M->ce); cudaFree(M->cs); cudaFree(M->IL); cudaFree(M->g); cudaFree(M->part); cudaFree(M->dots);
    cudaFree(M->V); cudaFree(M->w); cudaFree(M->z); cudaFree(M->t);
    if (M->dots_host) cudaFreeHost(M->dots_host);
    delete M;
}

// Host setup of the edge table (reading R16), the RT0 mass rows (reading
// R17) and cell signs; the lumped inverse is formed on the device.
std::string mixed_setup(const Hierarchy& H) {
    if (H.mix) return "";
    const DevLevel& L = H.lev[H.fine_ref];
    if (L.dist.on || H.nranks > 1) return "mixed system: single-GPU hierarchies only";
    std::vector<HostLevel> host = build_icosahedral_levels(H.fine_ref);
    const HostLevel& HL = host[H.fine_ref];
    const int64_t n = HL.n, ld = L.ld, nz = H.nz;
    MixedSystem* M = new MixedSystem();
    M->ne = 3 * n / 2;
    M->ldh = (M->ne + 31) & ~int64_t(31);
    M->off_z = nz * M->ldh;
    M->off_p = M->off_z + (nz - 1) * ld;
    M->ntot = M->off_p + nz * ld;
    M->omega = std::sqrt(H.w2);
    const int64_t ldh = M->ldh;
    std::vector<int32_t> eca(ldh, 0), ecb(ldh, 0), esa(ldh, 0), ee(6 * ldh, 0), ce(3 * ld, 0);
    std::vector<double> eg(6 * ldh, 0.0), cs(3 * ld, 0.0);
    std::vector<int32_t> esb(ldh, 0);
    int64_t ne = 0;
    for (int64_t c = 0; c < n; ++c)
        for (int j = 0; j < 3; ++j) {
            const int32_t o = HL.nbr[3 * c + j];
            cs[j * ld + c] = (c < o) ? 1.0 : -1.0;
            if (c < o) {
                int jo = 0;
                while (HL.nbr[3 * o + jo] != (int32_t)c) ++jo;
                eca[ne] = (int32_t)c;
                ecb[ne] = o;
                esa[ne] = j;
                esb[ne] = jo;
                ce[j * ld + c] = (int32_t)ne;
                ce[jo * ld + o] = (int32_t)ne;
                ++ne;
            }
        }
    // Gram matrix of the outward flux-normalised RT0 functions of a cell:
    // G_jl = ((s_0 + s_1) + s_2) / (12 area), s_q = (m_q - P_{j+2}).(m_q - P_{l+2}),
    // m_q = 0.5 (P_q + P_{q+1}) (edge-midpoint rule, exact for quadratics)
    auto gram = [&](int64_t c, double G[3][3]) {
        const double* Pv[3] = {&HL.vtx[(3 * c + 0) * 3], &HL.vtx[(3 * c + 1) * 3], &HL.vtx[(3 * c + 2) * 3]};
        double m[3][3];
        for (int q = 0; q < 3; ++q)
            for (int d = 0; d < 3; ++d) m[q][d] = 0.5 * (Pv[q][d] + Pv[(q + 1) % 3][d]);
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) {
                const double* A = Pv[(j + 2) % 3];
                const double* B = Pv[(l + 2) % 3];
                double s[3];
                for (int q = 0; q < 3; ++q) {
                    const double ax = m[q][0] - A[0], ay = m[q][1] - A[1], az = m[q][2] - A[2];
                    const double bx = m[q][0] - B[0], by = m[q][1] - B[1], bz = m[q][2] - B[2];
                    s[q] = (ax * bx + ay * by) + az * bz;
                }
                G[j][l] = ((s[0] + s[1]) + s[2]) / (12.0 * HL.area[c]);
            }
    };
    for (int64_t e = 0; e < ne; ++e)
        for (int side = 0; side < 2; ++side) {
            const int64_t c = side ? ecb[e] : eca[e];
            const int j = side ? esb[e] : esa[e];
            double G[3][3];
            gram(c, G);
            for (int l = 0; l < 3; ++l) {
                eg[(3 * side + l) * ldh + e] = (cs[j * ld + c] * cs[l * ld + c]) * G[j][l];
                ee[(3 * side + l) * ldh + e] = ce[l * ld + c];
            }
        }
    auto up = [&](auto** dst, const auto& src) -> bool {
        using T = typename std::decay_t<decltype(src)>::value_type;
        if (cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * src.size()) != cudaSuccess) return false;
        return cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    };
    bool ok = up(&M->eca, eca) && up(&M->ecb, ecb) && up(&M->esa, esa) && up(&M->ee, ee) && up(&M->eg, eg) &&
              up(&M->ce, ce) && up(&M->cs, cs);
    ok = ok && cudaMalloc(&M->IL, sizeof(double) * M->off_p) == cudaSuccess &&
         cudaMemset(M->IL, 0, sizeof(double) * M->off_p) == cudaSuccess;
    ok = ok && cudaMalloc(&M->g, sizeof(double) * nz * ld) == cudaSuccess &&
         cudaMemset(M->g, 0, sizeof(double) * nz * ld) == cudaSuccess;
    M->nblocks = (int)flat_grid(H);
    ok = ok && cudaMalloc(&M->part, sizeof(double) * kLinMax * M->nblocks) == cudaSuccess;
    ok = ok && cudaMalloc(&M->dots, sizeof(double) * 64) == cudaSuccess;
    ok = ok && cudaHostAlloc(&M->dots_host, sizeof(double) * 64, cudaHostAllocDefault) == cudaSuccess;
    if (!ok) {
        mixed_free(M);
        return "mixed system: device allocation failed";
    }
    H.mix = M;
    const MixView V = view(H);
    const int64_t nt = M->ne > n ? M->ne : n;
    k_mixed_il<<<nblk(nt), kMixBlock>>>(V, L.geom, M->esa, M->IL);
    ++H.launches;
    if (cudaDeviceSynchronize() != cudaSuccess) return "mixed system: setup kernel failed";
    return "";
}

void launch_mixed_apply(const Hierarchy& H, const double* x, double* y, cudaStream_t s) {
    const MixView V = view(H);
    ProfScope ps(H, kKMixed, H.fine_ref, s);
    k_mixed_apply_h<<<nblk(V.ne), kMixBlock, 0, s>>>(V, x, y);
    k_mixed_apply_zp<<<nblk(V.n), kMixBlock, 0, s>>>(V, x, y);
    H.launches += 2;
}

// x = M^-1 f: Eq. 6 with the lumped mass and one V-cycle (p), or a copy (p == nullptr)
void mixed_precond(const Hierarchy& H, const hmg_mg_params* p, const double* f, double* x, cudaStream_t s) {
    const MixedSystem& M = *H.mix;
    if (!p) {
        cudaMemcpyAsync(x, f, sizeof(double) * M.ntot, cudaMemcpyDeviceToDevice, s);
        return;
    }
    const MixView V = view(H);
    {
        ProfScope ps(H, kKMixed, H.fine_ref, s);
        k_mixed_pre_p<<<nblk(V.n), kMixBlock, 0, s>>>(V, f, M.g);
        ++H.launches;
    }
    vcycle_fine(H, *p, M.g, x + M.off_p, s);
    ProfScope ps(H, kKMixed, H.fine_ref, s);
    k_mixed_pre_u<<<nblk(V.ne + V.n), kMixBlock, 0, s>>>(V, f, x);
    ++H.launches;
}

// dot = 1: M.dots[i] = <v_i, w> for i < nv; dot = 2: M.dots[0] = <w, w>.
void mixed_dots(const Hierarchy& H, const double* w, const double* const* v, int nv, int dot, cudaStream_t s) {
    const MixedSystem& M = *H.mix;
    ProfScope ps(H, kKMixed, H.fine_ref, s);
    const unsigned g = (unsigned)M.nblocks;
    const int64_t N2 = M.ntot / 2;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    if (dot == 2) {
        k_dots<1, true><<<g, kDotBlock, 0, s>>>(GsArgs{}, w2, N2, M.part);
        k_gs_final<<<1, 32, 0, s>>>(M.part, M.nblocks, M.dots);
        H.launches += 2;
        return;
    }
    // groups of at most 4 vectors (measured: 8 per pass streams at 3.6 TB/s, 4 at 5.2)
    for (int i0 = 0; i0 < nv;) {
        const int left = nv - i0;
        const int G = left >= 4 ? 4 : left >= 2 ? 2 : 1;
        GsArgs A{};
        for (int i = 0; i < G; ++i) A.v[i] = reinterpret_cast<const double2*>(v[i0 + i]);
        if (G == 4) k_dots<4, false><<<g, kDotBlock, 0, s>>>(A, w2, N2, M.part);
        if (G == 2) k_dots<2, false><<<g, kDotBlock, 0, s>>>(A, w2, N2, M.part);
        if (G == 1) k_dots<1, false><<<g, kDotBlock, 0, s>>>(A, w2, N2, M.part);
        k_gs_final<<<G, 32, 0, s>>>(M.part, M.nblocks, M.dots + i0);
        H.launches += 2;
        i0 += G;
    }
}

// w_out = w_in - sum_i c_i v_i (add: w_out = 0 + sum_i c_i v_i; w_in unused),
// terms in order i; w_in == w_out allowed
void mixed_update(const Hierarchy& H, const double* win, double* wout, const double* const* v, const double* c, int nv,
                  bool add, cudaStream_t s) {
    const MixedSystem& M = *H.mix;
    ProfScope ps(H, kKMixed, H.fine_ref, s);
    const unsigned g = (unsigned)M.nblocks;
    const int64_t N2 = M.ntot / 2;
    const double2* in = add ? nullptr : reinterpret_cast<const double2*>(win);
    double2* out = reinterpret_cast<double2*>(wout);
    for (int i0 = 0; i0 < nv;) {
        const int left = nv - i0;
        const int G = left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
        GsArgs A{};
        for (int i = 0; i < G; ++i) {
            A.v[i] = reinterpret_cast<const double2*>(v[i0 + i]);
            A.c[i] = c[i0 + i];
        }
#define HMG_UPD(GG)                                                                 \
    if (G == GG) {                                                                  \
        if (add) k_upd<GG, true><<<g, kDotBlock, 0, s>>>(A, in, out, N2);           \
        else k_upd<GG, false><<<g, kDotBlock, 0, s>>>(A, in, out, N2);              \
    }
        HMG_UPD(8) HMG_UPD(4) HMG_UPD(2) HMG_UPD(1)
#undef HMG_UPD
        ++H.launches;
        in = out;                 // later groups continue from the partial result
        i0 += G;
    }
}

void mixed_vec(const Hierarchy& H, int op, const double* x, const double* b, double sc, double* y, cudaStream_t s) {
    const MixedSystem& M = *H.mix;
    ProfScope ps(H, kKMixed, H.fine_ref, s);
    const unsigned g = (unsigned)M.nblocks;
    if (op == 0)
        k_scale2<<<g, kDotBlock, 0, s>>>(reinterpret_cast<const double2*>(x), sc, reinterpret_cast<double2*>(y),
                                         M.ntot / 2);
    if (op == 1) k_vec<1><<<g, kDotBlock, 0, s>>>(x, b, y, M.ntot);
    if (op == 2) k_vec<2><<<g, kDotBlock, 0, s>>>(x, b, y, M.ntot);
    ++H.launches;
}

int mixed_lin_max() { return kLinMax; }

}  // namespace hmg
