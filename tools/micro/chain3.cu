// z / back-substitution chains of one warp from shared memory: batched (as
// small_tile.cuh) vs batched with the next batch's operands prefetched.
#include <cstdio>
#include <cstdint>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;
constexpr int W = 32;
#define LOADZ(K0, R, U, D, Y)                                              \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
        const int q = ((K0) + i) * W + t;                                  \
        R[i] = Z[q];                                                       \
        U[i] = A1[((K0) + i > 0) ? q - W : q];                             \
        D[i] = A2[q];                                                      \
        Y[i] = A3[q];                                                      \
    }
#define CHAINZ(K0, R, U, D, Y)                                             \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
        const double num = ((K0) + i == 0) ? R[i] : R[i] - U[i] * zprev;   \
        R[i] = div_fast_z(num, D[i], Y[i], slow);                          \
        zprev = R[i];                                                      \
    }                                                                      \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) Z[((K0) + i) * W + t] = R[i];
template <int MODE>
__global__ void kz(long long* cyc, double* out, int nz, int reps) {
    extern __shared__ double smz[];
    double *A1 = smz, *A2 = smz + 64 * W, *A3 = smz + 128 * W, *Z = smz + 192 * W;
    const int t = threadIdx.x;
    for (int k = 0; k < 64; ++k) { A1[k * W + t] = -0.3; A2[k * W + t] = 2.0 + k; A3[k * W + t] = 1.0 / (2.0 + k); Z[k * W + t] = 0.5 * t + k + 1; }
    __syncwarp();
    bool slow = false;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double zprev = 0.0;
        if (MODE == 0) {
            for (int k0 = 0; k0 < nz; k0 += 8) {
                double rr[8], um[8], dd[8], yy[8];
                LOADZ(k0, rr, um, dd, yy)
                CHAINZ(k0, rr, um, dd, yy)
            }
        } else {
            double ar[8], au[8], ad[8], ay[8], br[8], bu[8], bd[8], by[8];
            LOADZ(0, ar, au, ad, ay)
            for (int k0 = 0; k0 < nz; k0 += 16) {
                if (k0 + 8 < nz) { LOADZ(k0 + 8, br, bu, bd, by) }
                CHAINZ(k0, ar, au, ad, ay)
                if (k0 + 8 >= nz) break;
                if (k0 + 16 < nz) { LOADZ(k0 + 16, ar, au, ad, ay) }
                CHAINZ(k0 + 8, br, bu, bd, by)
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[t] = Z[t] + slow;
    if (t == 0) cyc[MODE] = t1 - t0;
}
#define LOADB(K1, ZZ, GG, UO)                                              \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
        const int q = ((K1) - i) * W + t;                                  \
        ZZ[i] = Z[q];                                                      \
        GG[i] = G[q];                                                      \
        UO[i] = U[q];                                                      \
    }
#define CHAINB(K1, ZZ, GG, UO)                                             \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
        dl = ((K1) - i >= nz - 1) ? ZZ[i] : ZZ[i] - GG[i] * dl;            \
        UO[i] = UO[i] + 0.8 * dl;                                          \
    }                                                                      \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) U[((K1) - i) * W + t] = UO[i];
template <int MODE>
__global__ void kb(long long* cyc, double* out, int nz, int reps) {
    __shared__ double Z[64 * W], G[64 * W], U[64 * W];
    const int t = threadIdx.x;
    for (int k = 0; k < 64; ++k) { Z[k * W + t] = 0.5 * t + k; G[k * W + t] = 0.01 * k; U[k * W + t] = 1.0; }
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double dl = 0.0;
        if (MODE == 0) {
            for (int k1 = nz - 1; k1 >= 0; k1 -= 8) {
                double zz[8], gg[8], uo[8];
                LOADB(k1, zz, gg, uo)
                CHAINB(k1, zz, gg, uo)
            }
        } else {
            double az[8], ag[8], au[8], bz[8], bg[8], bu[8];
            LOADB(nz - 1, az, ag, au)
            for (int k1 = nz - 1; k1 >= 0; k1 -= 16) {
                if (k1 - 8 >= 0) { LOADB(k1 - 8, bz, bg, bu) }
                CHAINB(k1, az, ag, au)
                if (k1 - 8 < 0) break;
                if (k1 - 16 >= 0) { LOADB(k1 - 16, az, ag, au) }
                CHAINB(k1 - 8, bz, bg, bu)
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[t] = U[t];
    if (t == 0) cyc[2 + MODE] = t1 - t0;
}
int main() {
    long long* c; double* o; cudaMallocManaged(&c, 128); cudaMallocManaged(&o, 32 * 8);
    int nz = 64, reps = 200;
    for (int i = 0; i < 2; ++i) {
        cudaFuncSetAttribute(kz<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000); cudaFuncSetAttribute(kz<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
        kz<0><<<1, 32, 65536>>>(c, o, nz, reps); kz<1><<<1, 32, 65536>>>(c, o, nz, reps);
        kb<0><<<1, 32>>>(c, o, nz, reps); kb<1><<<1, 32>>>(c, o, nz, reps);
        cudaDeviceSynchronize();
    }
    double L = nz * (double)reps;
    printf("z chain cycles/layer: batched %.1f  prefetched %.1f ; back: batched %.1f  prefetched %.1f\n", c[0] / L, c[1] / L, c[2] / L, c[3] / L);
}
