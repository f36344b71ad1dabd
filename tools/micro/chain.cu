// Microbenchmark of the Thomas z-chain per layer for one warp, operands in smem.
#include <cstdio>
#include <cstdint>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;
template <int MODE>
__global__ void k(long long* cyc, double* out, int nz, int reps) {
    __shared__ double A[4][64][16];
    __shared__ double Z[64][16];
    const int t = threadIdx.x;
    for (int k = 0; k < 64; ++k) { A[0][k][t & 15] = 1.0 + 0.01 * k; A[1][k][t & 15] = -0.3; A[2][k][t & 15] = 2.0 + k; A[3][k][t & 15] = 1.0 / (2.0 + k); Z[k][t & 15] = 0.5 * t; }
    __syncwarp();
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double zprev = 0.0;
        bool slow = false;
#pragma unroll 8
        for (int k = 0; k < nz; ++k) {
            const double rr = Z[k][t & 15];
            const double num = (k == 0) ? rr : rr - A[1][k][t & 15] * zprev;
            double zk;
            if (MODE == 0) zk = div_fast(num, A[2][k][t & 15], A[3][k][t & 15], slow);
            else if (MODE == 1) zk = num * A[3][k][t & 15];
            else if (MODE == 2) zk = num / A[2][k][t & 15];
            Z[k][t & 15] = zk;
            zprev = zk;
        }
        acc += zprev + slow;
    }
    if (MODE == 3) {   // batched: all operands of 8 layers loaded first
        for (int r = 0; r < reps; ++r) {
            double zprev = 0.0;
            bool slow = false;
            for (int k0 = 0; k0 < nz; k0 += 8) {
                double rr[8], a1[8], dd[8], yy[8], zz[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) { rr[i] = Z[k0 + i][t & 15]; a1[i] = A[1][k0 + i][t & 15]; dd[i] = A[2][k0 + i][t & 15]; yy[i] = A[3][k0 + i][t & 15]; }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const double num = (k0 + i == 0) ? rr[i] : rr[i] - a1[i] * zprev;
                    zz[i] = div_fast(num, dd[i], yy[i], slow);
                    zprev = zz[i];
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) Z[k0 + i][t & 15] = zz[i];
            }
            acc += zprev + slow;
        }
    }
    long long t1 = clock64();
    out[t] = acc;
    if (t == 0) cyc[MODE] = t1 - t0;
}
int main() {
    long long* c; double* o; cudaMallocManaged(&c, 128); cudaMallocManaged(&o, 32 * 8);
    int nz = 64, reps = 100;
    for (int i = 0; i < 2; ++i) {
        k<0><<<1, 32>>>(c, o, nz, reps); k<1><<<1, 32>>>(c, o, nz, reps); k<2><<<1, 32>>>(c, o, nz, reps); k<3><<<1, 32>>>(c, o, nz, reps);
        cudaDeviceSynchronize();
    }
    printf("cycles/layer: div_fast %.1f  mul-only %.1f  '/' %.1f  batched-8 div_fast %.1f\n", c[0] / (double)(nz * reps), c[1] / (double)(nz * reps), c[2] / (double)(nz * reps), c[3] / (double)(nz * reps));
}
