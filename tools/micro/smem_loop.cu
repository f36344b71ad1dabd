// Microbenchmark: one warp streaming over [64][32] fp64 shared-memory planes.
#include <cstdio>
__global__ void k(long long* cyc, double* out, int nz) {
    extern __shared__ double sm[];
    double* a = sm; double* b2 = sm + 64 * 32; double* c = sm + 2 * 64 * 32;
    const int j = threadIdx.x;
    for (int k = 0; k < 64; ++k) { a[k * 32 + j] = k + j; b2[k * 32 + j] = 0.5 * k; c[k * 32 + j] = 0; }
    __syncwarp();
    long long t0 = clock64();
    for (int k0 = 0; k0 < nz; k0 += 4) {
        double r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = a[(k0 + i) * 32 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i) c[(k0 + i) * 32 + j] = r[i];
    }
    long long t1 = clock64();
    for (int k = 0; k < nz; ++k) c[k * 32 + j] = a[k * 32 + j] * b2[k * 32 + j];
    long long t2 = clock64();
    double acc = 0;
#pragma unroll 8
    for (int k = 0; k < nz; ++k) acc = acc + a[k * 32 + j];
    long long t3 = clock64();
    out[j] = acc + c[j];
    if (j == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    long long* c; double* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 256);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int smem : {3 * 64 * 32 * 8, 200 * 1024}) {
        for (int r = 0; r < 2; ++r) { k<<<1, 32, smem>>>(c, o, 64); cudaDeviceSynchronize(); }
        printf("smem %d: copy batched %.1f  mul-copy %.1f  reduce %.1f cycles/layer  %s\n", smem, c[0] / 64.0, c[1] / 64.0, c[2] / 64.0, cudaGetErrorString(cudaGetLastError()));
    }
}
