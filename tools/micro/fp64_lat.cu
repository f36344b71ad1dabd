// Microbenchmark: dependent-chain latency of fp64 add/mul/fma and the
// shared-reciprocal division on sm_100a (single thread, clock64).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x = a, y = b;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = __fma_rn(x, y, a);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = x / y;
    long long t4 = clock64();
    float f = (float)a;
    for (int i = 0; i < n; ++i) f = __fadd_rn(f, (float)b);
    long long t5 = clock64();
    out[threadIdx.x] = x + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
    double* o; long long* c; cudaMallocManaged(&o, 32*8); cudaMallocManaged(&c, 64);
    int n = 4096;
    k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); cudaDeviceSynchronize();
    printf("cycles per dependent op: dadd %.1f dmul %.1f dfma %.1f ddiv %.1f fadd %.1f\n",
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
    return 0;
}
