// Microbenchmark: cost of tcgen05.st (x2) per layer-step and of tcgen05.ld (x16) + wait, one warp.
#include <cstdio>
#include <cstdint>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;
__global__ void k(long long* cyc, double* out, double a, int n) {
    __shared__ uint32_t slot;
    __shared__ double sm[64 * 32];
    const int lane = threadIdx.x;
    if (threadIdx.x < 32) ptx::tmem_alloc(&slot, 256);
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tb = slot;
    double x = a + lane;
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) { x = x * 1.0000001 + 0.5; ptx::tmem_st_f64(tb + 2u * (k & 63), x); }
    ptx::tmem_wait_st();
    long long t1 = clock64();
    for (int k = 0; k < n; ++k) { x = x * 1.0000001 + 0.5; sm[(k & 63) * 32 + lane] = x; }
    __syncwarp();
    long long t2 = clock64();
    double acc = 0;
    for (int k = 0; k < n / 8; ++k) {
        uint32_t r[16];
        ptx::tmem_ld_8f64(tb + 16u * (k & 7), r);
        ptx::tmem_wait_ld();
        for (int i = 0; i < 8; ++i) acc = acc * 0.5 + ptx::f64_from(r[2 * i], r[2 * i + 1]);
    }
    long long t3 = clock64();
    for (int k = 0; k < n; ++k) { x = x * 1.0000001 + 0.5; }
    long long t4 = clock64();
    out[lane] = x + acc;
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
    ptx::tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tb, 256);
}
int main() {
    long long* c; double* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 32 * 8);
    int n = 4096;
    for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(c, o, 1.0, n); cudaDeviceSynchronize(); }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    printf("per step: chain+STTM %.1f  chain+STS %.1f  (LDTM x16+wait+8 dep ops)/8 %.1f  chain only %.1f cycles\n",
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n);
}
