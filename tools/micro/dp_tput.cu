// fp64 FMA throughput per SM (independent chains, many warps) and the cost of div_fast.
#include <cstdio>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;
template <int MODE>
__global__ void k(double* out, int n) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
    const double b = 0.999999, c = 1e-9, y = 1.0 / b;
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = __fma_rn(a[i], b, c);
            if (MODE == 1) { bool s = false; a[i] = div_fast(a[i], b, y, s); if (s) a[i] = 0.0; }
        }
    }
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    double* o;
    cudaMalloc(&o, 148 * 8 * 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int n = 2000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, n); else k<1><<<148 * 8, 256>>>(o, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = 148.0 * 8 * 256 * n * 8;
        printf("%s: %.2f G ops/s = %.1f per SM per clk at 1.965 GHz\n", mode ? "div_fast" : "dfma", ops / ms / 1e6,
               ops / (ms * 1e-3) / 148 / 1.965e9);
    }
}
