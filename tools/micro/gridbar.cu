// Microbenchmarks for the coarse-level design: fp64 dependent-op latency and
// the cost of a software grid barrier in a cooperative launch.
#include <cooperative_groups.h>
#include <cuda/atomic>
#include <cstdio>
#include <cstdint>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;

template <int OP>
__global__ void k_lat(long long* cyc, double* out, int n) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.999999, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) a = __dadd_rn(a, c);
        if (OP == 1) a = __dmul_rn(a, b);
        if (OP == 2) a = __fma_rn(a, b, c);
        if (OP == 3) { bool s = false; a = div_fast(a, b, 1.0 / b, s); }
        if (OP == 4) a = a / b;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[OP] = t1 - t0;
}

struct Bar {
    unsigned count;
    unsigned gen;
};

__device__ __forceinline__ void grid_bar(Bar* B, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(B->count), gen(B->gen);
        const unsigned g = gen.load(cuda::memory_order_relaxed);
        if (cnt.fetch_add(1, cuda::memory_order_acq_rel) == nb - 1) {
            cnt.store(0, cuda::memory_order_relaxed);
            gen.fetch_add(1, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) {}
        }
    }
    __syncthreads();
}

__global__ void k_bar(Bar* B, int iters, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) grid_bar(B, gridDim.x);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_cg(int iters, long long* cyc) {
    auto g = cooperative_groups::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_empty() {}

int main() {
    long long* c;
    double* o;
    cudaMallocManaged(&c, 1024);
    cudaMallocManaged(&o, 1024 * 8);
    const int n = 4096;
    for (int r = 0; r < 2; ++r) {
        k_lat<0><<<1, 32>>>(c, o, n); k_lat<1><<<1, 32>>>(c, o, n); k_lat<2><<<1, 32>>>(c, o, n);
        k_lat<3><<<1, 32>>>(c, o, n); k_lat<4><<<1, 32>>>(c, o, n);
        cudaDeviceSynchronize();
    }
    printf("cycles per dependent op: dadd %.1f dmul %.1f dfma %.1f div_fast %.1f div %.1f\n", c[0] / (double)n,
           c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
    Bar* B;
    cudaMalloc(&B, sizeof(Bar));
    cudaMemset(B, 0, sizeof(Bar));
    int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int nb : {1, 10, 40, 80, 148}) {
        for (int th : {32, 128}) {
            void* args[] = {&B, &iters, &c};
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                cudaLaunchCooperativeKernel((void*)k_bar, nb, th, args, 0, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            void* args2[] = {&iters, &c};
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)k_cg, nb, th, args2, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms2;
            cudaEventElapsedTime(&ms2, e0, e1);
            printf("grid barrier nb=%3d th=%3d: own %.3f us  cg %.3f us  (err %s)\n", nb, th, ms * 1e3 / iters,
                   ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // dependent-launch gap: empty kernels back to back
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(e0);
        for (int i = 0; i < 1000; ++i) k_empty<<<148, 128>>>();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("back-to-back empty kernel: %.3f us\n", ms);
    // same inside a CUDA graph
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 1000; ++i) k_empty<<<148, 128, 0, s>>>();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of empty kernels: %.3f us each\n", ms);
    return 0;
}
