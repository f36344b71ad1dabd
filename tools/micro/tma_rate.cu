// Microbenchmark: per-SM throughput of 2-D TMA tensor loads (box 128 x G fp64) through an
// S-stage mbarrier ring, 1 producer lane + 1 consumer warp that only waits/releases.
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;
struct Maps { CUtensorMap m[8]; };
template <int G>
__global__ void k(const __grid_constant__ Maps maps, int narr, int nz, int S, long long* cyc, int ld) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + S;
    double* st = (double*)(sm + 1024);
    const int stage_d = narr * G * 128;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); } ptx::fence_mbar_init(); }
    __syncthreads();
    const int x = blockIdx.x * 128;
    long long t0 = clock64();
    int ng = nz / G;
    if (warp == 1) {
        int s = 0; unsigned ph = 0;
        for (int g = 0; g < ng; ++g) {
            ptx::mbar_wait(&empty[s], ph ^ 1);
            if (lane == 0) {
                ptx::mbar_arrive_expect_tx(&full[s], narr * G * 128 * 8);
                for (int a = 0; a < narr; ++a) ptx::tma_load_2d(st + s * stage_d + a * G * 128, &maps.m[a], x, g * G, &full[s]);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1; }
        }
    } else {
        int s = 0; unsigned ph = 0; double acc = 0;
        for (int g = 0; g < ng; ++g) {
            ptx::mbar_wait(&full[s], ph);
            acc += st[s * stage_d + lane];
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
        }
        if (acc == 12345.0) cyc[1] = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = clock64() - t0;
}
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    const int ld = 327680, nz = 64, narr = 7;
    double* buf[8]; for (int a = 0; a < 8; ++a) { cudaMalloc(&buf[a], (size_t)ld * nz * 8); cudaMemset(buf[a], 0, (size_t)ld * nz * 8); }
    long long* cyc; cudaMallocManaged(&cyc, 64);
    for (int G : {1, 2, 4, 8}) {
        Maps m; memset(&m, 0, sizeof(m));
        for (int a = 0; a < narr; ++a) {
            cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)nz}; cuuint64_t str[1] = {(cuuint64_t)ld * 8};
            cuuint32_t box[2] = {128, (cuuint32_t)G}; cuuint32_t es[2] = {1, 1};
            enc(&m.m[a], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf[a], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        for (int S : {2, 4, 8}) {
            size_t smem = 1024 + (size_t)S * narr * G * 128 * 8;
            if (smem > 220 * 1024) continue;
            auto kern = G == 1 ? k<1> : G == 2 ? k<2> : G == 4 ? k<4> : k<8>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            for (int grid : {1, 148, 2560}) {
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                kern<<<grid, 64, smem>>>(m, narr, nz, S, cyc, ld);
                cudaEventRecord(e0);
                kern<<<grid, 64, smem>>>(m, narr, nz, S, cyc, ld);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                double bytes = (double)grid * narr * nz * 128 * 8;
                printf("G %d S %d grid %5d: %8.1f us  %7.1f GB/s  (block0 %lld cycles, %.0f B/cycle/CTA)  %s\n", G, S, grid, ms * 1e3, bytes / (ms * 1e-3) / 1e9, cyc[0], narr * nz * 128 * 8.0 / cyc[0], cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
}
