// Microbenchmark: the ceiling of the fine sweep's data movement WITHOUT its
// arithmetic.  Persistent CTAs (tile = blockIdx.x + i * grid, as k_sweep_st),
// one producer warp streaming per G layers: the D/U band rows (one 3-D box),
// G rows of b and G + 1 rows of u through an S-stage mbarrier ring; 4 consumer
// warps, thread = column, writing one output double per layer.  Variants:
//   layout 0: layer-major [nz][ld] arrays (the library's layout)
//   layout 1: tile-blocked [ntiles][nz][128] (each tile's rows contiguous)
//   wmode 0: no output, 1: st.global per layer, 2: TMA store of the stage's
//            G output rows from shared memory (bulk tensor s2g)
//   cps: CTAs per SM (ring budget 220 KB / cps)
// Prints us and GB/s over 40 B/dof (D, U, b, u read, out written).
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../../paper_1605_00492_b200/csrc/sm100_ptx.cuh"
using namespace hmg;

struct Maps { CUtensorMap bands, b, u, out; };

__device__ __forceinline__ void tma4(void* dst, const void* m, int x, int y, int z, int w, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3, %4, %5}], [%6], %7;" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(ptx::smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_st2(const void* m, int x, int y, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(ptx::smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_st3(const void* m, int x, int y, int z, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(ptx::smem_u32(src)) : "memory");
}

template <int G, int LAYOUT, int WMODE>
__global__ void __launch_bounds__(160) k(const __grid_constant__ Maps maps, double* out, int nz, int64_t ld, int ntiles,
                                         int S) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = (uint64_t*)sm;
    uint64_t* empty = full + S;
    double* st = (double*)(sm + 1024);
    constexpr int STAGE = (2 * G + G + (G + 1) + (WMODE == 2 ? G : 0)) * 128;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 4); }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int ng = nz / G;
    if (warp == 4) {
        const uint64_t pf = ptx::policy_evict_first(), pl = ptx::policy_evict_last();
        int s = 0; unsigned ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
            for (int g = 0; g < ng; ++g) {
                ptx::mbar_wait(&empty[s], ph ^ 1);
                if (lane == 0) {
                    double* d = st + (size_t)s * STAGE;
                    ptx::mbar_arrive_expect_tx(&full[s], (2 * G + G + G + 1) * 128 * 8);
                    if (LAYOUT == 0) {
                        ptx::tma_load_3d_hint(d, &maps.bands, t * 128, g * G, 0, &full[s], pf);
                        ptx::tma_load_2d_hint(d + 2 * G * 128, &maps.b, t * 128, g * G, &full[s], pf);
                        ptx::tma_load_2d_hint(d + 3 * G * 128, &maps.u, t * 128, g * G, &full[s], pl);
                    } else {
                        tma4(d, &maps.bands, 0, g * G, 0, t, &full[s], pf);
                        ptx::tma_load_3d_hint(d + 2 * G * 128, &maps.b, 0, g * G, t, &full[s], pf);
                        ptx::tma_load_3d_hint(d + 3 * G * 128, &maps.u, 0, g * G, t, &full[s], pl);
                    }
                }
                __syncwarp();
                if (++s == S) { s = 0; ph ^= 1; }
            }
    } else {
        const int j = threadIdx.x;
        int s = 0; unsigned ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
            for (int g = 0; g < ng; ++g) {
                ptx::mbar_wait(&full[s], ph);
                double* d = st + (size_t)s * STAGE;
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const int k = g * G + kk;
                    const double v = d[kk * 128 + j] * d[3 * G * 128 + (kk + 1) * 128 + j] +
                                     d[G * 128 + kk * 128 + j] * d[2 * G * 128 + kk * 128 + j];
                    if (WMODE == 1) {
                        if (LAYOUT == 0) out[(int64_t)k * ld + (int64_t)t * 128 + j] = v;
                        else out[((int64_t)t * nz + k) * 128 + j] = v;
                    } else if (WMODE == 2) {
                        d[(2 * G + G + G + 1) * 128 + kk * 128 + j] = v;
                    } else if (v == 1234.5) {
                        out[0] = v;
                    }
                }
                if (WMODE == 4 && g == ng - 1) {      // a back-substitution-long pause after each tile
                    const long long t0 = clock64();
                    while (clock64() - t0 < (long long)nz * 140) {}
                }
                if (WMODE == 4) {
                    const int k = g * G;
                    if (LAYOUT == 0) out[(int64_t)k * ld + (int64_t)t * 128 + j] = d[j];
                    if (LAYOUT == 0) out[(int64_t)(k + 1) * ld + (int64_t)t * 128 + j] = d[128 + j];
                }
                if (WMODE == 3 && g == ng - 1) {      // the tile's outputs in one burst after its last stage
                    const double v = d[j];
                    for (int k = 0; k < nz; ++k) {
                        if (LAYOUT == 0) out[(int64_t)k * ld + (int64_t)t * 128 + j] = v + k;
                        else out[((int64_t)t * nz + k) * 128 + j] = v + k;
                    }
                }
                if (WMODE == 2) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (threadIdx.x == 0) {
                        if (LAYOUT == 0) tma_st2(&maps.out, t * 128, g * G, d + (2 * G + G + G + 1) * 128);
                        else tma_st3(&maps.out, 0, g * G, t, d + (2 * G + G + G + 1) * 128);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn enc;
static CUtensorMap mk(void* base, int rank, std::vector<cuuint64_t> dims, std::vector<cuuint64_t> strides_b,
                      std::vector<cuuint32_t> box) {
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base, dims.data(), strides_b.data(), box.data(), es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

template <int G, int LAYOUT, int WMODE>
void run(double* D, double* B, double* U, double* O, int nz, int64_t ld, int cps, int sms) {
    const int ntiles = (int)(ld / 128);
    Maps m;
    memset(&m, 0, sizeof(m));
    const cuuint64_t E = 8;
    if (LAYOUT == 0) {
        m.bands = mk(D, 3, {(cuuint64_t)ld, (cuuint64_t)nz, 2}, {ld * E, ld * nz * E}, {128, G, 2});
        m.b = mk(B, 2, {(cuuint64_t)ld, (cuuint64_t)nz}, {ld * E}, {128, G});
        m.u = mk(U, 2, {(cuuint64_t)ld, (cuuint64_t)nz}, {ld * E}, {128, G + 1});
        m.out = mk(O, 2, {(cuuint64_t)ld, (cuuint64_t)nz}, {ld * E}, {128, G});
    } else {
        m.bands = mk(D, 4, {128, (cuuint64_t)nz, 2, (cuuint64_t)ntiles}, {128 * E, 128 * nz * E, 2 * 128 * nz * E},
                     {128, G, 2, 1});
        m.b = mk(B, 3, {128, (cuuint64_t)nz, (cuuint64_t)ntiles}, {128 * E, 128 * nz * E}, {128, G, 1});
        m.u = mk(U, 3, {128, (cuuint64_t)nz, (cuuint64_t)ntiles}, {128 * E, 128 * nz * E}, {128, G + 1, 1});
        m.out = mk(O, 3, {128, (cuuint64_t)nz, (cuuint64_t)ntiles}, {128 * E, 128 * nz * E}, {128, G, 1});
    }
    constexpr int STAGE = (2 * G + G + (G + 1) + (WMODE == 2 ? G : 0)) * 128;
    const size_t budget = (cps == 1 ? 220 : cps == 2 ? 110 : 72) * 1024;
    int S = (int)((budget - 1024) / (STAGE * 8));
    if (S > 32) S = 32;
    const size_t smem = 1024 + (size_t)S * STAGE * 8;
    auto kern = k<G, LAYOUT, WMODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int cap = cps * sms, rounds = (ntiles + cap - 1) / cap, grid = (ntiles + rounds - 1) / rounds;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) kern<<<grid, 160, smem>>>(m, O, nz, ld, ntiles, S);
    cudaEventRecord(e0);
    const int it = 20;
    for (int w = 0; w < it; ++w) kern<<<grid, 160, smem>>>(m, O, nz, ld, ntiles, S);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / it, bytes = 40.0 * ld * nz;
    printf("G %d layout %d wmode %d cps %d S %2d grid %4d: %7.1f us %6.0f GB/s  %s\n", G, LAYOUT, WMODE, cps, S, grid,
           us, bytes / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = (EncodeFn)p;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nz = 64;
    const int64_t ld = 327680;
    double *D, *B, *U, *O;
    cudaMalloc(&D, ld * nz * 16);
    cudaMalloc(&B, ld * nz * 8);
    cudaMalloc(&U, ld * nz * 8);
    cudaMalloc(&O, ld * nz * 8);
    cudaMemset(D, 0, ld * nz * 16);
    cudaMemset(B, 0, ld * nz * 8);
    cudaMemset(U, 0, ld * nz * 8);
    for (int cps : {2}) {
        run<2, 0, 3>(D, B, U, O, nz, ld, cps, sms);
        run<2, 0, 1>(D, B, U, O, nz, ld, cps, sms);
        run<2, 0, 4>(D, B, U, O, nz, ld, cps, sms);
    }
    return 0;
    for (int cps : {1, 2, 3}) {
        run<2, 0, 0>(D, B, U, O, nz, ld, cps, sms);
        run<2, 0, 1>(D, B, U, O, nz, ld, cps, sms);
        run<2, 0, 2>(D, B, U, O, nz, ld, cps, sms);
        run<2, 1, 0>(D, B, U, O, nz, ld, cps, sms);
        run<2, 1, 1>(D, B, U, O, nz, ld, cps, sms);
        run<2, 1, 2>(D, B, U, O, nz, ld, cps, sms);
        run<4, 0, 1>(D, B, U, O, nz, ld, cps, sms);
        run<4, 1, 1>(D, B, U, O, nz, ld, cps, sms);
        run<8, 1, 1>(D, B, U, O, nz, ld, cps, sms);
    }
    return 0;
}
