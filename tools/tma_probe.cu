// Streaming probe: how fast can the lower-triangle 64 x 64 tiles of a
// row-major fp64 n x n matrix be pulled through a 4-stage shared-memory ring
// by 148 CTAs (no arithmetic), per load method:
//   0  per-thread 16-byte cp.async (LDGSTS), 512 threads x 4 chunks per tile
//   1  TMA, four 16 x 64 boxes per tile, SWIZZLE_128B, L2 promotion 256B
//   2  TMA, one 64 x 64 box per tile, no swizzle, L2 promotion 256B
//   3  TMA, four 16 x 64 boxes, SWIZZLE_128B, no L2 promotion
//   4  TMA, two 32 x 64 boxes per tile, no swizzle
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -o tools/_build/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define NT 512
#define STAGES 4
#define TILE 4096

typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned par) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.shared::cta.b64 s, [%0];\n\t}\n" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}\n" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_arrive(unsigned long long* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ unsigned long long pol_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c, int r, unsigned long long* bar,
                                      unsigned long long pol) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(sa(dst)), "l"((unsigned long long)m), "r"(sa(bar)),
                 "r"(c), "r"(r), "l"(pol) : "memory");
}

__device__ long long tile_row(long long t) {
    long long I = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    return I;
}

__global__ void __launch_bounds__(NT, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const double* K,
                                                       long long ldk, long long ntt, int mode, double* sink,
                                                       int polmode) {
    extern __shared__ __align__(1024) double smem[];
    double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + STAGES * TILE);
    unsigned long long* empty = full + STAGES;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, mode == 0 ? NT : 1);
            mbar_init(empty + s, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = ntt * blockIdx.x / gridDim.x, t1 = ntt * (blockIdx.x + 1) / gridDim.x;
    const int nt = (int)(t1 - t0);
    const unsigned long long pol = polmode == 0 ? pol_first() : polmode == 1 ? 0x12F0000000000000ull
                                                                             : 0x1000000000000000ull;
    auto produce = [&](int lt) {
        const int stg = lt % STAGES;
        if (lt >= STAGES) mbar_wait(empty + stg, ((lt / STAGES) - 1) & 1);
        const long long t = t0 + lt, I = tile_row(t), J = t - I * (I + 1) / 2;
        double* dst = ring + stg * TILE;
        if (mode == 0) {
            const double* src = K + (I * 64) * ldk + J * 64;
            for (int u = 0; u < 4; ++u) {
                const int row = (tid >> 5) + 16 * u, c2 = (tid & 31) * 2;
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa(dst + row * 64 + c2)),
                             "l"(src + row * ldk + c2), "l"(pol));
            }
            cp_arrive(full + stg);
        } else if (tid == 0) {
            mbar_expect(full + stg, TILE * 8);
            if (mode == 1 || mode == 3)
                for (int b = 0; b < 4; ++b) tma2d(dst + b * 1024, &map, (int)(J * 64 + 16 * b), (int)(I * 64), full + stg, pol);
            else if (mode == 2)
                tma2d(dst, &map, (int)(J * 64), (int)(I * 64), full + stg, pol);
            else
                for (int b = 0; b < 2; ++b) tma2d(dst + b * 2048, &map, (int)(J * 64 + 32 * b), (int)(I * 64), full + stg, pol);
        }
    };
    for (int lt = 0; lt < STAGES - 1 && lt < nt; ++lt) produce(lt);
    double acc = 0.0;
    for (int lt = 0; lt < nt; ++lt) {
        if (lt + STAGES - 1 < nt) {
            if (mode == 0 || tid == 0) produce(lt + STAGES - 1);
        }
        const int stg = lt % STAGES;
        mbar_wait(full + stg, (lt / STAGES) & 1);
        const double* tl = ring + stg * TILE;
        acc += tl[(lane * 64 + warp * 4) % TILE] + tl[(lane * 64 + warp * 4 + 2048 + 1) % TILE];
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stg);
    }
    if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 10000;
    const long long ldk = (n + 31) / 32 * 32;
    double* K;
    cudaMalloc(&K, sizeof(double) * n * ldk);
    cudaMemset(K, 0, sizeof(double) * n * ldk);
    double* sink;
    cudaMalloc(&sink, 8);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    encode_fn enc = (encode_fn)fp;
    const long long nt1 = (n + 63) / 64, ntt = nt1 * (nt1 + 1) / 2;
    const double bytes = (double)ntt * TILE * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t smem = STAGES * TILE * 8 + 2048 + 1024;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode <= 4; ++mode) {
        CUtensorMap map;
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n}, str[1] = {(cuuint64_t)ldk * 8};
        cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
        CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
        CUtensorMapL2promotion pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        if (mode == 2) { box[0] = 64; sw = CU_TENSOR_MAP_SWIZZLE_NONE; }
        if (mode == 3) pr = CU_TENSOR_MAP_L2_PROMOTION_NONE;
        if (mode == 4) { box[0] = 32; sw = CU_TENSOR_MAP_SWIZZLE_NONE; }
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, K, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         sw, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("mode %d encode failed %d\n", mode, (int)r); continue; }
        for (int polmode = 0; polmode < 3; ++polmode) {
        for (int w = 0; w < 3; ++w) stream_kernel<<<148, NT, smem>>>(map, K, ldk, ntt, mode, sink, polmode);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int w = 0; w < reps; ++w) stream_kernel<<<148, NT, smem>>>(map, K, ldk, ntt, mode, sink, polmode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("mode %d pol %d: %.2f us per pass, %.0f GB/s (%s)\n", mode, polmode, ms * 1e3 / reps,
               bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(err));
        }
    }
    return 0;
}
