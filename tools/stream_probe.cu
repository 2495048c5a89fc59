// Read-stream probe: how fast can 148 persistent CTAs pull a matrix's
// lower-triangle 64 x 64 fp64 tiles into shared memory, by layout and copy
// method (consumers read every element once from shared memory, no math):
//   mode 0  packed tiles (each 32 KB tile contiguous), one cp.async.bulk per tile
//   mode 1  row-major storage, per-thread 16-byte cp.async (the current ring)
//   mode 2  row-major storage, 64 cp.async.bulk row pieces of 512 B per tile
//   mode 3  plain grid-stride ld.global.nc.v2 over the packed buffer (reference)
// Usage: stream_probe n stages reps
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/stream_probe.cu -o tools/_build/stream_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define NT 512
#define TB 64
#define TILE (TB * TB)

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
__device__ __forceinline__ unsigned long long pol_normal() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ int g_policy;   // 0 evict_first, 1 evict_normal
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                     unsigned long long pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void cpa16(void* dst, const void* src, unsigned long long pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa(dst)), "l"(src), "l"(pol));
}

__device__ long long tile_row(long long t) {
    long long I = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    return I;
}

__global__ void __launch_bounds__(NT, 1) ring_kernel(const double* K, long long ldk, long long ntt, int mode,
                                                     int stages, double* sink) {
    extern __shared__ __align__(128) double smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + stages * TILE);
    unsigned long long* empty = full + stages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long t0 = ntt * blockIdx.x / gridDim.x, t1 = ntt * (blockIdx.x + 1) / gridDim.x;
    const int nt = (int)(t1 - t0);
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full + s, mode == 1 ? NT : 1);
            mbar_init(empty + s, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long pol = g_policy ? pol_normal() : pol_first();
    auto issue = [&](int lt) {
        const int st = lt % stages;
        double* dst = smem + st * TILE;
        const long long t = t0 + lt;
        if (mode == 0) {
            if (tid == 0) {
                mbar_expect(full + st, TILE * 8);
                bulk(dst, K + t * TILE, TILE * 8, full + st, pol);
            }
        } else {
            const long long I = tile_row(t), J = t - I * (I + 1) / 2;
            const double* kt = K + I * TB * ldk + J * TB;
            if (mode == 1) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int row = (tid >> 5) + 16 * u;
                    cpa16(dst + row * TB + 2 * (tid & 31), kt + row * ldk + 2 * (tid & 31), pol);
                }
                cp_arrive(full + st);
            } else {
                if (tid == 0) mbar_expect(full + st, TILE * 8);
                __syncwarp();
                if (tid < 32) {
                    for (int row = lane; row < TB; row += 32) bulk(dst + row * TB, kt + row * ldk, TB * 8, full + st, pol);
                }
            }
        }
    };
    const bool producer = (mode == 1) || (warp == 0);
    for (int lt = 0; lt < stages - 1 && lt < nt; ++lt)
        if (producer) issue(lt);
    double acc = 0.0;
    for (int lt = 0; lt < nt; ++lt) {
        const int tn = lt + stages - 1;
        if (tn < nt && producer) {
            const int st = tn % stages;
            if (tn >= stages) mbar_wait(empty + st, ((tn / stages) - 1) & 1);
            issue(tn);
        }
        const int st = lt % stages;
        mbar_wait(full + st, (lt / stages) & 1);
        const double2* tile = reinterpret_cast<const double2*>(smem + st * TILE);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2 v = tile[tid + NT * u];
            acc += v.x + v.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
    }
    if (acc == 12345.678) sink[blockIdx.x] = acc;
}

__global__ void plain_kernel(const double2* K, long long n2, double* sink) {
    double acc = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(K + i + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) acc += K[i].x;
    if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 10000;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    const long long NTs = (n + TB - 1) / TB, ntt = NTs * (NTs + 1) / 2, ldk = NTs * TB;
    const size_t rowmajor = (size_t)ldk * ldk * 8, packed = (size_t)ntt * TILE * 8;
    double *K, *sink;
    cudaMalloc(&K, rowmajor > packed ? rowmajor : packed);
    cudaMemset(K, 0, rowmajor > packed ? rowmajor : packed);
    cudaMalloc(&sink, 4096 * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)packed;
    {
        const int pm = getenv("PROBE_POLICY") ? atoi(getenv("PROBE_POLICY")) : 0;
        cudaMemcpyToSymbol(g_policy, &pm, sizeof(int));
    }
    for (int stages = 3; stages <= 6; ++stages) {
        if (argc > 2 && atoi(argv[2]) > 0 && stages != atoi(argv[2])) continue;
        const size_t smem = (size_t)stages * TILE * 8 + 2 * stages * 8;
        cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int mode = 0; mode < 3; ++mode) {
            for (int w = 0; w < 3; ++w) ring_kernel<<<sms, NT, smem>>>(K, ldk, ntt, mode, stages, sink);
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) ring_kernel<<<sms, NT, smem>>>(K, ldk, ntt, mode, stages, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const cudaError_t err = cudaGetLastError();
            printf("{\"n\": %lld, \"mode\": %d, \"stages\": %d, \"us\": %.2f, \"GBps\": %.0f, \"err\": \"%s\"}\n", n, mode,
                   stages, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9, cudaGetErrorString(err));
        }
    }
    for (int occ = 1; occ <= 4; occ *= 2) {
        for (int w = 0; w < 3; ++w) plain_kernel<<<sms * occ, 1024 / occ * occ / occ, 0>>>((const double2*)K, packed / 16, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) plain_kernel<<<sms * 2 * occ, 512, 0>>>((const double2*)K, packed / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"n\": %lld, \"mode\": 3, \"ctas_per_sm\": %d, \"us\": %.2f, \"GBps\": %.0f}\n", n, 2 * occ,
               ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9);
    }
    return 0;
}
