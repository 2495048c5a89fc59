// Latency probes for the single-CTA pencil's critical path (developer tool):
// dependent DFMA chain, rcp.approx.f64 + 2 Newton steps, 5-level f64 warp
// reduction, CTA barrier with 32 warps, generic vs shared loads.  Prints cycles.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
}
__global__ void probe(double* out, long long* cyc, double a, int iters) {
    __shared__ double sh[1024];
    sh[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a + threadIdx.x * 1e-9;
    long long t0, t1;
    // 1: dependent DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
    // 2: rcp chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fast_rcp(x + 1.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
    // 3: warp reduction (5 levels, f64)
    t0 = clock64();
    for (int i = 0; i < iters; ++i)
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
    // 4: barrier, all 32 warps
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x += 1e-9; asm volatile("barrier.sync 0;" ::: "memory"); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
    // 5: dependent generic load chain through smem
    double* gp = sh;
    int idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { idx = ((int)gp[idx] + 1) & 1023; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
    // 6: sqrt (IEEE) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = sqrt(x + 2.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
    // 7: div (IEEE) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = 1.0 / (x + 3.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0) / iters;
    out[threadIdx.x] = x + idx;
}
int main() {
    double* d; long long* c; long long h[8] = {0};
    cudaMalloc(&d, 8192); cudaMalloc(&c, 64);
    probe<<<1, 1024>>>(d, c, 1.5, 1000);
    probe<<<1, 1024>>>(d, c, 1.5, 1000);
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("{\"dfma_dep\": %lld, \"rcp_newton2\": %lld, \"shfl5_f64\": %lld, \"bar_32w\": %lld, \"ld_generic_smem\": %lld, \"sqrt\": %lld, \"div\": %lld}\n",
           h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
    return 0;
}
