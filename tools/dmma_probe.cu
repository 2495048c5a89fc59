// DMMA (mma.sync.m8n8k4.f64) latency and throughput vs independent chains per warp
// and warps per SM (developer probe).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
    double c[CH][2];
    for (int u = 0; u < CH; ++u) c[u][0] = c[u][1] = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < CH; ++u) dmma(c[u][0], c[u][1], 1.0000001, 0.9999999);
    long long t1 = clock64();
    double s = 0; for (int u = 0; u < CH; ++u) s += c[u][0] + c[u][1];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[CH] = (t1 - t0) / iters;
}
int main() {
    double* d; long long* c; long long h[16] = {0};
    cudaMalloc(&d, 8); cudaMalloc(&c, 128);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // latency: 1 warp, 1 chain
    k<1><<<1, 32>>>(d, c, 1000); k<1><<<1, 32>>>(d, c, 1000);
    cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
    printf("latency_1chain_1warp_cycles %lld\n", h[1]);
    // throughput: 148 CTAs x W warps x CH chains
    for (int w : {4, 8, 16, 32}) {
        float ms;
        const int it = 2000;
        k<4><<<148, 32 * w>>>(d, c, it);
        cudaEventRecord(e0); k<4><<<148, 32 * w>>>(d, c, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256 * 4 * it * 148.0 * w;
        printf("warps/SM %2d chains 4: %.1f TFLOP/s\n", w, fl / (ms * 1e-3) / 1e12);
        k<8><<<148, 32 * w>>>(d, c, it);
        cudaEventRecord(e0); k<8><<<148, 32 * w>>>(d, c, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 256 * 8 * it * 148.0 * w;
        printf("warps/SM %2d chains 8: %.1f TFLOP/s\n", w, fl / (ms * 1e-3) / 1e12);
    }
    return 0;
}
