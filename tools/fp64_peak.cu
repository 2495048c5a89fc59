// FP64 FMA peak of this GPU (DFMA pipe), for the matrix-free operator's
// roofline: every thread runs 8 independent FMA chains, 148 x 8 CTAs of 256
// threads, timed with CUDA events after a warm-up.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = threadIdx.x * 1e-3 + u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = fma(c[u], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u];
    if (s == 12345.678) out[0] = s;   // keep the chains alive
}

__global__ void exp_kernel(double* out, int iters, double a) {
    double s = threadIdx.x * 1e-6;
    double t = 0.0;
    for (int i = 0; i < iters; ++i) {
        t += exp(-s);
        s = fma(s, a, 1e-9);
    }
    if (t == 12345.678) out[0] = t;
}


// DMMA m8n8k4 (FP64 tensor) throughput: 4 independent accumulator chains per warp.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
    double c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = threadIdx.x * 1e-3 + u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(c[2 * u], c[2 * u + 1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u];
    if (s == 12345.678) out[0] = s;
}
// DMMA and DFMA interleaved: if they share one pipe the time is the sum.
__global__ void mix_kernel(double* out, int iters, double a, double b) {
    double c[8], f[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { c[u] = threadIdx.x * 1e-3 + u; f[u] = c[u] * 0.5; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(c[2 * u], c[2 * u + 1], a, b);
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = fma(f[u], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u] + f[u];
    if (s == 12345.678) out[0] = s;
}

static float time_it(void (*k)(double*, int, double, double), int b, int t, double* d, int it) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<b, t>>>(d, it, 0.999999, 1e-7);
    cudaEventRecord(e0); k<<<b, t>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms = 0.f; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d;
    cudaMalloc(&d, 8);
    const int blocks = sms * 8, threads = 256, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    exp_kernel<<<blocks, threads>>>(d, iters / 8, 0.9999);
    cudaEventRecord(e0);
    exp_kernel<<<blocks, threads>>>(d, iters / 8, 0.9999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2 = 0.f;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double exps = (double)(iters / 8) * blocks * threads;
    const float dm_ms = time_it(dmma_kernel, blocks, threads, d, iters / 4);
    const double dm_flops = 2.0 * 256.0 * 4.0 * (iters / 4) * (double)blocks * (threads / 32);
    const float mx_ms = time_it(mix_kernel, blocks, threads, d, iters / 4);
    printf("{\"dmma_tflops\": %.3f, \"dmma_ms\": %.3f, \"mix_ms\": %.3f, \"dfma_alone_equiv_ms\": %.3f}\n",
           dm_flops / (dm_ms * 1e-3) / 1e12, dm_ms, mx_ms, ms / 4.0);
    printf("{\"fp64_fma_tflops\": %.3f, \"fp64_exp_per_s\": %.4g, \"sms\": %d, \"dfma_ms\": %.3f, \"exp_ms\": %.3f}\n",
           flops / (ms * 1e-3) / 1e12, exps / (ms2 * 1e-3), sms, ms, ms2);
    return 0;
}
