// Dependent-chain latency (cycles per operation, one warp) of the FP64
// operations the single-CTA dense kernels are built from, and the check that
// the Markstein quotient q' = RN(q + r y), y = RN(1/b), q = RN(a y),
// r = fma(-q, b, a) equals RN(a / b) on random operands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_latency.cu -o tools/_build/fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, double y0, int n) {
    double x = x0, y = y0;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    t1 = clock64();
    cyc[1] = t1 - t0;
    // div_rn chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(x, y) + 1.0;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // sqrt chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dsqrt_rn(x) + 1.0;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // DSETP + select chain (clamp-like)
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double z = x * 1.0000001; x = (fabs(z) < 1e-300) ? -1e-300 : z; }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // shuffle + dadd chain (warp reduction step)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    t1 = clock64();
    cyc[5] = t1 - t0;
    // markstein quotient chain with a fixed reciprocal
    const double r = __ddiv_rn(1.0, y);
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const double q = x * r;
        const double e = fma(-q, y, x);
        x = fma(e, r, q) + 1.0;
    }
    t1 = clock64();
    cyc[6] = t1 - t0;
    out[threadIdx.x] = x;
}

__device__ unsigned long long rng(unsigned long long& s) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s;
}

__global__ void mk_check(unsigned long long seed, long long per_thread, unsigned long long* bad, double* ex) {
    unsigned long long s = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
    for (long long i = 0; i < per_thread; ++i) {
        // random significands and exponents in [-60, 60]
        const unsigned long long ua = rng(s), ub = rng(s);
        const int ea = (int)(rng(s) % 121) - 60, eb = (int)(rng(s) % 121) - 60;
        double a = __longlong_as_double((long long)((ua & 0x000FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + ea) << 52)));
        double b = __longlong_as_double((long long)((ub & 0x000FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + eb) << 52)));
        if (ua & (1ull << 63)) a = -a;
        if (ub & (1ull << 62)) b = -b;
        if ((i & 7) == 0) b = __longlong_as_double((long long)(0x3FFFFFFFFFFFFFFFull - (ub & 0xFF)));   // near-all-ones significands
        const double y = __ddiv_rn(1.0, b);
        const double q = __dmul_rn(a, y);
        const double e = fma(-q, b, a);
        const double qm = fma(e, y, q);
        const double qd = __ddiv_rn(a, b);
        if (__double_as_longlong(qm) != __double_as_longlong(qd)) {
            const unsigned long long k = atomicAdd(bad, 1ull);
            if (k < 4) { ex[3 * k] = a; ex[3 * k + 1] = b; ex[3 * k + 2] = qm - qd; }
        }
    }
}

int main() {
    double* out; long long* cyc; unsigned long long* bad; double* ex;
    cudaMalloc(&out, 1024); cudaMalloc(&cyc, 64); cudaMalloc(&bad, 8); cudaMalloc(&ex, 12 * 8);
    cudaMemset(bad, 0, 8);
    const int n = 4096;
    lat<<<1, 32>>>(out, cyc, 1.1, 0.999, n);
    long long h[8];
    cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost);
    const char* names[7] = {"dfma", "dadd", "div_rn(+add)", "sqrt_rn(+add)", "dmul+setp+sel", "shfl+dadd", "markstein(+add)"};
    for (int i = 0; i < 7; ++i) printf("{\"op\": \"%s\", \"cycles\": %.1f}\n", names[i], (double)h[i] / n);
    const long long per = 1 << 14;
    mk_check<<<148 * 4, 256>>>(12345ull, per, bad, ex);
    unsigned long long nb = 0; double hex[12];
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hex, ex, 96, cudaMemcpyDeviceToHost);
    printf("{\"markstein_pairs\": %lld, \"mismatches\": %llu}\n", (long long)148 * 4 * 256 * per, nb);
    for (unsigned long long k = 0; k < nb && k < 4; ++k) printf("  a=%.17g b=%.17g diff=%g\n", hex[3 * k], hex[3 * k + 1], hex[3 * k + 2]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
