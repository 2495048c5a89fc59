// Developer probe: cost of one one-sided Jacobi round (the Ritz pencil's
// critical path) with parts switched off.  T = 36, 18 pairs, 1024 threads.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
    double r;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double hx = 0.5 * x;
    r = r * fma(-hx * r, r, 1.5);
    r = r * fma(-hx * r, r, 1.5);
    return r;
}
template <int MODE>   // bit0: no V, bit1: no rotation math, bit2: no shuffles, bit3: no barrier
__global__ void jac(double* gX, long long* out, int rounds) {
    __shared__ double X[36 * 36], Vc[36 * 36];
    const int n = 36, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int e = tid; e < n * n; e += blockDim.x) { X[e] = gX[e]; Vc[e] = (e % 37 == 0) ? 1.0 : 0.0; }
    __syncthreads();
    const int i0 = lane, i1 = lane + 32, Te = 36, np = 18;
    long long t0 = clock64();
    for (int rr = 0; rr < rounds; ++rr) {
        const int round = rr % 35;
        for (int slot = warp; slot < np; slot += nw) {
            int pa = slot == 0 ? Te - 1 : slot - 1 + round;
            if (slot != 0 && pa >= Te - 1) pa -= Te - 1;
            int pb = Te - 2 - slot + round;
            if (pb >= Te - 1) pb -= Te - 1;
            const int p = min(pa, pb), q = max(pa, pb);
            const double xp0 = X[p * n + i0], xp1 = i1 < n ? X[p * n + i1] : 0.0;
            const double xq0 = X[q * n + i0], xq1 = i1 < n ? X[q * n + i1] : 0.0;
            double app = fma(xp1, xp1, xp0 * xp0), aqq = fma(xq1, xq1, xq0 * xq0), apq = fma(xp1, xq1, xp0 * xq0);
            if (!(MODE & 4)) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    app += __shfl_xor_sync(0xffffffffu, app, o);
                    aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
                    apq += __shfl_xor_sync(0xffffffffu, apq, o);
                }
            }
            double c = 0.8, sn = 0.6;
            if (MODE & 16) {
                // t = sgn |e| / (|d| + sqrt(d^2 + e^2)), d = aqq - app, e = 2 apq
                const double d = aqq - app, e = 2.0 * apq;
                const double w = fma(d, d, e * e);
                const double r = w * fast_rsqrt(w);
                double t = fabs(e) * fast_rcp(fabs(d) + r);
                if ((d < 0.0) != (e < 0.0) && d != 0.0) t = -t;
                c = fast_rsqrt(fma(t, t, 1.0));
                sn = t * c;
            } else if (!(MODE & 2)) {
                const double tau = (aqq - app) * fast_rcp(2.0 * apq);
                const double at = fabs(tau);
                const double w = fma(tau, tau, 1.0);
                double t = fast_rcp(at + w * fast_rsqrt(w));
                if (tau < 0.0) t = -t;
                c = fast_rsqrt(fma(t, t, 1.0));
                sn = t * c;
            }
            X[p * n + i0] = c * xp0 - sn * xq0;
            X[q * n + i0] = sn * xp0 + c * xq0;
            if (i1 < n) { X[p * n + i1] = c * xp1 - sn * xq1; X[q * n + i1] = sn * xp1 + c * xq1; }
            if (!(MODE & 1)) {
                const double vp = Vc[p * n + i0], vq = Vc[q * n + i0];
                Vc[p * n + i0] = c * vp - sn * vq;
                Vc[q * n + i0] = sn * vp + c * vq;
                if (i1 < n) {
                    const double vp1 = Vc[p * n + i1], vq1 = Vc[q * n + i1];
                    Vc[p * n + i1] = c * vp1 - sn * vq1;
                    Vc[q * n + i1] = sn * vp1 + c * vq1;
                }
            }
        }
        if (MODE & 32) { if (warp < 18) asm volatile("barrier.sync 1, 576;" ::: "memory"); }
        else if (!(MODE & 8)) asm volatile("barrier.sync 0;" ::: "memory");
    }
    long long t1 = clock64();
    if (tid == 0) out[MODE] = (t1 - t0) / rounds;
    if (tid < 36) gX[tid] = X[tid] + Vc[tid];
}
// FP32 round (same structure): X, V floats; rotation from rcp/rsqrt approx f32
__global__ void jac32(double* gX, long long* out, int rounds) {
    __shared__ float X[36 * 36], Vc[36 * 36];
    const int n = 36, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int e = tid; e < n * n; e += blockDim.x) { X[e] = (float)gX[e]; Vc[e] = (e % 37 == 0) ? 1.f : 0.f; }
    __syncthreads();
    const int i0 = lane, i1 = lane + 32, Te = 36, np = 18;
    long long t0 = clock64();
    for (int rr = 0; rr < rounds; ++rr) {
        const int round = rr % 35;
        for (int slot = warp; slot < np; slot += nw) {
            int pa = slot == 0 ? Te - 1 : slot - 1 + round;
            if (slot != 0 && pa >= Te - 1) pa -= Te - 1;
            int pb = Te - 2 - slot + round;
            if (pb >= Te - 1) pb -= Te - 1;
            const int p = min(pa, pb), q = max(pa, pb);
            const float xp0 = X[p * n + i0], xp1 = i1 < n ? X[p * n + i1] : 0.f;
            const float xq0 = X[q * n + i0], xq1 = i1 < n ? X[q * n + i1] : 0.f;
            const float vp0 = Vc[p * n + i0], vq0 = Vc[q * n + i0];
            const float vp1 = i1 < n ? Vc[p * n + i1] : 0.f, vq1 = i1 < n ? Vc[q * n + i1] : 0.f;
            float app = fmaf(xp1, xp1, xp0 * xp0), aqq = fmaf(xq1, xq1, xq0 * xq0), apq = fmaf(xp1, xq1, xp0 * xq0);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                app += __shfl_xor_sync(0xffffffffu, app, o);
                aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
                apq += __shfl_xor_sync(0xffffffffu, apq, o);
            }
            const float tau = (aqq - app) * __frcp_rn(2.f * apq);
            const float at = fabsf(tau);
            float t = __frcp_rn(at + sqrtf(fmaf(tau, tau, 1.f)));
            if (tau < 0.f) t = -t;
            const float c = rsqrtf(fmaf(t, t, 1.f)), sn = t * c;
            X[p * n + i0] = c * xp0 - sn * xq0;
            X[q * n + i0] = sn * xp0 + c * xq0;
            Vc[p * n + i0] = c * vp0 - sn * vq0;
            Vc[q * n + i0] = sn * vp0 + c * vq0;
            if (i1 < n) {
                X[p * n + i1] = c * xp1 - sn * xq1; X[q * n + i1] = sn * xp1 + c * xq1;
                Vc[p * n + i1] = c * vp1 - sn * vq1; Vc[q * n + i1] = sn * vp1 + c * vq1;
            }
        }
        asm volatile("barrier.sync 0;" ::: "memory");
    }
    long long t1 = clock64();
    if (tid == 0) out[63] = (t1 - t0) / rounds;
    if (tid < 36) gX[tid] = X[tid] + Vc[tid];
}
int main() {
    double h[36 * 36];
    for (int i = 0; i < 36 * 36; ++i) h[i] = (i % 37 == 0 ? 3.0 : 0.01 * ((i * 7919) % 101 - 50));
    double* d; long long* o; long long ho[64] = {0};
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, sizeof(ho)); cudaMemset(o, 0, sizeof(ho));
    const int R = 210;
#define RUN(M) cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice); jac<M><<<1, 1024>>>(d, o, R); cudaDeviceSynchronize();
    RUN(0) RUN(0) RUN(1) RUN(2) RUN(4) RUN(8) RUN(7) RUN(15) RUN(16) RUN(32) RUN(48)
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("{\"cheaprot\": %lld, \"bar18\": %lld, \"cheaprot+bar18\": %lld}\n", ho[16], ho[32], ho[48]);
    printf("{\"full\": %lld, \"noV\": %lld, \"norot\": %lld, \"noshfl\": %lld, \"nobar\": %lld, \"only_ld_st_bar\": %lld, \"only_ld_st\": %lld}\n",
           ho[0], ho[1], ho[2], ho[4], ho[8], ho[7], ho[15]);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice); jac32<<<1, 1024>>>(d, o, R); cudaDeviceSynchronize();
    jac32<<<1, 1024>>>(d, o, R); cudaDeviceSynchronize();
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("{\"fp32_round\": %lld}\n", ho[63]);
    // 256-thread variant (18 warps needed -> use 576)
    return 0;
}
