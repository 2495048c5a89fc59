// Cycle cost of the pencil's column-parallel forward substitution (n = 36) on
// one CTA, by variant, to locate where its time goes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/csolve_probe.cu -o tools/_build/csolve_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double div_by_rcp(double a, double b, double y) {
    const unsigned ea = ((unsigned)__double2hiint(a) >> 20) & 0x7ffu, eb = ((unsigned)__double2hiint(b) >> 20) & 0x7ffu;
    if (ea - 543u > 960u || eb - 543u > 960u) return __ddiv_rn(a, b);
    const double q = __dmul_rn(a, y);
    const double r = fma(-q, b, a);
    return fma(r, y, q);
}

template <int V>
__global__ void probe(const double* Lg, const double* Bg, int n, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* L = sm;
    double* B = sm + n * n;
    double* Y = sm + 2 * n * n;
    double* rinv = sm + 3 * n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) { L[e] = Lg[e]; B[e] = Bg[e]; }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) rinv[i] = 1.0 / L[i * n + i];
    __syncthreads();
    const long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep) {
        if (V == 3) {
            // warp per column, lanes own rows lane, lane + 32 (right-looking)
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
            for (int c = warp; c < n; c += nw) {
                double a0 = B[lane * n + c], a1 = (lane + 32 < n) ? B[(lane + 32) * n + c] : 0.0;
                const double r0 = rinv[lane], r1 = (lane + 32 < n) ? rinv[lane + 32] : 0.0;
                for (int j = 0; j < n; ++j) {
                    const double lj0 = (lane > j) ? L[lane * n + j] : 0.0;
                    const double lj1 = (lane + 32 > j && lane + 32 < n) ? L[(lane + 32) * n + j] : 0.0;
                    const double accj = __shfl_sync(0xffffffffu, j < 32 ? a0 : a1, j & 31);
                    const double rj = __shfl_sync(0xffffffffu, j < 32 ? r0 : r1, j & 31);
                    const double yj = div_by_rcp(accj, L[j * n + j], rj);
                    if (lane == (j & 31)) { if (j < 32) a0 = yj; else a1 = yj; }
                    if (lane > j) a0 = sub_rn(a0, mul_rn(lj0, yj));
                    if (lane + 32 > j && lane + 32 < n) a1 = sub_rn(a1, mul_rn(lj1, yj));
                }
                Y[lane * n + c] = a0;
                if (lane + 32 < n) Y[(lane + 32) * n + c] = a1;
            }
            __syncthreads();
            continue;
        }
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            for (int i = 0; i < n; ++i) {
                double a = B[i * n + c];
                const double* li = L + i * n;
                if (V == 2) {
                    int j = 0;
                    for (; j + 8 <= i; j += 8) {
                        double m[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) m[u] = mul_rn(li[j + u], Y[(j + u) * n + c]);
#pragma unroll
                        for (int u = 0; u < 8; ++u) a = sub_rn(a, m[u]);
                    }
                    for (; j < i; ++j) a = sub_rn(a, mul_rn(li[j], Y[j * n + c]));
                } else {
                    for (int j = 0; j < i; ++j) a = sub_rn(a, mul_rn(li[j], Y[j * n + c]));
                }
                if (V == 1) Y[i * n + c] = a * rinv[i];
                else Y[i * n + c] = __ddiv_rn(a, li[i]);
            }
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[V] = (t1 - t0) / 10;
    if (threadIdx.x < n) out[threadIdx.x] = Y[threadIdx.x];
}

int main() {
    const int n = 36;
    double hL[n * n], hB[n * n];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            hL[i * n + j] = (j < i) ? 0.01 * ((i * 7 + j * 3) % 11) : (j == i ? 1.0 + 0.1 * i : 0.0);
            hB[i * n + j] = 0.5 + 0.01 * ((i + 2 * j) % 13);
        }
    double *L, *B, *out; long long* cyc;
    double yref[64], ywarp[64];
    cudaMalloc(&L, sizeof hL); cudaMalloc(&B, sizeof hB); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
    cudaMemcpy(L, hL, sizeof hL, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    const int smem = (3 * n * n + n) * 8;
    for (int nt : {32, 64, 1024}) {
        probe<0><<<1, nt, smem>>>(L, B, n, out, cyc);
        probe<1><<<1, nt, smem>>>(L, B, n, out, cyc);
        probe<2><<<1, nt, smem>>>(L, B, n, out, cyc);
        probe<3><<<1, nt, smem>>>(L, B, n, out, cyc);
        long long h[4];
        cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
        printf("threads %4d: div_rn %lld cycles, rcp-mul %lld, batched+div %lld, warp-per-column %lld (%s)\n", nt, h[0],
               h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
