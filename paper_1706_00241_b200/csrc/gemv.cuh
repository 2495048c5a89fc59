// Block-level stored-Gram GEMV (kernel K1 of SURVEY.md section 2).
//
// Replaces _core.matvec (_core.pyx:16-28) inside the CG loop (solvers.py:169)
// and the GPC K-products (gpc.py:182,191,206).  A = shift*I + S K S is never
// materialised (the reference builds it at gpc.py:178): the CTA stages
// x' = s (.) v for a column tile into shared memory once, then streams its own
// contiguous rows of K with 16-byte non-allocating loads, DCG_RG rows at a
// time so every thread keeps 2*DCG_RG independent 16 B loads in flight.
// Per-warp row partials land in shared memory and are summed over warps in a
// fixed order (deterministic), then handed to the caller's epilogue which
// sees (local row, sum_j K[row, j] x'_j).
#pragma once
#include "common.cuh"

// s_x[c] = s[c0+c] * v[c0+c] (or v) for c < cn; pads one zero when cn is odd.
template <bool kCrossCta>
__device__ __forceinline__ void stage_x_tile(double* s_x, const double* v, const double* s,
                                             long long c0, int cn) {
    for (int c = threadIdx.x; c < cn; c += blockDim.x) {
        double vv = kCrossCta ? ld_cg(v + c0 + c) : __ldg(v + c0 + c);
        s_x[c] = s ? mul_rn(__ldg(s + c0 + c), vv) : vv;
    }
    if ((cn & 1) && threadIdx.x == 0) s_x[cn] = 0.0;
}

// Rows [r0, r1) of the slab K (row-major, leading dimension ldk, n columns).
// `s_red` needs DCG_NW * DCG_RB doubles, `s_x` min(n, DCG_QT) + 1 doubles.
// Epilogue `epi(row, t)` runs on thread (row - batch start) after a barrier.
// All threads of the CTA must call this (it contains CTA barriers).
template <bool kCrossCta, class Epi>
__device__ __forceinline__ void block_gemv(const double* __restrict__ K, long long ldk, long long n,
                                           const double* v, const double* s, long long r0,
                                           long long r1, double* s_x, double* s_red, Epi&& epi) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x;
    const bool single_tile = n <= DCG_QT;
    if (single_tile) {
        cta_sync();
        stage_x_tile<kCrossCta>(s_x, v, s, 0, (int)n);
        cta_sync();
    }
    for (long long rb0 = r0; rb0 < r1; rb0 += DCG_RB) {
        const int nb = (int)min((long long)DCG_RB, r1 - rb0);
        for (long long c0 = 0; c0 < n; c0 += DCG_QT) {
            const int cn = (int)min((long long)DCG_QT, n - c0);
            if (!single_tile) {
                cta_sync();
                stage_x_tile<kCrossCta>(s_x, v, s, c0, cn);
                cta_sync();
            }
            const int cn2 = cn & ~1;
            for (int g = 0; g < nb; g += DCG_RG) {
                double acc[DCG_RG];
                const double* rowp[DCG_RG];
#pragma unroll
                for (int rr = 0; rr < DCG_RG; ++rr) {
                    acc[rr] = 0.0;
                    const int lr = min(g + rr, nb - 1);   // tail rows re-read the last row
                    rowp[rr] = K + (rb0 + lr) * ldk + c0;
                }
#pragma unroll 2
                for (int c = 2 * tid; c < cn2; c += 2 * NT) {
                    const double2 xv = *reinterpret_cast<const double2*>(s_x + c);
#pragma unroll
                    for (int rr = 0; rr < DCG_RG; ++rr) {
                        const double2 kv = ld_stream2(rowp[rr] + c);
                        acc[rr] = fma(kv.x, xv.x, acc[rr]);
                        acc[rr] = fma(kv.y, xv.y, acc[rr]);
                    }
                }
                if ((cn & 1) && tid == 0) {
#pragma unroll
                    for (int rr = 0; rr < DCG_RG; ++rr)
                        acc[rr] = fma(ld_stream(rowp[rr] + cn - 1), s_x[cn - 1], acc[rr]);
                }
#pragma unroll
                for (int rr = 0; rr < DCG_RG; ++rr) {
                    const double t = warp_sum(acc[rr]);
                    if (lane == 0 && g + rr < nb) {
                        double* slot = s_red + warp * DCG_RB + g + rr;
                        *slot = (c0 == 0) ? t : (*slot + t);
                    }
                }
            }
        }
        cta_sync();
        if (tid < nb) {
            double t = 0.0;
#pragma unroll 4
            for (int w = 0; w < DCG_NW; ++w) t += s_red[w * DCG_RB + tid];
            epi(rb0 + tid, t);
        }
        cta_sync();
    }
}
