// Matrix-free RBF operator (kernel K7 of SURVEY.md section 2; config 5).
//
// K_ij = var * exp(-||x_i - x_j||^2 / (2 l^2)) (i != j), K_ii = var + jitter,
// is never stored: every product regenerates it tile by tile from the data
// X (n x d, row-major, read through L2).  Elements are computed exactly as
// the stored-Gram builder does (rbf_tile_kernel, _core.pyx:97-114): the
// squared distance accumulated in ascending coordinate order with separate
// rounded sub / mul / add, then var * exp(-acc * inv_two_ell2) - so a
// matrix-free product equals the stored-Gram product up to the summation
// order of the row sums.
//
// Row-owned form: a CTA owns 64-row chunks of its row range and sweeps all
// 64-column tiles; warp w computes columns 4w..4w+3 of each tile and lane l
// rows 2l, 2l+1 (8 elements per thread per tile).  X_I and X_J are staged
// transposed in shared memory so a thread's 2 row coordinates and 4 column
// coordinates are one 16-byte and two 16-byte (warp-broadcast) loads per
// coordinate.  The operator is FP64-pipe bound (3d + exp flops per element).
#pragma once
#include "common.cuh"

#define MF_TB 64

// shared memory (doubles) of rbf_rows_gemv for data dimension `dim`
__host__ __device__ __forceinline__ long long rbf_mf_smem_doubles(int dim) {
    return 2LL * dim * MF_TB + MF_TB + DCG_NW * MF_TB;
}

struct RbfParams {
    const double* X;
    long long n;
    int dim;
    double var, inv2, diag;
};

// the 8 kernel values of this thread in tile (rows gi0 + {2l, 2l+1}, cols gj0 + 4w + {0..3});
// xit: dim x 64 (rows of the I chunk), xjt: dim x 64 (J tile); out-of-range -> 0
__device__ __forceinline__ void rbf_tile_values(const RbfParams& p, const double* xit, const double* xjt,
                                                long long gi0, long long gj0, long long row_end, double k[2][4]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    for (int t = 0; t < p.dim; ++t) {
        const double2 xi = *reinterpret_cast<const double2*>(xit + t * MF_TB + 2 * lane);
        const double2 xa = *reinterpret_cast<const double2*>(xjt + t * MF_TB + 4 * warp);
        const double2 xb = *reinterpret_cast<const double2*>(xjt + t * MF_TB + 4 * warp + 2);
        const double xr[2] = {xi.x, xi.y};
        const double xc[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double diff = sub_rn(xr[r], xc[c]);
                acc[r][c] = add_rn(acc[r][c], mul_rn(diff, diff));
            }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const long long gi = gi0 + 2 * lane + r, gj = gj0 + 4 * warp + c;
            double v;
            if (gi >= row_end || gj >= p.n) v = 0.0;
            else if (gi == gj) v = p.diag;
            else v = mul_rn(p.var, exp(mul_rn(-acc[r][c], p.inv2)));
            k[r][c] = v;
        }
}

// stage rows [g0, g0 + 64) of X transposed into dst (dim x 64), zero beyond `end`
__device__ __forceinline__ void rbf_stage_rows(const RbfParams& p, long long g0, long long end, double* dst) {
    for (int e = threadIdx.x; e < p.dim * MF_TB; e += blockDim.x) {
        const int r = e / p.dim, t = e - (e / p.dim) * p.dim;   // coalesced over the row-major X
        const long long g = g0 + r;
        dst[t * MF_TB + r] = (g < end) ? __ldg(p.X + g * p.dim + t) : 0.0;
    }
}

// t_i = sum_j K_ij (s_j v_j) for rows [r0, r1) (global indices); epi(i, t_i)
// on one thread per row.  `smem` holds rbf_mf_smem_doubles(dim).  All CTA
// threads call (contains CTA barriers).
template <class Epi>
__device__ void rbf_rows_gemv(const RbfParams& p, long long r0, long long r1, const double* v, const double* s,
                              double* smem, Epi&& epi) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* xit = smem;
    double* xjt = xit + p.dim * MF_TB;
    double* vj = xjt + p.dim * MF_TB;
    double* red = vj + MF_TB;
    for (long long i0 = r0; i0 < r1; i0 += MF_TB) {
        cta_sync();
        rbf_stage_rows(p, i0, r1, xit);
        double row[2] = {0.0, 0.0};
        for (long long j0 = 0; j0 < p.n; j0 += MF_TB) {
            cta_sync();
            rbf_stage_rows(p, j0, p.n, xjt);
            if (tid < MF_TB) {
                const long long j = j0 + tid;
                double vv = 0.0;
                if (j < p.n) {
                    vv = ld_cg(v + j);
                    if (s) vv = mul_rn(__ldg(s + j), vv);
                }
                vj[tid] = vv;
            }
            cta_sync();
            double k[2][4];
            rbf_tile_values(p, xit, xjt, i0, j0, r1, k);
            const double2 va = *reinterpret_cast<const double2*>(vj + 4 * warp);
            const double2 vb = *reinterpret_cast<const double2*>(vj + 4 * warp + 2);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                row[r] = fma(k[r][0], va.x, row[r]);
                row[r] = fma(k[r][1], va.y, row[r]);
                row[r] = fma(k[r][2], vb.x, row[r]);
                row[r] = fma(k[r][3], vb.y, row[r]);
            }
        }
        // combine the 16 warps' column groups in a fixed order
        red[warp * MF_TB + 2 * lane] = row[0];
        red[warp * MF_TB + 2 * lane + 1] = row[1];
        cta_sync();
        if (tid < MF_TB && i0 + tid < r1) {
            double t = 0.0;
#pragma unroll 4
            for (int w = 0; w < DCG_NW; ++w) t += red[w * MF_TB + tid];
            epi(i0 + tid, t);
        }
    }
    cta_sync();
}
