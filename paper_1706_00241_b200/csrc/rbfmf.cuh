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

// exp(x) for x <= 0 without branches (the kernel argument -|d|^2 / (2 l^2)):
// k = rint(x log2 e), r = x - k ln 2 (two-part ln 2), |r| <= ln2 / 2; degree-13
// Taylor polynomial (truncation r^14 / 14! < 5e-18) in Horner form, scaled by
// adding k to the exponent field; x < -708 returns 0.  A few ulp; ~25 FP64
// instructions against the general-purpose exp's range checks and branches.
__device__ __forceinline__ double rbf_exp_neg(double x) {
    const bool under = x < -708.0;
    x = fmax(x, -708.0);
    const double kf = rint(x * 1.4426950408889634074);
    double r = fma(kf, -6.93147180369123816490e-01, x);
    r = fma(kf, -1.90821492927058770002e-10, r);
    double p = 1.6059043836821614599e-10;            // 1/13!
    p = fma(p, r, 2.0876756987868098979e-09);        // 1/12!
    p = fma(p, r, 2.5052108385441718775e-08);        // 1/11!
    p = fma(p, r, 2.7557319223985890653e-07);        // 1/10!
    p = fma(p, r, 2.7557319223985890653e-06);        // 1/9!
    p = fma(p, r, 2.4801587301587301587e-05);        // 1/8!
    p = fma(p, r, 1.9841269841269841270e-04);        // 1/7!
    p = fma(p, r, 1.3888888888888888889e-03);        // 1/6!
    p = fma(p, r, 8.3333333333333333333e-03);        // 1/5!
    p = fma(p, r, 4.1666666666666666667e-02);        // 1/4!
    p = fma(p, r, 1.6666666666666666667e-01);        // 1/3!
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const long long bits = __double_as_longlong(p) + ((long long)(int)kf << 52);
    return under ? 0.0 : __longlong_as_double(bits);
}

// shared memory (doubles) of rbf_rows_gemv for data dimension `dim`
__host__ __device__ __forceinline__ long long rbf_mf_smem_doubles(int dim) {
    return 2LL * dim * MF_TB + MF_TB + DCG_NW * MF_TB + 2 * MF_TB;
}

struct RbfParams {
    const double* X;
    long long n;
    int dim;
    double var, inv2, diag;
};

// the 8 kernel values of this thread in tile (rows gi0 + {2l, 2l+1}, cols gj0 + 4w + {0..3});
// xit: dim x 64 (rows of the I chunk), xjt: dim x 64 (J tile); out-of-range -> 0.
// FAST: the squared distance as |x_i|^2 + |x_j|^2 - 2 x_i.x_j from the staged
// row norms nI / nJ (one FMA per coordinate; the cancellation error is ~eps
// |x|^2 absolute in the exponent, ~1e-16 relative in K) and the branch-free
// exponential; otherwise the stored builder's exact difference form
// (bit-identical elements).
template <bool FAST>
__device__ __forceinline__ void rbf_tile_values(const RbfParams& p, const double* xit, const double* xjt,
                                                long long gi0, long long gj0, long long row_end, double k[2][4],
                                                const double* nI = nullptr, const double* nJ = nullptr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    const double* pi = xit + 2 * lane;
    const double* pj = xjt + 4 * warp;
#pragma unroll 4
    for (int t = 0; t < p.dim; ++t, pi += MF_TB, pj += MF_TB) {
        const double2 xi = *reinterpret_cast<const double2*>(pi);
        const double2 xa = *reinterpret_cast<const double2*>(pj);
        const double2 xb = *reinterpret_cast<const double2*>(pj + 2);
        const double xr[2] = {xi.x, xi.y};
        const double xc[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if constexpr (FAST) {
                    acc[r][c] = fma(xr[r], xc[c], acc[r][c]);
                } else {
                    const double diff = sub_rn(xr[r], xc[c]);
                    acc[r][c] = add_rn(acc[r][c], mul_rn(diff, diff));
                }
            }
    }
    if constexpr (FAST) {
        const double2 ni = *reinterpret_cast<const double2*>(nI + 2 * lane);
        const double2 na = *reinterpret_cast<const double2*>(nJ + 4 * warp);
        const double2 nb = *reinterpret_cast<const double2*>(nJ + 4 * warp + 2);
        const double nr[2] = {ni.x, ni.y};
        const double nc[4] = {na.x, na.y, nb.x, nb.y};
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = fmax(0.0, fma(-2.0, acc[r][c], nr[r] + nc[c]));
    }
    const long long gib = gi0 + 2 * lane, gjb = gj0 + 4 * warp;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double v;
            if constexpr (FAST) v = p.var * rbf_exp_neg(-acc[r][c] * p.inv2);
            else v = mul_rn(p.var, exp(mul_rn(-acc[r][c], p.inv2)));
            v = (gib + r == gjb + c) ? p.diag : v;
            v = (gib + r < row_end && gjb + c < p.n) ? v : 0.0;
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

// squared norms of the staged rows (dim x 64 transposed) into nrm[64], fixed order
__device__ __forceinline__ void rbf_stage_norms(const RbfParams& p, const double* xt, double* nrm) {
    if (threadIdx.x < MF_TB) {
        double a = 0.0;
        for (int t = 0; t < p.dim; ++t) a = fma(xt[t * MF_TB + threadIdx.x], xt[t * MF_TB + threadIdx.x], a);
        nrm[threadIdx.x] = a;
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
    double* nI = red + DCG_NW * MF_TB;
    double* nJ = nI + MF_TB;
    for (long long i0 = r0; i0 < r1; i0 += MF_TB) {
        cta_sync();
        rbf_stage_rows(p, i0, r1, xit);
        cta_sync();
        rbf_stage_norms(p, xit, nI);
        double row[2] = {0.0, 0.0};
        for (long long j0 = 0; j0 < p.n; j0 += MF_TB) {
            cta_sync();
            rbf_stage_rows(p, j0, p.n, xjt);
            cta_sync();
            rbf_stage_norms(p, xjt, nJ);
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
            rbf_tile_values<true>(p, xit, xjt, i0, j0, r1, k, nI, nJ);
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

// The unsharded operator's symmetric half-evaluation (each lower-triangle
// tile generated once, serving its row and column sums) runs on the FP64
// tensor pipe: rbfmma.cuh.  The row-owned form above serves row slabs
// (sharded operators) and the multi-vector product.
