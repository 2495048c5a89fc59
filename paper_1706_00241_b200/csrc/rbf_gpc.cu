// RBF Gram assembly (K6) and the GPC Laplace-Newton element-wise glue (K8).
//
// rbf_tile_kernel restates _core.rbf_gram / rbf_cross (_core.pyx:97-132):
// squared distances accumulate left to right over dimensions with separate
// multiply/add, the diagonal is exactly var + jitter, and every entry is
// evaluated directly from (x_i, x_j).  Because (a-b)^2 == (b-a)^2 bit for bit,
// K[i][j] == K[j][i] exactly without mirroring, so a row slab [row0, row0+rows)
// can be built independently on each rank of a row-sharded operator.
//
// The GPC kernels restate gpc.py:126-209 (sigmoid, logaddexp, curvature,
// Newton right-hand side and update, psi) with deterministic reductions.
#include "common.cuh"
#include "symgemv.cuh"

#define RBF_T 64     // tile edge (rows and columns per CTA)
#define RBF_D 32     // dimensions staged per round

// A CTA evaluates a 64 x 64 tile, 16 entries per thread (columns tx, tx + 32;
// rows ty + 8 rr): the staging and barriers of a tile are shared by four
// times the entries of a 32 x 32 tile.
__global__ void __launch_bounds__(256)
    rbf_tile_kernel(const double* __restrict__ xr, long long nr_total, const double* __restrict__ xc,
                    long long nc, long long dim, double var, double inv2l2, double jitter, int gram,
                    long long row0, long long rows, double* out, long long ldo) {
    __shared__ double sbuf[2 * RBF_T * (RBF_D + 1)];
    double (*sr)[RBF_D + 1] = reinterpret_cast<double (*)[RBF_D + 1]>(sbuf);
    double (*sc)[RBF_D + 1] = reinterpret_cast<double (*)[RBF_D + 1]>(sbuf + RBF_T * (RBF_D + 1));
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const long long i0 = (long long)blockIdx.y * RBF_T;        // local row tile
    const long long j0 = (long long)blockIdx.x * RBF_T;
    // whole square Gram: evaluate the tiles on and below the diagonal only
    // and store each off-diagonal tile a second time, transposed -- the
    // mirrored value is the directly evaluated one bit for bit (see above)
    const bool mirror = gram && row0 == 0 && rows == nc;
    if (mirror && blockIdx.x > blockIdx.y) return;
    double acc[8][2];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
    for (long long t0 = 0; t0 < dim; t0 += RBF_D) {
        const int tn = (int)min((long long)RBF_D, dim - t0);
        for (int e = threadIdx.x; e < RBF_T * RBF_D; e += 256) {
            const int r = e / RBF_D, t = e % RBF_D;
            const long long gi = row0 + i0 + r, gj = j0 + r;
            sr[r][t] = (t < tn && i0 + r < rows) ? xr[gi * dim + t0 + t] : 0.0;
            sc[r][t] = (t < tn && gj < nc) ? xc[gj * dim + t0 + t] : 0.0;
        }
        cta_sync();
        for (int t = 0; t < tn; ++t) {
            const double c0 = sc[tx][t], c1 = sc[tx + 32][t];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const double rv = sr[ty + 8 * rr][t];
                const double d0 = sub_rn(rv, c0), d1 = sub_rn(rv, c1);
                acc[rr][0] = add_rn(acc[rr][0], mul_rn(d0, d0));
                acc[rr][1] = add_rn(acc[rr][1], mul_rn(d1, d1));
            }
        }
        cta_sync();
    }
    double vals[8][2];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
        const long long li = i0 + ty + 8 * rr;
        const long long gi = row0 + li;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long j = j0 + tx + 32 * h;
            double val;
            if (gram && gi == j) val = add_rn(var, jitter);
            else val = mul_rn(var, exp(mul_rn(-acc[rr][h], inv2l2)));
            vals[rr][h] = val;
            if (j < nc && li < rows) out[li * ldo + j] = val;
        }
    }
    if (!mirror || blockIdx.x == blockIdx.y) return;
    // transposed copy through shared memory (the staging buffer is free
    // again): rows of the mirror tile stored coalesced
    double (*tt)[RBF_T + 1] = reinterpret_cast<double (*)[RBF_T + 1]>(sbuf);
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
        tt[ty + 8 * rr][tx] = vals[rr][0];
        tt[ty + 8 * rr][tx + 32] = vals[rr][1];
    }
    cta_sync();
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long orow = j0 + ty + 8 * rr, ocol = i0 + tx + 32 * h;   // K[j][i] = K[i][j]
            if (orow < nc && ocol < rows) out[orow * ldo + ocol] = tt[tx + 32 * h][ty + 8 * rr];
        }
    }
}

// The tiles [t_lo, t_hi) of the packed lower-triangle copy (symgemv.cuh:
// tile-row order, 32 KB per tile, XOR swizzle, zero beyond n) evaluated
// directly from X with rbf_tile_kernel's operation sequence, so every entry
// is bitwise the stored Gram's: a rank's share of a tile-sharded Gram is built
// without the row-major matrix.
__global__ void __launch_bounds__(256)
    rbf_packed_kernel(const double* __restrict__ x, long long n, long long dim, double var, double inv2l2,
                      double jitter, long long t_lo, double* __restrict__ out) {
    __shared__ double sbuf[2 * RBF_T * (RBF_D + 1)];
    double (*sr)[RBF_D + 1] = reinterpret_cast<double (*)[RBF_D + 1]>(sbuf);
    double (*sc)[RBF_D + 1] = reinterpret_cast<double (*)[RBF_D + 1]>(sbuf + RBF_T * (RBF_D + 1));
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const long long t = t_lo + blockIdx.x;
    const long long I = sym_tile_row(t), J = t - sym_tile_row_base(I);
    const long long i0 = I * RBF_T, j0 = J * RBF_T;
    double acc[8][2];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
    for (long long t0 = 0; t0 < dim; t0 += RBF_D) {
        const int tn = (int)min((long long)RBF_D, dim - t0);
        for (int e = threadIdx.x; e < RBF_T * RBF_D; e += 256) {
            const int r = e / RBF_D, c = e % RBF_D;
            sr[r][c] = (c < tn && i0 + r < n) ? x[(i0 + r) * dim + t0 + c] : 0.0;
            sc[r][c] = (c < tn && j0 + r < n) ? x[(j0 + r) * dim + t0 + c] : 0.0;
        }
        cta_sync();
        for (int c = 0; c < tn; ++c) {
            const double c0 = sc[tx][c], c1 = sc[tx + 32][c];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const double rv = sr[ty + 8 * rr][c];
                const double d0 = sub_rn(rv, c0), d1 = sub_rn(rv, c1);
                acc[rr][0] = add_rn(acc[rr][0], mul_rn(d0, d0));
                acc[rr][1] = add_rn(acc[rr][1], mul_rn(d1, d1));
            }
        }
        cta_sync();
    }
    double* dst = out + (t - t_lo) * (RBF_T * RBF_T);
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
        const int r = ty + 8 * rr;
        const long long gi = i0 + r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = tx + 32 * h;
            const long long j = j0 + c;
            double val = 0.0;
            if (gi < n && j < n) val = gi == j ? add_rn(var, jitter) : mul_rn(var, exp(mul_rn(-acc[rr][h], inv2l2)));
            dst[sym_swz(r, c)] = val;
        }
    }
}

int dcg_rbf_packed_launch(cudaStream_t st, const double* x, long long n, long long dim, double var, double inv2l2,
                          double jitter, long long t_lo, long long t_hi, double* out) {
    if (t_hi <= t_lo) return DCG_OK;
    if (t_hi - t_lo > 0x7fffffffLL) return DCG_E_UNSUPPORTED;
    rbf_packed_kernel<<<(unsigned)(t_hi - t_lo), 256, 0, st>>>(x, n, dim, var, inv2l2, jitter, t_lo, out);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_rbf_launch(cudaStream_t st, const double* xr, long long nr_total, const double* xc, long long nc,
                   long long dim, double var, double inv2l2, double jitter, int gram, long long row0,
                   long long rows, double* out, long long ldo) {
    if (rows <= 0 || nc <= 0) return DCG_OK;
    dim3 grid((unsigned)((nc + RBF_T - 1) / RBF_T), (unsigned)((rows + RBF_T - 1) / RBF_T));
    rbf_tile_kernel<<<grid, 256, 0, st>>>(xr, nr_total, xc, nc, dim, var, inv2l2, jitter, gram, row0, rows,
                                          out, ldo);
    DCG_LAUNCHED();
    return DCG_OK;
}

// ----------------------------------------------------------------------------
// logistic likelihood pieces (gpc.py:126-157)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double sigmoid_ref(double z) {
    if (z >= 0.0) return div_rn(1.0, add_rn(1.0, exp(-z)));
    const double ez = exp(z);
    return div_rn(ez, add_rn(1.0, ez));
}

// numpy logaddexp(0, z)
__device__ __forceinline__ double logaddexp0(double z) {
    const double x = 0.0;
    if (x == z) return x + 0.69314718055994530942;
    const double tmp = x - z;
    if (tmp > 0.0) return add_rn(x, log1p(exp(-tmp)));
    if (tmp <= 0.0) return add_rn(z, log1p(exp(tmp)));
    return tmp;   // NaN
}

__device__ void derivs_finalize_body(const double* part, int nb, DevStatus* st, double* llpsi);

// grad/h for f; per-CTA partials of  -sum logaddexp(0, -y f)  and  f'a (a may be NULL).
// With `last` (the context's persistent counter) the last CTA to finish also
// runs the finalisation (derivs_finalize_kernel's thread split and sums: the
// same values), one launch instead of two.
__global__ void derivs_kernel(long long n, const double* f, const double* y, const double* a, double* grad,
                              double* h, double* part, unsigned int* last, DevStatus* st, double* llpsi) {
    __shared__ double red[40];
    double ll = 0.0, fa = 0.0, bad = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double fi = f[i], yi = y[i];
        if (yi != 1.0 && yi != -1.0) bad += 1.0;   // gpc.py:135-139 (counted, reported by dcg_gpc_init)
        ll += logaddexp0(mul_rn(-yi, fi));
        const double pi = sigmoid_ref(fi);
        grad[i] = sub_rn(mul_rn(add_rn(yi, 1.0), 0.5), pi);
        h[i] = mul_rn(pi, sigmoid_ref(-fi));
        if (a) fa = fma(fi, a[i], fa);
    }
    ll = block_sum(ll, red);
    fa = block_sum(fa, red);
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ll;
        part[2 * blockIdx.x + 1] = fa;
        part[2 * gridDim.x + blockIdx.x] = bad;
    }
    if (!last) return;
    if (cta_last_arrival(last, gridDim.x)) derivs_finalize_body(part, gridDim.x, st, llpsi);
}

__device__ void derivs_finalize_body(const double* part, int nb, DevStatus* st, double* llpsi) {
    __shared__ double red[40];
    double ll = 0.0, fa = 0.0, bad = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        ll += ld_cg(part + 2 * b);
        fa += ld_cg(part + 2 * b + 1);
        bad += ld_cg(part + 2 * nb + b);
    }
    ll = block_sum(ll, red);
    fa = block_sum(fa, red);
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) {
        const double loglik = -ll;
        st->status = DCG_OK;
        st->info = (long long)bad;   // labels not in {-1, +1}
        st->value = loglik;
        st->value2 = sub_rn(loglik, mul_rn(0.5, fa));   // psi = loglik - f'a/2 (gpc.py:209)
        if (llpsi) {
            llpsi[0] = st->value;
            llpsi[1] = st->value2;
        }
    }
}

__global__ void derivs_finalize_kernel(const double* part, int nb, DevStatus* st, double* llpsi) {
    derivs_finalize_body(part, nb, st, llpsi);
}

// s = sqrt(h); inner = h f + grad   (gpc.py:177,181)
__global__ void newton_prep_kernel(long long n, const double* f, const double* grad, const double* h, double* s,
                                   double* inner) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        s[i] = sqrt(h[i]);
        inner[i] = add_rn(mul_rn(h[i], f[i]), grad[i]);
    }
}

// newton_prep plus xs = s (.) x_prev, the operand of the next solve's first
// product A x_prev (formed as the symmetric product stages it: s_j * x_j)
__global__ void newton_prep2_kernel(long long n, const double* f, const double* grad, const double* h,
                                    const double* x, double* s, double* inner, double* xs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double si = sqrt(h[i]);
        s[i] = si;
        inner[i] = add_rn(mul_rn(h[i], f[i]), grad[i]);
        xs[i] = mul_rn(si, x[i]);
    }
}

// a = inner - s x   (gpc.py:190)
__global__ void newton_a_kernel(long long n, const double* inner, const double* s, const double* x, double* a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        a[i] = sub_rn(inner[i], mul_rn(s[i], x[i]));
}

int dcg_derivs_launch(dcg_context* ctx, cudaStream_t st, long long n, const double* f, const double* y,
                      const double* a, double* grad, double* h, double* part, DevStatus* ds, double* llpsi) {
    int nb = ctx->sm_count * 2;
    if ((long long)nb * 256 > n) nb = (int)max(1LL, (n + 255) / 256);
    // partials, then the finalisation by the last CTA (its arrival counter:
    // the context's persistent line, reset by that CTA)
    derivs_kernel<<<nb, 256, 0, st>>>(n, f, y, a, grad, h, part, dcg_sync_line(ctx, DCG_SW_DERIVS), ds, llpsi);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_newton_prep_launch(dcg_context* ctx, cudaStream_t st, long long n, const double* f, const double* grad,
                           const double* h, double* s, double* inner) {
    newton_prep_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(n, f, grad, h, s, inner);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_newton_prep2_launch(dcg_context* ctx, cudaStream_t st, long long n, const double* f, const double* grad,
                            const double* h, const double* x, double* s, double* inner, double* xs) {
    newton_prep2_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(n, f, grad, h, x, s, inner, xs);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_newton_a_launch(dcg_context* ctx, cudaStream_t st, long long n, const double* inner, const double* s,
                        const double* x, double* a) {
    newton_a_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(n, inner, s, x, a);
    DCG_LAUNCHED();
    return DCG_OK;
}
