// Row-sharded def-CG building blocks (include/defcg_b200.h L5).
//
// One process per GPU owns a contiguous slab of K's rows and the same rows of
// every n-vector.  The iteration of _run_loop (solvers.py:131-204) is split at
// its two reductions; the caller runs the collectives (all-gather of p,
// all-reduce of the p'Ap partial, all-reduce of [r'r, AW'r]) between these
// kernels.  Scalars live in a device-resident dcg_shard_state: every kernel
// reads it at entry, and only the last CTA to arrive (after every CTA has read
// it) writes it, so kernels enqueued after convergence are no-ops and ranks
// never diverge.  All reductions are fixed-order.
#include "common.cuh"
#include "gemv.cuh"

#define SH_NT 512

int dcg_rbf_mf_check(const dcg_operator* op);
int dcg_rbf_rows_product(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* X, int k,
                         const double* s_in, const double* s_out, double shift, double* Y,
                         const dcg_shard_state* gate);

namespace {

int shard_grid(const dcg_context* ctx, long long rows) {
    long long g = (rows + SH_NT - 1) / SH_NT;
    if (g > ctx->sm_count) g = ctx->sm_count;
    return g < 1 ? 1 : (int)g;
}
int slot_stride(int k) { return ((1 + k) + 1) & ~1; }

// workspace: G x ps CTA partials + a 16-byte arrival counter (zero between uses)
struct ShardWs {
    double* parts;
    unsigned int* counter;
};
int shard_ws(dcg_context* ctx, cudaStream_t st, int G, int ps, ShardWs* w) {
    const size_t bytes = al(sizeof(double) * (size_t)G * ps) + 256;
    int rc = dcg_ws_reserve(ctx, bytes);
    if (rc) return rc;
    char* base = static_cast<char*>(ctx->ws);
    w->parts = reinterpret_cast<double*>(base);
    // the arrival counter is one of the context's persistent words: the last
    // CTA to arrive returns it to zero (cta_last_arrival), so no memset per launch
    w->counter = dcg_sync_line(ctx, DCG_SW_SHARD);
    (void)st;
    return DCG_OK;
}

// Per-CTA partials over rows [r0, r1): slot 0 = sum_i u_i^2 (thread per row),
// slot 1 + j = sum_i M[i][j] w_i ((row group, j) threads, coalesced rows of M).
// Result in out[0..k] (shared), all threads call.
__device__ void cta_row_partials(long long r0, long long r1, int k, const double* u, const double* w,
                                 const double* M, double* out, double* s_scr, double* s_tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double sq = 0.0;
    if (u)
        for (long long i = r0 + tid; i < r1; i += SH_NT) sq = add_rn(sq, mul_rn(u[i], u[i]));
    int swk = 1;
    while (swk < k) swk <<= 1;
    double c = 0.0;
    if (k > 0) {
        const int j = tid & (swk - 1), grp = tid / swk, ngrp = SH_NT / swk;
        if (j < k) {
            // thirty-two rows' loads ahead of their in-order FMAs (a warp reads one
            // row of M per load; a load per FMA was ~11 us at 510 rows x 32 columns)
            for (long long i = r0 + grp; i < r1; i += 32LL * ngrp) {
                double m[32], ww[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const long long ii = i + (long long)u * ngrp;
                    m[u] = ii < r1 ? __ldg(M + ii * k + j) : 0.0;
                    ww[u] = ii < r1 ? w[ii] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 32; ++u)
                    if (i + (long long)u * ngrp < r1) c = fma(m[u], ww[u], c);
            }
        }
        if (swk < 32)
            for (int o = swk; o < 32; o <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    sq = warp_sum(sq);
    if (lane == 0) s_tmp[warp] = sq;
    if (k > 0) {
        if (swk <= 32) {
            if (lane < swk) s_scr[warp * 32 + lane] = c;
        } else {
            s_scr[tid] = c;
        }
    }
    cta_sync();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < SH_NT / 32; ++q) t += s_tmp[q];
        out[0] = t;
    }
    if (tid < k) {
        double t = 0.0;
        if (swk <= 32) {
            for (int q = 0; q < SH_NT / 32; ++q) t += s_scr[q * 32 + tid];
        } else {
            for (int g = 0; g < SH_NT / swk; ++g) t += s_scr[g * swk + tid];
        }
        out[1 + tid] = t;
    }
    cta_sync();
}

// Sum of G per-CTA partials parts[b * stride], b = 0..G-1, in a FIXED order
// that is not one long chain: eight interleaved running sums (b mod 8), the
// loads of each batch of 32 issued ahead of their adds, then a pairwise
// combination.  One thread; every kernel of this file that sums per-CTA
// partials uses it, so the fused step and the three separate launches still
// agree bit for bit.  (148 dependent DADDs were ~2.8 us on every kernel's tail.)
__device__ __forceinline__ double ordered_sum(const double* parts, long long stride, int G) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int b0 = 0; b0 < G; b0 += 32) {
        double q[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) q[u] = (b0 + u < G) ? ld_cg(parts + (long long)(b0 + u) * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < 32; ++u)
            if (b0 + u < G) acc[u & 7] += q[u];
    }
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// Publish this CTA's nslots values, then the last CTA to arrive sums all CTAs'
// values in CTA order into out[0..nslots).  Returns true on the last CTA.
__device__ bool grid_reduce_slots(const double* mine, int nslots, double* parts, int ps, unsigned int* counter,
                                  double* out) {
    for (int v = threadIdx.x; v < nslots; v += blockDim.x) parts[(long long)blockIdx.x * ps + v] = mine[v];
    const bool last = cta_last_arrival(counter, gridDim.x);
    if (last) {
        for (int v = threadIdx.x; v < nslots; v += blockDim.x) out[v] = ordered_sum(parts + v, ps, (int)gridDim.x);
    }
    return last;
}

// mu = L^-T L^-1 c by warp 0 (forward substitution in the reference order,
// backward sweep as a wavefront), then a CTA barrier.  L in shared memory.
// Pivots are applied as reciprocals 1 / L_jj formed once per call (at most one
// extra rounding per unknown, as in the single-GPU solve kernel, solve.cu):
// a serial FP64 division per unknown is ~100 cycles on the dependent chain.
__device__ void cta_chol_solve(const double* L, int k, const double* c, double* mu) {
    __shared__ double s_rd[DCG_MAX_K];
    for (int j = threadIdx.x; j < k; j += blockDim.x) s_rd[j] = 1.0 / L[j * k + j];
    cta_sync();
    if ((threadIdx.x >> 5) == 0) {
        const int lane = threadIdx.x & 31;
        const int i0 = lane, i1 = lane + 32;
        double a0 = (i0 < k) ? c[i0] : 0.0;
        double a1 = (i1 < k) ? c[i1] : 0.0;
        for (int j = 0; j < k; ++j) {
            const double accj = __shfl_sync(0xffffffffu, (j < 32) ? a0 : a1, j & 31);
            const double yj = mul_rn(accj, s_rd[j]);
            if (lane == (j & 31)) {
                if (j < 32) a0 = yj; else a1 = yj;
            }
            if (i0 > j && i0 < k) a0 = sub_rn(a0, mul_rn(L[i0 * k + j], yj));
            if (i1 > j && i1 < k) a1 = sub_rn(a1, mul_rn(L[i1 * k + j], yj));
        }
        for (int j = k - 1; j >= 0; --j) {
            const double accj = __shfl_sync(0xffffffffu, (j < 32) ? a0 : a1, j & 31);
            const double xj = mul_rn(accj, s_rd[j]);
            if (lane == (j & 31)) {
                if (j < 32) a0 = xj; else a1 = xj;
            }
            if (i0 < j) a0 = sub_rn(a0, mul_rn(L[j * k + i0], xj));
            if (i1 < j && i1 < k) a1 = sub_rn(a1, mul_rn(L[j * k + i1], xj));
        }
        if (i0 < k) mu[i0] = a0;
        if (i1 < k) mu[i1] = a1;
    }
    cta_sync();
}

// sum_j M[i][j] v[j] in ascending j; the row's loads are issued eight ahead of
// their FMAs, sixteen while the row lasts (16-byte loads when the row allows
// it): one L2 latency per batch instead of one per term
__device__ __forceinline__ double row_dot(const double* M, long long i, int k, const double* v) {
    const double* row = M + i * k;
    double t = 0.0;
    int j = 0;
    if ((k & 1) == 0 && (reinterpret_cast<uintptr_t>(M) & 15) == 0) {
        for (; j + 32 <= k; j += 32) {
            double2 m[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) m[u] = __ldg(reinterpret_cast<const double2*>(row + j) + u);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                t = fma(m[u].x, v[j + 2 * u], t);
                t = fma(m[u].y, v[j + 2 * u + 1], t);
            }
        }
        for (; j + 16 <= k; j += 16) {
            double2 m[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) m[u] = __ldg(reinterpret_cast<const double2*>(row + j) + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                t = fma(m[u].x, v[j + 2 * u], t);
                t = fma(m[u].y, v[j + 2 * u + 1], t);
            }
        }
        for (; j + 8 <= k; j += 8) {
            double2 m[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = __ldg(reinterpret_cast<const double2*>(row + j) + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                t = fma(m[u].x, v[j + 2 * u], t);
                t = fma(m[u].y, v[j + 2 * u + 1], t);
            }
        }
    }
    for (; j < k; ++j) t = fma(__ldg(row + j), v[j], t);
    return t;
}

// ---- GEMV over the slab with two epilogues --------------------------------
// mode 0: out_i = (A v)_i and a p'Ap partial; mode 1: out_i = b_i - (A v)_i.
__global__ void __launch_bounds__(DCG_NT, 1)
    shard_gemv_kernel(int mode, const double* __restrict__ K, long long ldk, long long n, long long rows,
                      long long row0, const double* v, const double* s, double shift, const double* b, double* out,
                      double* part, double* parts, int ps, unsigned int* counter, const dcg_shard_state* state) {
    extern __shared__ __align__(16) double smem[];
    if (state && state->done) return;
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    const int xt = (int)min(n, (long long)DCG_QT) + 2;
    double* s_x = smem;
    double* s_red = smem + xt;
    __shared__ double s_tmp[40];
    __shared__ double s_out[2];
    double dot = 0.0;
    block_gemv<true>(K, ldk, n, v, s, r0, r1, s_x, s_red, [&](long long i, double t) {
        const long long g = row0 + i;
        const double vi = ld_cg(v + g);
        const double ax = s ? add_rn(mul_rn(shift, vi), mul_rn(s[g], t)) : add_rn(mul_rn(shift, vi), t);
        if (mode == 0) {
            out[i] = ax;
            dot = fma(vi, ax, dot);
        } else {
            out[i] = sub_rn(b[i], ax);
        }
    });
    if (mode == 0 && part) {
        dot = block_sum(dot, s_tmp);
        if (threadIdx.x == 0) s_out[0] = dot;
        cta_sync();
        grid_reduce_slots(s_out, 1, parts, ps, counter, part);
    }
}

// RBF slabs: `out` already holds t = K_slab (s (.) v) (dcg_rbf_rows_product);
// the same epilogues as shard_gemv_kernel, in place.
__global__ void __launch_bounds__(DCG_NT, 1)
    shard_rbf_epi_kernel(int mode, long long rows, long long row0, const double* v, const double* s, double shift,
                         const double* b, const double* t_rows, double* out, double* part, double* parts, int ps,
                         unsigned int* counter, const dcg_shard_state* state) {
    if (state && state->done) return;
    __shared__ double s_tmp[40];
    __shared__ double s_out[2];
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    double dot = 0.0;
    for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const long long g = row0 + i;
        const double t = t_rows ? ld_cg(t_rows + i) : out[i];
        const double vi = ld_cg(v + g);
        const double ax = s ? add_rn(mul_rn(shift, vi), mul_rn(s[g], t)) : add_rn(mul_rn(shift, vi), t);
        if (mode == 0) {
            out[i] = ax;
            dot = fma(vi, ax, dot);
        } else {
            out[i] = sub_rn(b[i], ax);
        }
    }
    if (mode == 0 && part) {
        dot = block_sum(dot, s_tmp);
        if (threadIdx.x == 0) s_out[0] = dot;
        cta_sync();
        grid_reduce_slots(s_out, 1, parts, ps, counter, part);
    }
}

size_t shard_gemv_smem(long long n) { return sizeof(double) * ((size_t)min(n, (long long)DCG_QT) + 2 + DCG_NW * DCG_RB); }

__global__ void __launch_bounds__(SH_NT)
    shard_partials_kernel(long long rows, int k, const double* u, const double* w, const double* M, double* part,
                          double* parts, int ps, unsigned int* counter) {
    __shared__ double s_scr[SH_NT];
    __shared__ double s_tmp[40];
    __shared__ double s_out[DCG_MAX_K + 2];
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    cta_row_partials(r0, r1, k, u, w, M, s_out, s_scr, s_tmp);
    grid_reduce_slots(s_out, 1 + k, parts, ps, counter, part);
}

__global__ void __launch_bounds__(SH_NT)
    shard_start_kernel(long long rows, int k, const double* red, const double* Lg, const double* W,
                       const double* xprev, double* x0, dcg_shard_state* state, double tol, long long max_iters,
                       long long ell, const double* AW = nullptr, double* r = nullptr) {
    __shared__ double s_L[DCG_MAX_K * DCG_MAX_K];
    __shared__ double s_y[DCG_MAX_K];
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    if (k > 0) {
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) s_L[e] = Lg[e];
        cta_sync();
        cta_chol_solve(s_L, k, red + 1, s_y);
    }
    for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        x0[i] = k > 0 ? add_rn(xprev[i], row_dot(W, i, k, s_y)) : xprev[i];
        // r0 = r_prev - (AW) c: A x0 = A x_prev + (A W) c with the basis' own AW
        // (the single-GPU solve's warm start, solve.cu): no second product
        if (r && k > 0) r[i] = sub_rn(r[i], row_dot(AW, i, k, s_y));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        state->rr = 0.0;
        state->norm_b = sqrt(red[0]);
        state->rel = 0.0;
        state->alpha = state->beta = state->d = 0.0;
        state->tol = tol;
        state->it = 0;
        state->max_iters = max_iters;
        state->done = 0;
        state->status = DCG_OK;
        state->info = 0;
        state->ell = ell;
    }
}

__global__ void __launch_bounds__(SH_NT)
    shard_begin_kernel(long long rows, int k, const double* red, const double* Lg, const double* W, const double* r,
                       double* p, double* x, dcg_shard_state* state, double* history, double* log_r, double* log_p,
                       double* log_mu, unsigned int* counter) {
    __shared__ double s_L[DCG_MAX_K * DCG_MAX_K];
    __shared__ double s_mu[DCG_MAX_K];
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    const double norm_b = state->norm_b;
    const long long ell = state->ell, max_iters = state->max_iters;
    const double tol = state->tol;
    const double rr = red[0];
    bool zero = norm_b == 0.0;
    const double rel = zero ? 0.0 : sqrt(rr) / norm_b;
    const bool cont = !zero && rel > tol && 0 < max_iters;
    if (zero) {
        // solvers.py:142-147: x = zeros (not x0), history [0.0], log.r = [zeros]
        for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            x[i] = 0.0;
            if (log_r) log_r[i] = 0.0;
        }
    } else {
        if (k > 0) {
            for (int e = threadIdx.x; e < k * k; e += blockDim.x) s_L[e] = Lg[e];
            cta_sync();
            cta_chol_solve(s_L, k, red + 1, s_mu);
        }
        for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            const double ri = r[i];
            const double pi = k > 0 ? sub_rn(ri, row_dot(W, i, k, s_mu)) : ri;
            p[i] = pi;
            if (log_r) log_r[i] = ri;
            if (cont && ell > 0 && log_p) log_p[i] = pi;
        }
    }
    if (cta_last_arrival(counter, gridDim.x) && threadIdx.x == 0) {
        state->rr = rr;
        state->rel = rel;
        state->done = cont ? 0 : 1;
        history[0] = rel;
        if (cont && ell > 0 && k > 0 && log_mu)
            for (int j = 0; j < k; ++j) log_mu[j] = s_mu[j];
    }
}

__global__ void __launch_bounds__(SH_NT)
    shard_update_kernel(int mode, long long rows, int k, const double* red_d, double* x, double* r, const double* p,
                        const double* ap, const double* AW, double* part, dcg_shard_state* state, double* log_r,
                        double* log_d, double* log_alpha, double* parts, int ps, unsigned int* counter) {
    __shared__ double s_scr[SH_NT];
    __shared__ double s_tmp[40];
    __shared__ double s_out[DCG_MAX_K + 2];
    if (state->done) return;
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    const long long it = state->it, ell = state->ell;
    const long long n_loc = rows;
    if (mode != 2) {
        const double d = red_d[0];
        if (!(d > 0.0) && !(d != d)) {   // solvers.py:170-172: d <= 0 (NaN falls through, as in numpy)
            if (cta_last_arrival(counter, gridDim.x) && threadIdx.x == 0) {
                state->status = DCG_E_BREAKDOWN;
                state->info = it;
                state->done = 1;
            }
            return;
        }
        const double alpha = state->rr / d;
        for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            x[i] = add_rn(x[i], mul_rn(alpha, p[i]));
            if (mode == 0) r[i] = sub_rn(r[i], mul_rn(alpha, ap[i]));
        }
        if (mode == 1) {
            if (cta_last_arrival(counter, gridDim.x) && threadIdx.x == 0) {
                state->alpha = alpha;
                state->d = d;
                state->it = it + 1;
                if (it < ell) {
                    log_d[it] = d;
                    log_alpha[it] = alpha;
                }
            }
            return;
        }
        cta_sync();
        const bool log = log_r && it < ell;   // (it + 1) - 1 < ell
        if (log)
            for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) log_r[(it + 1) * n_loc + i] = r[i];
        cta_row_partials(r0, r1, k, r, r, AW, s_out, s_scr, s_tmp);
        if (grid_reduce_slots(s_out, 1 + k, parts, ps, counter, part) && threadIdx.x == 0) {
            state->alpha = alpha;
            state->d = d;
            state->it = it + 1;
            if (it < ell) {
                log_d[it] = d;
                log_alpha[it] = alpha;
            }
        }
        return;
    }
    // mode 2: r was recomputed as b - A x; `it` already counts this iteration
    const bool log = log_r && (it - 1) < ell;
    if (log)
        for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) log_r[it * n_loc + i] = r[i];
    cta_row_partials(r0, r1, k, r, r, AW, s_out, s_scr, s_tmp);
    grid_reduce_slots(s_out, 1 + k, parts, ps, counter, part);
}

__global__ void __launch_bounds__(SH_NT)
    shard_direction_kernel(long long rows, int k, const double* red, const double* Lg, const double* W,
                           const double* r, double* p, dcg_shard_state* state, double* history, double* log_p,
                           double* log_mu, double* log_beta, unsigned int* counter) {
    __shared__ double s_L[DCG_MAX_K * DCG_MAX_K];
    __shared__ double s_mu[DCG_MAX_K];
    if (state->done) return;
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    const long long it = state->it, ell = state->ell, max_iters = state->max_iters;
    const double rr_new = red[0];
    const double beta = rr_new / state->rr;
    const double rel = sqrt(rr_new) / state->norm_b;
    const bool cont = (rel > state->tol) && (it < max_iters);
    const bool log_pn = cont && it < ell && log_p;
    if (k > 0) {
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) s_L[e] = Lg[e];
        cta_sync();
        cta_chol_solve(s_L, k, red + 1, s_mu);
    }
    for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const double ri = r[i];
        const double pi = k > 0 ? sub_rn(add_rn(mul_rn(beta, p[i]), ri), row_dot(W, i, k, s_mu))   // beta*p + r - W mu
                                : add_rn(ri, mul_rn(beta, p[i]));                                  // r + beta*p
        p[i] = pi;
        if (log_pn) log_p[it * rows + i] = pi;
    }
    if (cta_last_arrival(counter, gridDim.x) && threadIdx.x == 0) {
        history[it] = rel;
        if (it - 1 < ell && log_beta) log_beta[it - 1] = beta;
        if (log_pn && k > 0 && log_mu)
            for (int j = 0; j < k; ++j) log_mu[it * k + j] = s_mu[j];
        state->rr = rr_new;
        state->beta = beta;
        state->rel = rel;
        state->done = cont ? 0 : 1;
    }
}

// ---------------------------------------------------------------------------
// One def-CG iteration's vector phases in ONE cooperative launch (replicated
// vectors: the tile-share path, where the all-reduced t = K (s (.) p) is the
// only exchange of the iteration): the epilogue Ap = shift p + s (.) t and
// p'Ap, [grid barrier] alpha, x, r, [r'r, AW'r], [grid barrier] beta, mu, p --
// the work of dcg_shard_epilogue(0) + dcg_shard_update(0) +
// dcg_shard_direction in one launch (~50 -> ~20 us at n = 5 10^4, k = 32).
// Every CTA reduces the per-CTA partials itself in CTA order (the order of
// grid_reduce_slots), so all CTAs -- and all ranks, whose t is bitwise the
// same -- hold the same scalars.  The state is read by every CTA before the
// first barrier and written by CTA 0 after the second.
// ---------------------------------------------------------------------------
struct StepArgs {
    long long rows;
    int k, ps;
    const double* t;
    const double* s;
    double shift;
    double *x, *r, *p, *ap;
    const double *W, *AW, *Lg;
    dcg_shard_state* state;
    double* history;
    double *log_r, *log_p, *log_d, *log_alpha, *log_beta, *log_mu;
    double* parts;        // G x ps
    double* dparts;       // gepi p'Ap partials
    int gepi;             // CTAs of dcg_shard_epilogue's row partition
    unsigned int* bar;    // the context's persistent barrier line
    unsigned long long* timers;   // optional (DCG_STEP_TIMERS): ns per phase, CTA 0 / thread 0
};

// ordered_sum's arithmetic on values already staged in shared memory
__device__ __forceinline__ double ordered_sum_staged(const double* vals, int stride, int G) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    int b = 0;
    for (; b + 8 <= G; b += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += vals[(b + u) * stride];
    }
    for (int u = 0; b + u < G; ++u) acc[u] += vals[(b + u) * stride];
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// out[v] = ordered sum over the G CTAs of parts[b * stride + v], v < nslots, by
// every CTA: all threads stage the G x stride block in shared memory with one
// round of loads (a thread per slot loading its own column took four L2
// round trips), then a thread per slot sums its column -- ordered_sum's values.
__device__ __forceinline__ void step_reduce(const double* parts, int stride, int G, int nslots, double* out,
                                            double* stage) {
    const int total = G * stride;
    for (int e = threadIdx.x; e < total; e += blockDim.x) stage[e] = ld_cg(parts + e);
    cta_sync();
    for (int v = threadIdx.x; v < nslots; v += blockDim.x) out[v] = ordered_sum_staged(stage + v, stride, G);
    cta_sync();
}

__global__ void __launch_bounds__(SH_NT) shard_step_kernel(StepArgs a) {
    __shared__ double s_scr[SH_NT];
    __shared__ double s_tmp[40];
    __shared__ double s_out[DCG_MAX_K + 2];
    __shared__ double s_red[DCG_MAX_K + 2];
    __shared__ double s_L[DCG_MAX_K * DCG_MAX_K];
    __shared__ double s_mu[DCG_MAX_K];
    extern __shared__ __align__(16) double s_stage[];   // max(G x ps, gepi) doubles
    unsigned long long t_mark = 0;
#define STEP_PHASE(id)                                                    \
    do {                                                                  \
        if (a.timers && blockIdx.x == 0 && threadIdx.x == 0) {            \
            const unsigned long long t_ = globaltimer_ns();               \
            if (t_mark) a.timers[id] += t_ - t_mark;                       \
            t_mark = t_;                                                  \
        }                                                                 \
    } while (0)
    STEP_PHASE(15);
    const dcg_shard_state st = *a.state;   // every CTA reads the state before the first barrier
    if (st.done) return;                   // uniform: nobody arrives at a barrier
    const int k = a.k, tid = threadIdx.x;
    const long long rows = a.rows;
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x), r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    const long long it = st.it, ell = st.ell;
    if (k > 0)
        for (int e = tid; e < k * k; e += blockDim.x) s_L[e] = a.Lg[e];
    // ---- Ap and the p'Ap partials: over the epilogue kernel's row partition
    // (a.gepi virtual CTAs, taken blockIdx.x, + gridDim.x, ...), so that d is
    // bitwise the three-launch path's
    for (int vb = blockIdx.x; vb < a.gepi; vb += gridDim.x) {
        const long long e0 = part_begin(rows, a.gepi, vb), e1 = part_begin(rows, a.gepi, vb + 1);
        double dot = 0.0;
        for (long long i = e0 + tid; i < e1; i += blockDim.x) {
            const double ti = ld_cg(a.t + i);
            const double pi = a.p[i];
            const double ax = a.s ? add_rn(mul_rn(a.shift, pi), mul_rn(a.s[i], ti)) : add_rn(mul_rn(a.shift, pi), ti);
            a.ap[i] = ax;
            dot = fma(pi, ax, dot);
        }
        dot = block_sum(dot, s_tmp);
        if (tid == 0) a.dparts[vb] = dot;
    }
    STEP_PHASE(0);
    dcg_grid_barrier(a.bar, gridDim.x);
    STEP_PHASE(1);
    {
        // sum of the a.gepi partials (ordered_sum, as the epilogue kernel's last CTA), by every CTA
        step_reduce(a.dparts, 1, a.gepi, 1, s_red, s_stage);
    }
    const double d = s_red[0];
    STEP_PHASE(2);
    if (!(d > 0.0) && !(d != d)) {   // solvers.py:170-172: d <= 0 (NaN falls through, as in numpy)
        if (blockIdx.x == 0 && tid == 0) {
            a.state->status = DCG_E_BREAKDOWN;
            a.state->info = it;
            a.state->done = 1;
        }
        if (tid == 0) dcg_sync_exit(a.bar, gridDim.x);
        return;
    }
    const double alpha = st.rr / d;
    // ---- x, r and [r'r, AW'r] -----------------------------------------------
    const bool log = a.log_r && it < ell;
    for (long long i = r0 + tid; i < r1; i += blockDim.x) {
        a.x[i] = add_rn(a.x[i], mul_rn(alpha, a.p[i]));
        const double ri = sub_rn(a.r[i], mul_rn(alpha, ld_cg(a.ap + i)));   // (another CTA's epilogue rows)
        a.r[i] = ri;
        if (log) a.log_r[(it + 1) * rows + i] = ri;
    }
    cta_sync();
    STEP_PHASE(3);
    cta_row_partials(r0, r1, k, a.r, a.r, a.AW, s_out, s_scr, s_tmp);
    cta_sync();   // (x / r loop readers of ap; s_red's d has been read by everyone)
    STEP_PHASE(4);
    for (int v = tid; v < 1 + k; v += blockDim.x) a.parts[(long long)blockIdx.x * a.ps + v] = s_out[v];
    dcg_grid_barrier(a.bar, gridDim.x);
    STEP_PHASE(5);
    step_reduce(a.parts, a.ps, (int)gridDim.x, 1 + k, s_red, s_stage);
    STEP_PHASE(6);
    // ---- beta, mu, p -----------------------------------------------------------
    const long long itn = it + 1;
    const double rr_new = s_red[0];
    const double beta = rr_new / st.rr;
    const double rel = sqrt(rr_new) / st.norm_b;
    const bool cont = (rel > st.tol) && (itn < st.max_iters);
    const bool log_pn = cont && itn < ell && a.log_p;
    if (k > 0) cta_chol_solve(s_L, k, s_red + 1, s_mu);
    STEP_PHASE(7);
    for (long long i = r0 + tid; i < r1; i += blockDim.x) {
        const double ri = a.r[i];
        const double pi = k > 0 ? sub_rn(add_rn(mul_rn(beta, a.p[i]), ri), row_dot(a.W, i, k, s_mu))   // beta*p + r - W mu
                                : add_rn(ri, mul_rn(beta, a.p[i]));                                    // r + beta*p
        a.p[i] = pi;
        if (log_pn) a.log_p[itn * rows + i] = pi;
    }
    STEP_PHASE(8);
    if (blockIdx.x == 0 && tid == 0) {
        if (it < ell && a.log_d) {
            a.log_d[it] = d;
            a.log_alpha[it] = alpha;
        }
        a.history[itn] = rel;
        if (itn - 1 < ell && a.log_beta) a.log_beta[itn - 1] = beta;
        if (log_pn && k > 0 && a.log_mu)
            for (int j = 0; j < k; ++j) a.log_mu[itn * k + j] = s_mu[j];
        a.state->alpha = alpha;
        a.state->d = d;
        a.state->it = itn;
        a.state->rr = rr_new;
        a.state->beta = beta;
        a.state->rel = rel;
        a.state->done = cont ? 0 : 1;
    }
    if (tid == 0) dcg_sync_exit(a.bar, gridDim.x);
}

int check_slab(const dcg_operator* op) {
    if (!op || op->kind != DCG_OP_DENSE) return DCG_E_CONFIG;
    if (op->n < 0 || op->row0 < 0 || op->rows < 0 || op->row0 + op->rows > op->n) return DCG_E_CONFIG;
    if (op->ldk < op->n || (op->ldk & 1) || !aligned16(op->d_k)) return DCG_E_CONFIG;
    return DCG_OK;
}

int launch_gemv(dcg_context* ctx, cudaStream_t st, int mode, const dcg_operator* op, const double* v,
                const double* b, double* out, double* part, const dcg_shard_state* state) {
    if (op && op->kind == DCG_OP_RBF) {
        // matrix-free slab (config 5): the row-owned tensor-pipe product, then
        // the epilogue in place
        int rc = dcg_rbf_mf_check(op);
        if (rc) return rc;
        if (op->rows == 0) return DCG_OK;
        rc = dcg_rbf_rows_product(ctx, st, op, v, 0, op->d_s, nullptr, 0.0, out, state);
        if (rc) return rc;
        long long G = ctx->sm_count;
        if (G > op->rows) G = op->rows;
        ShardWs w;
        rc = shard_ws(ctx, st, (int)G, 2, &w);
        if (rc) return rc;
        shard_rbf_epi_kernel<<<(unsigned)G, DCG_NT, 0, st>>>(mode, op->rows, op->row0, v, op->d_s, op->shift, b,
                                                               nullptr, out, part, w.parts, 2, w.counter, state);
        DCG_LAUNCHED();
        return DCG_OK;
    }
    int rc = check_slab(op);
    if (rc) return rc;
    if (op->rows == 0) return DCG_OK;
    long long G = ctx->sm_count;
    if (G > op->rows) G = op->rows;
    ShardWs w;
    rc = shard_ws(ctx, st, (int)G, 2, &w);
    if (rc) return rc;
    const size_t smem = shard_gemv_smem(op->n);
    DCG_CUDA(cudaFuncSetAttribute(shard_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    shard_gemv_kernel<<<(unsigned)G, DCG_NT, smem, st>>>(mode, op->d_k, op->ldk, op->n, op->rows, op->row0, v,
                                                          op->d_s, op->shift, b, out, part, w.parts, 2, w.counter,
                                                          state);
    DCG_LAUNCHED();
    return DCG_OK;
}

}  // namespace

extern "C" int dcg_shard_apply_dot(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_v,
                                   double* d_out, double* d_part, const dcg_shard_state* d_state) {
    if (!ctx || !d_v || !d_out) return DCG_E_CONFIG;
    return launch_gemv(ctx, as_stream(stream), 0, op, d_v, nullptr, d_out, d_part, d_state);
}

extern "C" int dcg_shard_residual(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_v,
                                  const double* d_b, double* d_r, const dcg_shard_state* d_state) {
    if (!ctx || !d_v || !d_b || !d_r) return DCG_E_CONFIG;
    return launch_gemv(ctx, as_stream(stream), 1, op, d_v, d_b, d_r, nullptr, d_state);
}

// The slab epilogue of a product whose K (s (.) v) arrived by an all-reduce
// (dcg_shard_rbf_sym_partial): mode 0 out = (A v) rows + the p'Ap partial,
// mode 1 out = b - (A v) rows.  d_t is the full-length reduced vector.
extern "C" int dcg_shard_epilogue(dcg_context* ctx, void* stream, int mode, const dcg_operator* op, const double* d_v,
                                  const double* d_b, const double* d_t, double* d_out, double* d_part,
                                  const dcg_shard_state* d_state) {
    if (!ctx || !op || !d_v || !d_t || !d_out || (mode != 0 && mode != 1) || (mode == 1 && !d_b)) return DCG_E_CONFIG;
    if (op->rows == 0) return DCG_OK;
    cudaStream_t st = as_stream(stream);
    long long G = ctx->sm_count;
    if (G > op->rows) G = op->rows;
    ShardWs w;
    int rc = shard_ws(ctx, st, (int)G, 2, &w);
    if (rc) return rc;
    shard_rbf_epi_kernel<<<(unsigned)G, DCG_NT, 0, st>>>(mode, op->rows, op->row0, d_v, op->d_s, op->shift, d_b,
                                                           d_t + op->row0, d_out, mode == 0 ? d_part : nullptr, w.parts,
                                                           2, w.counter, d_state);
    DCG_LAUNCHED();
    return DCG_OK;
}

static unsigned long long* g_step_timers = nullptr;
// Developer diagnostic: ns accumulated per phase of dcg_shard_step by CTA 0 (DCG_STEP_TIMERS=1): epilogue + p'Ap
// partials, barrier, d, x / r, row partials, barrier, reduce, mu, p; slot 15 = unused.
extern "C" __attribute__((visibility("default"))) int dcg_debug_step_timers(unsigned long long* out16) {
    if (!g_step_timers || !out16) return DCG_E_CONFIG;
    DCG_CUDA(cudaMemcpy(out16, g_step_timers, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return DCG_OK;
}

// The vector phases of one iteration on replicated vectors in one cooperative
// launch (see shard_step_kernel): d_t = the all-reduced K (s (.) p) (all rows),
// s / shift the operator's scaling (A = shift I + s K s), logs optional.
extern "C" int dcg_shard_step(dcg_context* ctx, void* stream, long long rows, int k, const double* d_t,
                              const double* d_s, double shift, double* d_x, double* d_r, double* d_p, double* d_ap,
                              const double* d_w, const double* d_aw, const double* d_chol, dcg_shard_state* d_state,
                              double* d_history, double* d_log_r, double* d_log_p, double* d_log_d,
                              double* d_log_alpha, double* d_log_beta, double* d_log_mu) {
    if (!ctx || rows < 0 || k < 0 || !d_t || !d_x || !d_r || !d_p || !d_ap || !d_state || !d_history)
        return DCG_E_CONFIG;
    if (k > 0 && (!d_w || !d_aw || !d_chol)) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    if (d_log_r && (!d_log_d || !d_log_alpha)) return DCG_E_CONFIG;
    if (rows == 0) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const int G = shard_grid(ctx, rows), ps = slot_stride(k);
    long long gepi = ctx->sm_count;   // dcg_shard_epilogue's grid
    if (gepi > rows) gepi = rows;
    const size_t bytes = al(sizeof(double) * (size_t)G * ps) + al(sizeof(double) * (size_t)gepi);
    int rc = dcg_ws_reserve(ctx, bytes);
    if (rc) return rc;
    StepArgs a;
    a.rows = rows;
    a.k = k;
    a.ps = ps;
    a.t = d_t;
    a.s = d_s;
    a.shift = shift;
    a.x = d_x;
    a.r = d_r;
    a.p = d_p;
    a.ap = d_ap;
    a.W = d_w;
    a.AW = d_aw;
    a.Lg = d_chol;
    a.state = d_state;
    a.history = d_history;
    a.log_r = d_log_r;
    a.log_p = d_log_p;
    a.log_d = d_log_d;
    a.log_alpha = d_log_alpha;
    a.log_beta = d_log_beta;
    a.log_mu = d_log_mu;
    a.parts = static_cast<double*>(ctx->ws);
    a.dparts = reinterpret_cast<double*>(static_cast<char*>(ctx->ws) + al(sizeof(double) * (size_t)G * ps));
    a.gepi = (int)gepi;
    a.bar = dcg_sync_line(ctx, DCG_SW_SHARDSTEP);
    // DCG_STEP_TIMERS=1: per-phase device time of CTA 0 accumulated over the calls
    // (developer diagnostic, read with dcg_debug_step_timers)
    static const bool timers = getenv("DCG_STEP_TIMERS") != nullptr;
    a.timers = nullptr;
    if (timers) {
        if (!g_step_timers) {
            DCG_CUDA(cudaMalloc(&g_step_timers, 16 * sizeof(unsigned long long)));
            DCG_CUDA(cudaMemset(g_step_timers, 0, 16 * sizeof(unsigned long long)));
        }
        a.timers = g_step_timers;
    }
    const size_t smem = sizeof(double) * (size_t)((long long)G * ps > gepi ? (long long)G * ps : gepi);
    DCG_SMEM_ATTR(shard_step_kernel, smem);
    void* args[] = {&a};
    DCG_CUDA(cudaLaunchCooperativeKernel((const void*)shard_step_kernel, dim3(G), dim3(SH_NT), args, smem, st));
    DCG_LAUNCHED();
    return DCG_OK;
}

extern "C" int dcg_shard_partials(dcg_context* ctx, void* stream, long long rows, int k, const double* d_u,
                                  const double* d_w, const double* d_m, double* d_part) {
    if (!ctx || rows < 0 || k < 0 || !d_part || (k > 0 && (!d_w || !d_m))) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const int G = shard_grid(ctx, rows), ps = slot_stride(k);
    ShardWs w;
    int rc = shard_ws(ctx, st, G, ps, &w);
    if (rc) return rc;
    shard_partials_kernel<<<G, SH_NT, 0, st>>>(rows, k, d_u, d_w, d_m, d_part, w.parts, ps, w.counter);
    DCG_LAUNCHED();
    return DCG_OK;
}

extern "C" int dcg_shard_start(dcg_context* ctx, void* stream, long long rows, int k, const double* d_red,
                               const double* d_chol, const double* d_w, const double* d_xprev, double* d_x0,
                               dcg_shard_state* d_state, double tol, long long max_iters, long long ell) {
    if (!ctx || rows < 0 || k < 0 || !d_red || !d_xprev || !d_x0 || !d_state) return DCG_E_CONFIG;
    if (k > 0 && (!d_chol || !d_w)) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    shard_start_kernel<<<shard_grid(ctx, rows), SH_NT, 0, st>>>(rows, k, d_red, d_chol, d_w, d_xprev, d_x0, d_state,
                                                                 tol, max_iters, ell);
    DCG_LAUNCHED();
    return DCG_OK;
}

// dcg_shard_start plus r0 = r_prev - (AW) c in place of r (the rank's rows of
// AW; r holds r_prev = b - A x_prev): the warm start without the product
// r0 = b - A x0 (equal up to rounding).
extern "C" int dcg_shard_start_r(dcg_context* ctx, void* stream, long long rows, int k, const double* d_red,
                                 const double* d_chol, const double* d_w, const double* d_aw, const double* d_xprev,
                                 double* d_x0, double* d_r, dcg_shard_state* d_state, double tol, long long max_iters,
                                 long long ell) {
    if (!ctx || rows < 0 || k < 1 || !d_red || !d_xprev || !d_x0 || !d_state || !d_chol || !d_w || !d_aw || !d_r)
        return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    shard_start_kernel<<<shard_grid(ctx, rows), SH_NT, 0, st>>>(rows, k, d_red, d_chol, d_w, d_xprev, d_x0, d_state,
                                                                 tol, max_iters, ell, d_aw, d_r);
    DCG_LAUNCHED();
    return DCG_OK;
}

extern "C" int dcg_shard_begin(dcg_context* ctx, void* stream, long long rows, int k, const double* d_red,
                               const double* d_chol, const double* d_w, const double* d_r, double* d_p, double* d_x,
                               dcg_shard_state* d_state, double* d_history, double* d_log_r, double* d_log_p,
                               double* d_log_mu) {
    if (!ctx || rows < 0 || k < 0 || !d_red || !d_r || !d_p || !d_x || !d_state || !d_history) return DCG_E_CONFIG;
    if (k > 0 && (!d_chol || !d_w)) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const int G = shard_grid(ctx, rows);
    ShardWs w;
    int rc = shard_ws(ctx, st, G, 2, &w);
    if (rc) return rc;
    shard_begin_kernel<<<G, SH_NT, 0, st>>>(rows, k, d_red, d_chol, d_w, d_r, d_p, d_x, d_state, d_history, d_log_r,
                                            d_log_p, d_log_mu, w.counter);
    DCG_LAUNCHED();
    return DCG_OK;
}

extern "C" int dcg_shard_update(dcg_context* ctx, void* stream, int mode, long long rows, int k,
                                const double* d_red_d, double* d_x, double* d_r, const double* d_p,
                                const double* d_ap, const double* d_aw, double* d_part, dcg_shard_state* d_state,
                                double* d_log_r, double* d_log_d, double* d_log_alpha, double* d_log_beta) {
    (void)d_log_beta;
    if (!ctx || rows < 0 || k < 0 || mode < 0 || mode > 2 || !d_x || !d_r || !d_state) return DCG_E_CONFIG;
    if (mode != 2 && (!d_red_d || !d_p)) return DCG_E_CONFIG;
    if (mode == 0 && !d_ap) return DCG_E_CONFIG;
    if (mode != 1 && !d_part) return DCG_E_CONFIG;
    if (k > 0 && !d_aw) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    if (d_log_r && (!d_log_d || !d_log_alpha)) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    const int G = shard_grid(ctx, rows), ps = slot_stride(k);
    ShardWs w;
    int rc = shard_ws(ctx, st, G, ps, &w);
    if (rc) return rc;
    shard_update_kernel<<<G, SH_NT, 0, st>>>(mode, rows, k, d_red_d, d_x, d_r, d_p, d_ap, d_aw, d_part, d_state,
                                             d_log_r, d_log_d, d_log_alpha, w.parts, ps, w.counter);
    DCG_LAUNCHED();
    return DCG_OK;
}

extern "C" int dcg_shard_direction(dcg_context* ctx, void* stream, long long rows, int k, const double* d_red,
                                   const double* d_chol, const double* d_w, const double* d_r, double* d_p,
                                   dcg_shard_state* d_state, double* d_history, double* d_log_p, double* d_log_mu,
                                   double* d_log_beta) {
    if (!ctx || rows < 0 || k < 0 || !d_red || !d_r || !d_p || !d_state || !d_history) return DCG_E_CONFIG;
    if (k > 0 && (!d_chol || !d_w)) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const int G = shard_grid(ctx, rows);
    ShardWs w;
    int rc = shard_ws(ctx, st, G, 2, &w);
    if (rc) return rc;
    shard_direction_kernel<<<G, SH_NT, 0, st>>>(rows, k, d_red, d_chol, d_w, d_r, d_p, d_state, d_history, d_log_p,
                                                d_log_mu, d_log_beta, w.counter);
    DCG_LAUNCHED();
    return DCG_OK;
}
