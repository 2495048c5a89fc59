// Harmonic-Ritz extraction (recycle.py:95-159) and the basis-refresh Gram
// (recycle.py:66-92) as short pipelines with device-side decisions.
//
// Extraction, all kernels on one stream, no host synchronisation inside:
//   E1 zgather     Z = [W_prev, p_0..p_m-1], AZ = [AW_prev, (r_j - r_j+1)/alpha_j]
//                  (row-major n x T), per-CTA column sums of squares; the last
//                  CTA forms the norms, the keep list of non-zero columns and
//                  the plan (T_kept, or BasisDeficient when T_kept < k)
//   E2 zscale_fg   Zs = Z[:, keep] / norm, AZs likewise (n x T_kept) and the
//                  per-CTA partials of F = AZs'Zs, G = AZs'AZs
//   E3 fg_reduce   fixed-order reduction of the partials (one warp per entry)
//   E4 pencil      symmetrise, failing-pivot pruning, G u = theta F u (dense_small.cu)
//   E5 uscale      ||Zs u_j|| per selected vector (last CTA scales U)
//   E6 wnext       W_next = Zs U, AW_next = AZs U in the reference's i-k-j order
// The outcome (status, payload, T) is written to a device result block the
// caller reads whenever it joins the stream, so the extraction can overlap
// other work (the GPC Newton update) on a side stream.
#include "common.cuh"

int dcg_ritz_pencil_launch(cudaStream_t, const double*, const double*, int, int, int, int, double*, double*, double*,
                           int*, DevStatus*, const DevStatus*);
size_t dcg_pencil_smem(int T);

#define EX_NT 256
#define EX_ROWS 32

// ---------------------------------------------------------------------------- E1
// Column norms from the per-CTA partials (one warp per column, CTA order),
// the keep list of non-zero columns and the plan.  Results in shared memory
// (s_norm, s_keep, *s_t); `norms` (when non-null), keep and plan in global.
__device__ void zgather_finish(int T, int k, const double* part, double* s_norm, int* s_keep, int* s_t,
                               double* norms, int* keep, DevStatus* plan) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = warp; c < T; c += EX_NT / 32) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += ld_cg(part + (long long)b * T + c);
        s = warp_sum(s);
        if (lane == 0) {
            s_norm[c] = sqrt(s);
            if (norms) norms[c] = s_norm[c];
        }
    }
    cta_sync();
    if (tid == 0) {
        int t = 0;
        for (int c = 0; c < T; ++c)
            if (s_norm[c] > 0.0) s_keep[t++] = c;
        *s_t = t;
        if (norms) {
            for (int c = 0; c < t; ++c) keep[c] = s_keep[c];
            plan->count = t;
            plan->info = t;
            plan->aux = T;   // column stride of Zraw / AZraw
            plan->status = (t < k) ? DCG_E_BASIS_DEFICIENT : DCG_OK;   // recycle.py:131-132
        }
    }
    cta_sync();
}

__device__ void zgather_body(long long n, int kp, const double* __restrict__ Wp, const double* __restrict__ AWp,
                             int m, const double* __restrict__ P, const double* __restrict__ R,
                             const double* __restrict__ alpha, int k, double* Zraw, double* AZraw, double* part,
                             unsigned int* counter, double* norms, int* keep, DevStatus* plan,
                             const DevStatus* solve_st, bool coop, double* s_norm, int* s_keep, int* s_t) {
    extern __shared__ double sm[];
    if (solve_st) {
        // device-driven form: the finished solve's status block gives the
        // basis columns it used (pad) and the stored log length (aux)
        const bool bad = solve_st->status != DCG_OK;
        kp = (int)solve_st->pad;
        m = (int)solve_st->aux;
        if (bad || k > kp + m) {
            // recycle.py:104-108 (k > T: BasisDeficient(T)); a failed solve
            // leaves nothing to extract (its error surfaces from the solve)
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                plan->status = bad ? solve_st->status : DCG_E_BASIS_DEFICIENT;
                plan->info = kp + m;
                plan->count = kp + m;
                plan->aux = kp + m;
            }
            if (threadIdx.x == 0) *s_t = -1;   // nothing to scale (uniform over the grid)
            cta_sync();
            return;
        }
    }
    const int T = kp + m;
    double* zt = sm;                   // EX_ROWS x T
    double* azt = sm + EX_ROWS * T;    // EX_ROWS x T
    const int tid = threadIdx.x;
    const long long r0 = part_begin(n, gridDim.x, blockIdx.x), r1 = part_begin(n, gridDim.x, blockIdx.x + 1);
    double acc = 0.0;   // column tid's sum of squares (tid < T)
    for (long long i0 = r0; i0 < r1; i0 += EX_ROWS) {
        const int nr = (int)min((long long)EX_ROWS, r1 - i0);
        for (int e = tid; e < nr * kp; e += EX_NT) {
            const int r = e / kp, c = e % kp;
            zt[r * T + c] = Wp[(i0 + r) * kp + c];
            azt[r * T + c] = AWp[(i0 + r) * kp + c];
        }
        for (int e = tid; e < EX_ROWS * m; e += EX_NT) {
            const int j = e / EX_ROWS, r = e % EX_ROWS;
            if (r < nr) {
                const long long i = i0 + r;
                zt[r * T + kp + j] = P[(long long)j * n + i];
                azt[r * T + kp + j] = div_rn(sub_rn(R[(long long)j * n + i], R[(long long)(j + 1) * n + i]), alpha[j]);
            }
        }
        cta_sync();
        for (int e = tid; e < nr * T; e += EX_NT) {
            Zraw[i0 * T + e] = zt[e];
            AZraw[i0 * T + e] = azt[e];
        }
        if (tid < T)
            for (int r = 0; r < nr; ++r) acc = fma(zt[r * T + tid], zt[r * T + tid], acc);
        cta_sync();
    }
    if (tid < T) part[(long long)blockIdx.x * T + tid] = acc;
    if (coop) {
        // fused stage: every CTA forms the norms and the keep list itself
        // after a grid barrier (same partial order: same values); CTA 0
        // publishes them with the plan
        dcg_grid_barrier(counter, gridDim.x);   // (coop: the context's persistent barrier line)
        zgather_finish(T, k, part, s_norm, s_keep, s_t, blockIdx.x == 0 ? norms : nullptr, keep, plan);
        return;
    }
    if (!cta_last_arrival(counter, gridDim.x)) return;
    // last CTA: norms (one warp per column), keep list, plan
    zgather_finish(T, k, part, s_norm, s_keep, s_t, norms, keep, plan);
}

__global__ void __launch_bounds__(EX_NT)
    zgather_kernel(long long n, int kp, const double* __restrict__ Wp, const double* __restrict__ AWp, int m,
                   const double* __restrict__ P, const double* __restrict__ R, const double* __restrict__ alpha,
                   int k, double* Zraw, double* AZraw, double* part, unsigned int* counter, double* norms, int* keep,
                   DevStatus* plan, const DevStatus* solve_st) {
    __shared__ double s_norm[DCG_MAX_T];
    __shared__ int s_keep[DCG_MAX_T];
    __shared__ int s_t;
    zgather_body(n, kp, Wp, AWp, m, P, R, alpha, k, Zraw, AZraw, part, counter, norms, keep, plan, solve_st, false,
                 s_norm, s_keep, &s_t);
}

// ---------------------------------------------------------------------------- E2
// Register-blocked: thread (ta, tb) of a 16 x 16 grid owns F / G entries
// (a, b') with a = ta + 16 i, b' = tb + 16 j (b' < Tk: F[a][b'], else
// G[a][b' - Tk]), i < 4, j < 8 -- per staged row 12 shared loads feed up to
// 32 FMAs.  Each entry still accumulates over this CTA's rows in row order
// (fg_reduce then sums the CTAs in a fixed order), as before.
#define FG_BI 4
#define FG_BJ 8
__device__ void zscale_fg_body(long long n, const double* __restrict__ Zraw, const double* __restrict__ AZraw,
                               const double* norms, const int* keep, int T, int Tk, int region, double* Zs,
                               double* AZs, double* part) {
    extern __shared__ double sm[];
    const int npairs = 2 * Tk * Tk;
    // staged rows: [zs | azs] per row, 2 Tk wide, so b' indexes one array
    double* za = sm;                    // EX_ROWS x 2 Tk
    const int tid = threadIdx.x;
    // blockIdx.y picks the 64 x 128 region of the (a, b') grid (one region for Tk <= 64)
    const int nbj = (2 * Tk + 16 * FG_BJ - 1) / (16 * FG_BJ);
    const int a0 = (region / nbj) * 16 * FG_BI, b0 = (region % nbj) * 16 * FG_BJ;
    if (a0 >= Tk) return;
    const int ta = a0 + (tid >> 4), tb = b0 + (tid & 15);
    const long long r0 = part_begin(n, gridDim.x, blockIdx.x), r1 = part_begin(n, gridDim.x, blockIdx.x + 1);
    double acc[FG_BI][FG_BJ];
#pragma unroll
    for (int i = 0; i < FG_BI; ++i)
#pragma unroll
        for (int j = 0; j < FG_BJ; ++j) acc[i][j] = 0.0;
    const int W = 2 * Tk;
    for (long long i0 = r0; i0 < r1; i0 += EX_ROWS) {
        const int nr = (int)min((long long)EX_ROWS, r1 - i0);
        cta_sync();
        for (int e = tid; e < nr * Tk; e += EX_NT) {
            const int r = e / Tk, cc = e % Tk;
            const int c = keep[cc];
            const double nv = norms[c];
            const double zv = div_rn(Zraw[(i0 + r) * T + c], nv);
            const double av = div_rn(AZraw[(i0 + r) * T + c], nv);
            za[r * W + cc] = zv;
            za[r * W + Tk + cc] = av;
            if (region == 0) {
                Zs[(i0 + r) * Tk + cc] = zv;
                AZs[(i0 + r) * Tk + cc] = av;
            }
        }
        cta_sync();
        for (int r = 0; r < nr; ++r) {
            const double* row = za + r * W;
            double av[FG_BI], bv[FG_BJ];
#pragma unroll
            for (int i = 0; i < FG_BI; ++i) {
                const int a = ta + 16 * i;
                av[i] = a < Tk ? row[Tk + a] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < FG_BJ; ++j) {
                const int b = tb + 16 * j;
                bv[j] = b < W ? row[b] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < FG_BI; ++i)
#pragma unroll
                for (int j = 0; j < FG_BJ; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
    }
    double* out = part + (long long)blockIdx.x * npairs;
#pragma unroll
    for (int i = 0; i < FG_BI; ++i) {
        const int a = ta + 16 * i;
        if (a >= Tk) continue;
#pragma unroll
        for (int j = 0; j < FG_BJ; ++j) {
            const int b = tb + 16 * j;
            if (b < Tk) out[a * Tk + b] = acc[i][j];
            else if (b < W) out[Tk * Tk + a * Tk + (b - Tk)] = acc[i][j];
        }
    }
}

__global__ void __launch_bounds__(EX_NT)
    zscale_fg_kernel(long long n, const double* __restrict__ Zraw, const double* __restrict__ AZraw,
                     const double* __restrict__ norms, const int* __restrict__ keep, const DevStatus* plan, double* Zs,
                     double* AZs, double* part) {
    if (plan->status != DCG_OK) return;
    zscale_fg_body(n, Zraw, AZraw, norms, keep, (int)plan->aux, (int)plan->count, blockIdx.y, Zs, AZs, part);
}

// E1 + E2 as one cooperative launch (the norms after a grid barrier instead
// of a last-CTA pass and a second launch): same row partition, same partial
// orders, so the same Zs, AZs and F / G partials.  The F / G regions run one
// after the other in each CTA.
__global__ void __launch_bounds__(EX_NT)
    zstage1_coop_kernel(long long n, int kp, const double* __restrict__ Wp, const double* __restrict__ AWp, int m,
                        const double* __restrict__ P, const double* __restrict__ R, const double* __restrict__ alpha,
                        int k, double* Zraw, double* AZraw, double* part, unsigned int* counter, double* norms,
                        int* keep, DevStatus* plan, const DevStatus* solve_st, int nregions, double* Zs, double* AZs,
                        double* fgpart, double* Fraw, double* Graw) {
    __shared__ double s_norm[DCG_MAX_T];
    __shared__ int s_keep[DCG_MAX_T];
    __shared__ int s_t;
    zgather_body(n, kp, Wp, AWp, m, P, R, alpha, k, Zraw, AZraw, part, counter, norms, keep, plan, solve_st, true,
                 s_norm, s_keep, &s_t);
    const int t = s_t;
    if (t >= 0 && t >= k) {   // else failed / deficient: uniform over the grid
        const int T = solve_st ? (int)(solve_st->pad + solve_st->aux) : kp + m;
        for (int y = 0; y < nregions; ++y) {
            zscale_fg_body(n, Zraw, AZraw, s_norm, s_keep, T, t, y, Zs, AZs, fgpart);
            cta_sync();
        }
        // E3 after a second grid barrier: F and G from the partials, a warp
        // per entry with fg_reduce_kernel's lane split and warp sum (the same
        // values), the entries spread over every warp of the grid
        dcg_grid_barrier(counter, gridDim.x);
        const int npairs = 2 * t * t, lane = threadIdx.x & 31;
        const int nwarps = gridDim.x * (EX_NT / 32);
        for (int e = blockIdx.x * (EX_NT / 32) + (threadIdx.x >> 5); e < npairs; e += nwarps) {
            double sv = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) sv += ld_cg(fgpart + (long long)b * npairs + e);
            sv = warp_sum(sv);
            if (lane == 0) {
                if (e < t * t) Fraw[e] = sv;
                else Graw[e - t * t] = sv;
            }
        }
    }
    if (threadIdx.x == 0) dcg_sync_exit(counter, gridDim.x);
}

// ---------------------------------------------------------------------------- E3
__global__ void fg_reduce_kernel(const double* part, int nparts, const DevStatus* plan, double* Fraw, double* Graw) {
    if (plan->status != DCG_OK) return;
    const int Tk = (int)plan->count;
    const int npairs = 2 * Tk * Tk;
    const int lane = threadIdx.x & 31;
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (e >= npairs) return;
    double s = 0.0;
    for (int b = lane; b < nparts; b += 32) s += part[(long long)b * npairs + e];
    s = warp_sum(s);
    if (lane == 0) {
        if (e < Tk * Tk) Fraw[e] = s;
        else Graw[e - Tk * Tk] = s;
    }
}

// ---------------------------------------------------------------------------- E5
// ||Zs u_j||^2 partials for the selected vectors; the last CTA scales U.
// Rows are staged EX_ROWS at a time into shared memory with coalesced loads
// (a lane's dependent FMA chain over the Tk columns then reads shared memory:
// with the global loads inside the chain, in-order issue serialised one L2
// round trip per column -- 1.3 ms per call at n = 50k, T = 68).  A 16 x 16
// thread grid (two rows x up to four columns per thread per staged block)
// keeps every thread busy; with a warp per row only k of 32 lanes worked.
__global__ void __launch_bounds__(EX_NT)
    uscale_kernel(long long n, int k, const double* __restrict__ Zs, const DevStatus* plan, const DevStatus* pencil,
                  double* U, const int* active, double* Uexp, double* part, unsigned int* counter) {
    if (plan->status != DCG_OK || pencil->status != DCG_OK) return;
    extern __shared__ double sm[];
    const int Tk = (int)plan->count, na = (int)pencil->count;
    double* ue = sm;                       // Tk x k
    double* wp = ue + Tk * k;              // 16 row slots x 64
    double* zr = wp + 16 * 64;             // EX_ROWS x Tk staged rows
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < Tk * k; e += EX_NT) ue[e] = 0.0;
    cta_sync();
    for (int e = tid; e < na * k; e += EX_NT) ue[active[e / k] * k + e % k] = U[e];
    const long long r0 = part_begin(n, gridDim.x, blockIdx.x), r1 = part_begin(n, gridDim.x, blockIdx.x + 1);
    // thread (rs, jg): rows rs, rs + 16 of a staged block, columns jg + 16 q
    const int rs = tid >> 4, jg = tid & 15;
    double sq[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i0 = r0; i0 < r1; i0 += EX_ROWS) {
        const int nr = (int)min((long long)EX_ROWS, r1 - i0);
        cta_sync();
        for (int e = tid; e < nr * Tk; e += EX_NT) zr[e] = Zs[i0 * Tk + e];
        cta_sync();
        for (int rr = rs; rr < nr; rr += 16) {
            const double* z = zr + rr * Tk;
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c = 0; c < Tk; ++c) {
                const double zc = z[c];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (jg + 16 * q < k) v[q] = fma(zc, ue[c * k + jg + 16 * q], v[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) sq[q] = fma(v[q], v[q], sq[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) wp[rs * 64 + jg + 16 * q] = sq[q];
    cta_sync();
    if (tid < k) {
        double s = 0.0;
        for (int w = 0; w < 16; ++w) s += wp[w * 64 + tid];
        part[(long long)blockIdx.x * k + tid] = s;
    }
    if (!cta_last_arrival(counter, gridDim.x)) return;
    __shared__ double scale[DCG_MAX_K];
    for (int j = warp; j < k; j += EX_NT / 32) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += ld_cg(part + (long long)b * k + j);
        s = warp_sum(s);
        if (lane == 0) scale[j] = sqrt(s);
    }
    cta_sync();
    // u[:, j] /= ||Z u_j|| when positive (recycle.py:150-153)
    for (int e = tid; e < na * k; e += EX_NT) {
        const double sc = scale[e % k];
        if (sc > 0.0) U[e] = div_rn(U[e], sc);
    }
    cta_sync();
    for (int e = tid; e < Tk * k; e += EX_NT) Uexp[e] = 0.0;
    cta_sync();
    for (int e = tid; e < na * k; e += EX_NT) Uexp[active[e / k] * k + e % k] = U[e];
}

// ---------------------------------------------------------------------------- E6
// W_next = Zs U, AW_next = AZs U with the reference's accumulation order
// (_core.gemm i-k-j, recycle.py:157-158); z output = the surviving columns.
// A CTA takes EX_ROWS rows at a time: Zs / AZs rows staged coalesced into
// shared memory, then every thread runs (EX_ROWS k / EX_NT) independent
// column chains from there.
__global__ void __launch_bounds__(EX_NT)
    wnext_kernel(long long n, int k, const double* __restrict__ Zs, const double* __restrict__ AZs,
                 const DevStatus* plan, const DevStatus* pencil, const double* __restrict__ Uexp, const int* active,
                 double* w_next, double* aw_next, double* z_out, long long* result) {
    const bool ok = plan->status == DCG_OK && pencil->status == DCG_OK;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // result block: status, info, t_out
        if (plan->status != DCG_OK) {
            result[0] = plan->status;
            result[1] = plan->info;
            result[2] = plan->count;
        } else {
            result[0] = pencil->status;
            result[1] = pencil->info;
            result[2] = pencil->count;
        }
    }
    if (!ok) return;
    extern __shared__ double sm[];
    const int Tk = (int)plan->count, na = (int)pencil->count;
    double* ue = sm;                   // Tk x k
    double* zr = ue + Tk * k;          // EX_ROWS x Tk
    double* ar = zr + EX_ROWS * Tk;    // EX_ROWS x Tk
    for (int e = threadIdx.x; e < Tk * k; e += EX_NT) ue[e] = Uexp[e];
    const long long nblk = (n + EX_ROWS - 1) / EX_ROWS;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long i0 = blk * EX_ROWS;
        const int nr = (int)min((long long)EX_ROWS, n - i0);
        cta_sync();
        for (int e = threadIdx.x; e < nr * Tk; e += EX_NT) {
            zr[e] = Zs[i0 * Tk + e];
            if (aw_next) ar[e] = AZs[i0 * Tk + e];
        }
        cta_sync();
        for (int e = threadIdx.x; e < nr * k; e += EX_NT) {
            const int rr = e / k, j = e - (e / k) * k;
            const double* z = zr + rr * Tk;
            const double* az = ar + rr * Tk;
            double a = 0.0, b = 0.0;
            for (int c = 0; c < Tk; ++c) {
                const double u = ue[c * k + j];
                a = add_rn(a, mul_rn(z[c], u));
                if (aw_next) b = add_rn(b, mul_rn(az[c], u));
            }
            w_next[(i0 + rr) * k + j] = a;
            if (aw_next) aw_next[(i0 + rr) * k + j] = b;
        }
    }
    if (z_out) {
        const long long tz = n * na;
        for (long long e = blockIdx.x * (long long)EX_NT + threadIdx.x; e < tz; e += (long long)gridDim.x * EX_NT)
            z_out[e] = Zs[(e / na) * Tk + active[e % na]];
    }
}

// E5 + E6 as one cooperative launch: the ||Zs u_j|| partials, a grid barrier,
// every CTA forms the scales from the partials (warp per column, CTA order:
// the values of uscale's last CTA) and scales its shared copy of U, then
// W_next / AW_next for its row blocks (each element as in wnext).  No U
// round trip through global memory, one launch instead of two.
__device__ __forceinline__ void tail_body(long long n, int k, const double* __restrict__ Zs,
                                          const double* __restrict__ AZs, const DevStatus* plan,
                                          const DevStatus* pencil, double* U, const int* active, double* part,
                                          unsigned int* bar, double* w_next, double* aw_next, long long* result) {
    const bool ok = plan->status == DCG_OK && pencil->status == DCG_OK;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (plan->status != DCG_OK) {
            result[0] = plan->status;
            result[1] = plan->info;
            result[2] = plan->count;
        } else {
            result[0] = pencil->status;
            result[1] = pencil->info;
            result[2] = pencil->count;
        }
    }
    if (!ok) return;
    extern __shared__ double sm[];
    const int Tk = (int)plan->count, na = (int)pencil->count;
    double* ue = sm;                       // Tk x k (unscaled, then scaled)
    double* wp = ue + Tk * k;              // 16 row slots x 64
    double* zr = wp + 16 * 64;             // EX_ROWS x Tk
    double* ar = zr + EX_ROWS * Tk;        // EX_ROWS x Tk
    __shared__ double scale[DCG_MAX_K];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < Tk * k; e += EX_NT) ue[e] = 0.0;
    cta_sync();
    for (int e = tid; e < na * k; e += EX_NT) ue[active[e / k] * k + e % k] = U[e];
    // ---- E5: partial column norms (uscale's thread grid and order)
    const long long r0 = part_begin(n, gridDim.x, blockIdx.x), r1 = part_begin(n, gridDim.x, blockIdx.x + 1);
    const int rs = tid >> 4, jg = tid & 15;
    double sq[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i0 = r0; i0 < r1; i0 += EX_ROWS) {
        const int nr = (int)min((long long)EX_ROWS, r1 - i0);
        cta_sync();
        for (int e = tid; e < nr * Tk; e += EX_NT) zr[e] = Zs[i0 * Tk + e];
        cta_sync();
        for (int rr = rs; rr < nr; rr += 16) {
            const double* z = zr + rr * Tk;
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c = 0; c < Tk; ++c) {
                const double zc = z[c];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (jg + 16 * q < k) v[q] = fma(zc, ue[c * k + jg + 16 * q], v[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) sq[q] = fma(v[q], v[q], sq[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) wp[rs * 64 + jg + 16 * q] = sq[q];
    cta_sync();
    if (tid < k) {
        double sacc = 0.0;
        for (int w = 0; w < 16; ++w) sacc += wp[w * 64 + tid];
        part[(long long)blockIdx.x * k + tid] = sacc;
    }
    dcg_grid_barrier(bar, gridDim.x);
    for (int j = warp; j < k; j += EX_NT / 32) {
        double sacc = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) sacc += ld_cg(part + (long long)b * k + j);
        sacc = warp_sum(sacc);
        if (lane == 0) scale[j] = sqrt(sacc);
    }
    cta_sync();
    // u[:, j] /= ||Z u_j|| when positive (recycle.py:150-153), in shared memory;
    // CTA 0 also leaves the scaled U in global memory (the caller's copy)
    for (int e = tid; e < na * k; e += EX_NT) {
        const double sc = scale[e % k];
        const double u = sc > 0.0 ? div_rn(U[e], sc) : U[e];
        ue[active[e / k] * k + e % k] = u;
    }
    cta_sync();
    dcg_grid_barrier(bar, gridDim.x);   // every CTA has read the unscaled U
    if (blockIdx.x == 0)
        for (int e = tid; e < na * k; e += EX_NT) U[e] = ue[active[e / k] * k + e % k];
    // ---- E6: W_next = Zs U, AW_next = AZs U (wnext's element order)
    const long long nblk = (n + EX_ROWS - 1) / EX_ROWS;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long i0 = blk * EX_ROWS;
        const int nr = (int)min((long long)EX_ROWS, n - i0);
        cta_sync();
        for (int e = tid; e < nr * Tk; e += EX_NT) {
            zr[e] = Zs[i0 * Tk + e];
            if (aw_next) ar[e] = AZs[i0 * Tk + e];
        }
        cta_sync();
        if (aw_next) {
            for (int e = tid; e < nr * k; e += EX_NT) {
                const int rr = e / k, j = e - (e / k) * k;
                const double* z = zr + rr * Tk;
                const double* az = ar + rr * Tk;
                double a = 0.0, b = 0.0;
                for (int c = 0; c < Tk; ++c) {
                    const double u = ue[c * k + j];
                    a = add_rn(a, mul_rn(z[c], u));
                    b = add_rn(b, mul_rn(az[c], u));
                }
                w_next[(i0 + rr) * k + j] = a;
                aw_next[(i0 + rr) * k + j] = b;
            }
        } else {
            // AW_next not wanted (the caller refreshes the basis against the
            // next matrix before any use): W_next alone, same element order
            for (int e = tid; e < nr * k; e += EX_NT) {
                const int rr = e / k, j = e - (e / k) * k;
                const double* z = zr + rr * Tk;
                double a = 0.0;
                for (int c = 0; c < Tk; ++c) a = add_rn(a, mul_rn(z[c], ue[c * k + j]));
                w_next[(i0 + rr) * k + j] = a;
            }
        }
    }
}

__global__ void __launch_bounds__(EX_NT)
    tail_coop_kernel(long long n, int k, const double* __restrict__ Zs, const double* __restrict__ AZs,
                     const DevStatus* plan, const DevStatus* pencil, double* U, const int* active, double* part,
                     unsigned int* bar, double* w_next, double* aw_next, long long* result) {
    tail_body(n, k, Zs, AZs, plan, pencil, U, active, part, bar, w_next, aw_next, result);
    if (threadIdx.x == 0) dcg_sync_exit(bar, gridDim.x);
}

// ---------------------------------------------------------------------------- launch
static size_t extract_ws_bytes(dcg_context* ctx, long long n, int T, int k) {
    const int G = ctx->sm_count;
    const size_t nT = (size_t)n * T;
    return 4 * al(sizeof(double) * nT) + al(sizeof(double) * (size_t)G * T) + al(sizeof(double) * T) +
           2 * al(sizeof(int) * T) + 2 * al(sizeof(double) * T * T) + al(sizeof(double) * (size_t)G * 2 * T * T) +
           al(sizeof(double) * 5 * T * T) + 2 * al(sizeof(double) * T * k) + al(sizeof(double) * (size_t)G * k) +
           3 * al(sizeof(DevStatus)) + 2 * al(sizeof(unsigned int) * 4) + 8192;
}

// Enqueue the pipeline.  T is the column count (host-known), or with
// solve_st the upper bound k_prev_max + ell (the actual k_prev and m are read
// from the solve's status block on the device).
// stage: 0 = the whole pipeline; 1 = E1-E3 (the SM-wide column work, run on
// the main stream ahead of the Newton update); 2 = E4-E6 (the single-CTA
// pencil and the tail, on the side stream); 3 = E4 alone and 4 = E5-E6 alone
// (the pencil on the side stream, its SM-wide tail on the main stream once
// the pencil is done: on the side stream the tail only gets the SMs the main
// stream's products leave).  Stages share the context's
// workspace layout, so they must be enqueued with identical arguments.
static int extract_enqueue(dcg_context* ctx, cudaStream_t st, long long n, const dcg_krylov_log* log, long long m,
                           long long kp, long long T, const DevStatus* solve_st, const double* Wp, const double* AWp,
                           long long k, int selection, double* d_theta, double* d_u, double* d_z, double* d_w_next,
                           double* d_aw_next, long long* d_result, int stage = 0) {
    if (k > DCG_MAX_K || T > DCG_MAX_T) return DCG_E_UNSUPPORTED;
    int rc = dcg_ws_reserve(ctx, extract_ws_bytes(ctx, n, (int)T, (int)k));
    if (rc) return rc;
    const int G = ctx->sm_count;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    const size_t nT = (size_t)n * T;
    double* Zraw = ar.take<double>(nT);
    double* AZraw = ar.take<double>(nT);
    double* Zs = ar.take<double>(nT);
    double* AZs = ar.take<double>(nT);
    double* part = ar.take<double>((size_t)G * T);
    double* norms = ar.take<double>(T);
    int* keep = ar.take<int>(T);
    int* active = ar.take<int>(T);
    double* Fraw = ar.take<double>(T * T);
    double* Graw = ar.take<double>(T * T);
    double* fgpart = ar.take<double>((size_t)G * 2 * T * T);
    double* wk = ar.take<double>(5 * T * T);
    double* U = ar.take<double>(T * k);
    double* Uexp = ar.take<double>(T * k);
    double* upart = ar.take<double>((size_t)G * k);
    DevStatus* plan = ar.take<DevStatus>(1);
    DevStatus* pencil = ar.take<DevStatus>(1);
    unsigned int* counters = ar.take<unsigned int>(4);
    const double* P = log ? log->d_p : nullptr;
    const double* R = log ? log->d_r : nullptr;
    const double* alpha = log ? log->d_alpha : nullptr;

    int nb = G;
    if (n < (long long)nb * EX_ROWS) nb = (int)max(1LL, (n + EX_ROWS - 1) / EX_ROWS);
    const size_t sm1 = sizeof(double) * 2 * EX_ROWS * T;
    if (stage == 0 || stage == 1) {
    // (no memset of plan / pencil: every path of zgather and of the pencil
    // writes the fields that are read; the cooperative launches' barrier words
    // are the context's persistent lines)
    // regions of 64 x 128 (a, b') entries; Tk <= T decides on the device which are live
    int gy = (int)(((T + 16 * FG_BI - 1) / (16 * FG_BI)) * ((2 * T + 16 * FG_BJ - 1) / (16 * FG_BJ)));
    // one cooperative launch when the grid is co-resident (it is: nb <= SMs)
    int per_sm = 0;
    DCG_SMEM_ATTR(zstage1_coop_kernel, sm1);
    {
        static std::atomic<long long> occ_cache[DCG_MAX_DEVICES];
        rc = dcg_occupancy_cached(occ_cache, (const void*)zstage1_coop_kernel, EX_NT, sm1, &per_sm);
        if (rc) return rc;
    }
    if ((long long)per_sm * G >= nb) {
        int ikp = (int)kp, im = (int)m, ik = (int)k;
        unsigned int* line = dcg_sync_line(ctx, DCG_SW_ZSTAGE1);
        void* args[] = {(void*)&n,    (void*)&ikp,   (void*)&Wp,     (void*)&AWp,   (void*)&im,      (void*)&P,
                        (void*)&R,    (void*)&alpha, (void*)&ik,     (void*)&Zraw,  (void*)&AZraw,   (void*)&part,
                        (void*)&line, (void*)&norms, (void*)&keep, (void*)&plan, (void*)&solve_st, (void*)&gy,
                        (void*)&Zs,   (void*)&AZs,   (void*)&fgpart, (void*)&Fraw, (void*)&Graw};
        DCG_CUDA(cudaLaunchCooperativeKernel((const void*)zstage1_coop_kernel, dim3(nb), dim3(EX_NT), args, sm1, st));
        dcg_count_launch();
    } else {
        DCG_CUDA(cudaMemsetAsync(counters, 0, 16, st));   // the last-arrival counters (workspace)
        DCG_CUDA(cudaFuncSetAttribute(zgather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
        zgather_kernel<<<nb, EX_NT, sm1, st>>>(n, (int)kp, Wp, AWp, (int)m, P, R, alpha, (int)k, Zraw, AZraw, part,
                                               counters, norms, keep, plan, solve_st);
        DCG_LAUNCHED();
        DCG_CUDA(cudaFuncSetAttribute(zscale_fg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
        zscale_fg_kernel<<<dim3(nb, gy), EX_NT, sm1, st>>>(n, Zraw, AZraw, norms, keep, plan, Zs, AZs, fgpart);
        DCG_LAUNCHED();
        const int warps = (int)(2 * T * T);
        fg_reduce_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(fgpart, nb, plan, Fraw, Graw);
        DCG_LAUNCHED();
    }
    }
    if (stage == 1) return DCG_OK;
    if (stage != 4) {
        rc = dcg_ritz_pencil_launch(st, Fraw, Graw, (int)T, (int)k, selection == DCG_SELECT_LARGEST, 60, wk, d_theta,
                                    U, active, pencil, plan);
        if (rc) return rc;
    }
    if (stage == 3) return DCG_OK;
    // the cooperative tail (no z_out requested: the device-driven pipeline)
    if (!d_z) {
        const size_t smt = sizeof(double) * ((size_t)T * k + 16 * 64 + 2 * (size_t)EX_ROWS * T);
        int per_sm = 0;
        DCG_SMEM_ATTR(tail_coop_kernel, smt);
        {
            static std::atomic<long long> occ_cache[DCG_MAX_DEVICES];
            rc = dcg_occupancy_cached(occ_cache, (const void*)tail_coop_kernel, EX_NT, smt, &per_sm);
            if (rc) return rc;
        }
        if ((long long)per_sm * G >= nb) {
            int ik = (int)k;
            unsigned int* bar = dcg_sync_line(ctx, DCG_SW_TAIL);
            void* args[] = {(void*)&n,      (void*)&ik,     (void*)&Zs,      (void*)&AZs,      (void*)&plan,
                            (void*)&pencil, (void*)&U,      (void*)&active,  (void*)&upart,    (void*)&bar,
                            (void*)&d_w_next, (void*)&d_aw_next, (void*)&d_result};
            DCG_CUDA(cudaLaunchCooperativeKernel((const void*)tail_coop_kernel, dim3(nb), dim3(EX_NT), args, smt, st));
            dcg_count_launch();
            if (d_u) DCG_CUDA(cudaMemcpyAsync(d_u, U, sizeof(double) * T * k, cudaMemcpyDeviceToDevice, st));
            return DCG_OK;
        }
    }
    DCG_CUDA(cudaMemsetAsync(counters + 1, 0, sizeof(unsigned int), st));   // uscale's last-arrival counter
    const size_t sm5 = sizeof(double) * ((size_t)T * k + 16 * 64 + (size_t)EX_ROWS * T);
    DCG_CUDA(cudaFuncSetAttribute(uscale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm5));
    uscale_kernel<<<nb, EX_NT, sm5, st>>>(n, (int)k, Zs, plan, pencil, U, active, Uexp, upart, counters + 1);
    DCG_LAUNCHED();
    const size_t sm6 = sizeof(double) * ((size_t)T * k + 2 * (size_t)EX_ROWS * T);
    DCG_CUDA(cudaFuncSetAttribute(wnext_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6));
    wnext_kernel<<<G * 2, EX_NT, sm6, st>>>(n, (int)k, Zs, AZs, plan, pencil, Uexp, active, d_w_next, d_aw_next,
                                            d_z, d_result);
    DCG_LAUNCHED();
    if (d_u) DCG_CUDA(cudaMemcpyAsync(d_u, U, sizeof(double) * T * k, cudaMemcpyDeviceToDevice, st));
    return DCG_OK;
}

// Enqueue the extraction; `d_result` (3 x int64 on the device) receives
// status, info, t_out when the stream reaches the end.  Host-checkable
// argument errors return immediately.
extern "C" int dcg_ritz_extract_async(dcg_context* ctx, void* stream, long long n, const dcg_krylov_log* log,
                                      long long m, const dcg_basis* prev, long long k, int selection, double* d_theta,
                                      double* d_u, double* d_z, double* d_w_next, double* d_aw_next,
                                      long long* d_result) {
    if (!ctx || n < 0 || m < 0 || k < 0 || !d_result) return DCG_E_CONFIG;
    if (selection != DCG_SELECT_SMALLEST && selection != DCG_SELECT_LARGEST) return DCG_E_CONFIG;
    const long long kp = prev ? prev->k : 0;
    const long long T = kp + m;
    cudaStream_t st = as_stream(stream);
    if (k > T || k == 0) {
        // decided on the host (recycle.py:104-108 / k == 0): write the result block
        long long h[3] = {k > T ? (long long)DCG_E_BASIS_DEFICIENT : (long long)DCG_OK, T, T};
        DCG_CUDA(cudaMemcpyAsync(d_result, h, sizeof(h), cudaMemcpyHostToDevice, st));
        DCG_CUDA(cudaStreamSynchronize(st));   // h is a stack buffer
        return DCG_OK;
    }
    if (k > DCG_MAX_K || T > DCG_MAX_T) return DCG_E_UNSUPPORTED;
    if (m > 0 && (!log || log->ell < m || !log->d_p || !log->d_r || !log->d_alpha)) return DCG_E_CONFIG;
    if (kp > 0 && (!prev->d_w || !prev->d_aw)) return DCG_E_CONFIG;
    return extract_enqueue(ctx, st, n, m ? log : nullptr, m, kp, T, nullptr, kp ? prev->d_w : nullptr,
                           kp ? prev->d_aw : nullptr, k, selection, d_theta, d_u, d_z, d_w_next, d_aw_next, d_result);
}

// Device-driven form, enqueued right behind dcg_solve_async without waiting
// for it: the stored log length m and the basis columns the solve used are
// read from its status block (d_solve_status, the 64-byte block
// dcg_solve_async wrote); prev->k is the basis' column capacity (its columns
// compacted, stride = columns used), log->ell the log capacity.
extern "C" int dcg_ritz_extract_dev(dcg_context* ctx, void* stream, long long n, const dcg_krylov_log* log,
                                    const void* d_solve_status, const dcg_basis* prev, long long k, int selection,
                                    double* d_theta, double* d_w_next, double* d_aw_next, long long* d_result,
                                    int stage) {
    if (stage < 0 || stage > 4) return DCG_E_CONFIG;
    if (!ctx || n < 0 || k < 1 || !d_result || !d_solve_status || !log) return DCG_E_CONFIG;
    if (selection != DCG_SELECT_SMALLEST && selection != DCG_SELECT_LARGEST) return DCG_E_CONFIG;
    const long long kmax = prev ? prev->k : 0;
    const long long T = kmax + log->ell;
    if (kmax > 0 && (!prev->d_w || !prev->d_aw)) return DCG_E_CONFIG;
    if (log->ell > 0 && (!log->d_p || !log->d_r || !log->d_alpha)) return DCG_E_CONFIG;
    if (T < 1) {
        if (stage == 1 || stage == 3) return DCG_OK;
        // nothing can ever be extracted: BasisDeficient(0) (k >= 1 > T)
        DCG_CUDA(cudaMemsetAsync(d_result, 0, 3 * sizeof(long long), as_stream(stream)));
        long long* r0 = d_result;
        const long long code = DCG_E_BASIS_DEFICIENT;
        DCG_CUDA(cudaMemcpyAsync(r0, &code, sizeof(code), cudaMemcpyHostToDevice, as_stream(stream)));
        DCG_CUDA(cudaStreamSynchronize(as_stream(stream)));
        return DCG_OK;
    }
    return extract_enqueue(ctx, as_stream(stream), n, log, 0, 0, T, static_cast<const DevStatus*>(d_solve_status),
                           kmax ? prev->d_w : nullptr, kmax ? prev->d_aw : nullptr, k, selection, d_theta, nullptr,
                           nullptr, d_w_next, d_aw_next, d_result, stage);
}

// Synchronous form: enqueue, wait, and map the outcome to a status.
extern "C" int dcg_ritz_extract(dcg_context* ctx, void* stream, long long n, const dcg_krylov_log* log, long long m,
                                const dcg_basis* prev, long long k, int selection, double* d_theta, double* d_u,
                                double* d_z, double* d_w_next, double* d_aw_next, long long* t_out, long long* info) {
    if (info) *info = 0;
    const long long kp = prev ? prev->k : 0;
    if (t_out) *t_out = kp + m;
    if (!ctx) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    int rc = dcg_host_reserve(ctx, 64);
    if (rc) return rc;
    // the result block: a small allocation owned by the context (its device)
    if (!ctx->d_res) DCG_CUDA(cudaMalloc(&ctx->d_res, 64));
    long long* d_res = ctx->d_res;
    rc = dcg_ritz_extract_async(ctx, stream, n, log, m, prev, k, selection, d_theta, d_u, d_z, d_w_next, d_aw_next,
                                d_res);
    if (rc) return rc;
    long long* h = static_cast<long long*>(ctx->host);
    DCG_CUDA(cudaMemcpyAsync(h, d_res, 3 * sizeof(long long), cudaMemcpyDeviceToHost, st));
    DCG_CUDA(cudaStreamSynchronize(st));
    if (t_out) *t_out = h[2];
    if (h[0] != DCG_OK) {
        if (info) *info = h[1];
        return (int)h[0];
    }
    return DCG_OK;
}
