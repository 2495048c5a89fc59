// The whole CG / deflated-CG solve as ONE persistent cooperative kernel.
//
// Restates solvers.py:_run_loop (131-204) together with the warm-start
// correction of deflated_cg_solve (222-239): there is no host round trip per
// iteration.  One CTA per SM owns a contiguous, balanced row range of the
// system.  Per iteration:
//   phase G  Ap = shift p + s (.) K (s (.) p) for own rows, partial p'Ap   | grid barrier
//   phase U  alpha; x += alpha p; r -= alpha Ap (or true residual every
//            `recompute` iterations); partial r'r and AW'r (k dots)         | grid barrier
//   phase P  beta, mu = L^-T L^-1 AW'r (each CTA, redundantly), p update,
//            residual history / Krylov log writes                           | grid barrier
// Scalars are reduced from per-CTA partials in a fixed order by every CTA,
// so all CTAs take identical control-flow decisions (convergence, breakdown,
// max_iters) without a second barrier, and results are bit-reproducible.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemv.cuh"
#include "symgemv.cuh"
#include "rbfmma.cuh"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

namespace cg = cooperative_groups;


namespace {

struct SolveArgs {
    const double* K;
    const double* Kp;      // packed lower-triangle tiles (STRAT_SYMPK)
    long long ldk;
    long long n;
    const double* s;
    double shift;
    const double* b;
    const double* x0;
    const double* ax0;     // optional: A x0 computed ahead of the launch (x0 as passed, before any deflation correction)
    double* x;
    int k;                 // basis columns (the layout / maximum)
    const long long* kdev; // optional: columns in use, read on the device (<= k; 0 = plain CG)
    const double* W;
    const double* AW;
    const double* L;
    int warm;
    double tol;
    long long max_iters;
    long long ell;
    long long recompute;
    double* logP;
    double* logR;
    double* logD;
    double* logAlpha;
    double* logBeta;
    double* logMu;
    double* history;
    double* r;
    double* p;
    double* ap;
    double* partials;  // two buffers of G x ps: reductions 0 (r'r, W'r, AW'r) and 1 (p'Ap)
    double* colpart;   // symmetric strategy: per-tile partials
    double* rowpart;
    int ps;   // partial stride (doubles)
    DevStatus* st;
    unsigned int* bar;  // grid barrier arrival counter (zeroed per launch)
    unsigned long long* timers;   // optional per-phase ns accumulators (CTA 0, thread 0)
    RbfMma rbf;                   // matrix-free operator (STRAT_RBF)
    const long long* symtbl;      // symmetric strategies: host-computed pass-1 range table (dcg_sym_table)
};

// mu = L^-T L^-1 c for the k x k row-major lower factor of W'AW in shared
// memory, by one warp (lanes own rows lane and lane + 32).  This is the
// reference's chol_solve (solvers.py:152,190 -> _core.pyx:69-94): forward
// substitution in the reference's subtraction order; the backward sweep runs
// as a wavefront (subtractions as soon as x_j is known).  Pivots are applied as
// precomputed reciprocals (rdiag = 1 / L_jj): a serial FP64 division per
// unknown put ~17 us per iteration on the critical path at k = 16, the
// reciprocal costs at most one extra rounding per unknown.  Triangular solves, not an explicit inverse: W'AW can be
// ill-conditioned (random or nearly dependent W) and an explicit inverse
// loses the backward stability the projection relies on.
__device__ void warp_chol_solve(const double* L, const double* rdiag, int k, const double* c, double* out) {
    const int lane = threadIdx.x & 31;
    const int i0 = lane, i1 = lane + 32;
    double a0 = (i0 < k) ? c[i0] : 0.0;
    double a1 = (i1 < k) ? c[i1] : 0.0;
    for (int j = 0; j < k; ++j) {
        const double accj = __shfl_sync(0xffffffffu, (j < 32) ? a0 : a1, j & 31);
        const double yj = mul_rn(accj, rdiag[j]);
        if (lane == (j & 31)) {
            if (j < 32) a0 = yj; else a1 = yj;
        }
        if (i0 > j && i0 < k) a0 = sub_rn(a0, mul_rn(L[i0 * k + j], yj));
        if (i1 > j && i1 < k) a1 = sub_rn(a1, mul_rn(L[i1 * k + j], yj));
    }
    for (int j = k - 1; j >= 0; --j) {
        const double accj = __shfl_sync(0xffffffffu, (j < 32) ? a0 : a1, j & 31);
        const double xj = mul_rn(accj, rdiag[j]);
        if (lane == (j & 31)) {
            if (j < 32) a0 = xj; else a1 = xj;
        }
        if (i0 < j) a0 = sub_rn(a0, mul_rn(L[j * k + i0], xj));
        if (i1 < j && i1 < k) a1 = sub_rn(a1, mul_rn(L[j * k + i1], xj));
    }
    if (i0 < k) out[i0] = a0;
    if (i1 < k) out[i1] = a1;
}

// mu for the deflated update: warp 0 solves, then one CTA barrier.
__device__ __forceinline__ void solve_mu(const double* L, const double* rdiag, int k, const double* c, double* mu) {
    if ((threadIdx.x >> 5) == 0) warp_chol_solve(L, rdiag, k, c, mu);
    cta_sync();
}

// Fixed-order reduction of the per-CTA partials into shared memory (every CTA
// computes the identical values).  All 512 threads load in parallel: slot
// v = t % SW, CTA group t / SW, SW = next power of two >= nslots, so each
// thread issues at most ceil(G / (512 / SW)) independent loads; groups are then
// combined in a fixed order.  `scr` holds 512 doubles.
__device__ __forceinline__ void reduce_partials(const double* partials, int G, int ps, int nslots, double* out,
                                                double* scr) {
    const int tid = threadIdx.x;
    int sw = 1;
    while (sw < nslots) sw <<= 1;
    const int ng = DCG_NT / sw;
    const int v = tid & (sw - 1), gq = tid / sw;
    double a = 0.0;
    if (v < nslots) {
        // up to 16 independent loads in flight per thread (one latency round
        // for G <= 16 * 512 / sw CTAs: 148 CTAs with up to 32 slots); the adds
        // keep the ascending-g order
        for (int g0 = gq; g0 < G; g0 += 16 * ng) {
            double t[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int g = g0 + u * ng;
                t[u] = (g < G) ? ld_cg(partials + (long long)g * ps + v) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) a += t[u];
        }
    }
    if (sw <= 32) {
        // groups inside a warp share a slot at lanes v, v + sw, ...: butterfly over them
        for (int o = sw; o < 32; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const int lane = tid & 31, warp = tid >> 5;
        if (lane < sw) scr[warp * 32 + lane] = a;
        cta_sync();
        if (tid < nslots) {
            double t = 0.0;
#pragma unroll 4
            for (int w = 0; w < DCG_NW; ++w) t += scr[w * 32 + tid];
            out[tid] = t;
        }
    } else {
        scr[tid] = a;
        cta_sync();
        if (tid < nslots) {
            double t = 0.0;
            for (int g = 0; g < ng; ++g) t += scr[g * sw + tid];
            out[tid] = t;
        }
    }
    cta_sync();
}

// GEMV strategies of the persistent kernel
enum { STRAT_ROWS = 0, STRAT_SYM = 1, STRAT_RBF = 2, STRAT_SYMPK = 3 };

// Shared-memory doubles of the GEMV region for each strategy.
__host__ __device__ __forceinline__ long long gemv_region_doubles(int strat, long long n, int dim, int nteam) {
    if (strat == STRAT_SYM || strat == STRAT_SYMPK) return sym_smem_doubles();
    if (strat == STRAT_RBF) return rm_smem_doubles(dim, nteam);
    return min(n, (long long)DCG_QT) + 2 + DCG_NW * DCG_RB;
}

// Every exit writes the whole status block (the block is not cleared before
// the launch: in the asynchronous form it is the caller's buffer).
__device__ __forceinline__ void put_status(DevStatus* st, int status, int k, long long info, long long count,
                                           long long aux, double value, double value2) {
    st->status = status;
    st->pad = k;
    st->info = info;
    st->count = count;
    st->aux = aux;
    st->value = value;
    st->value2 = value2;
}

template <int STRAT>
__device__ __forceinline__ void solve_body(const SolveArgs& a) {
#define GSYNC() dcg_grid_barrier(a.bar, gridDim.x)
    // Phase timers (DCG_PHASE_TIMERS): CTA 0 / thread 0 attributes the time since
    // the previous mark to phase `id`; one predicated branch when disabled.
    unsigned long long t_mark = 0;
#define PHASE(id)                                                          \
    do {                                                                   \
        if (a.timers && blockIdx.x == 0 && threadIdx.x == 0) {             \
            const unsigned long long t_ = globaltimer_ns();                \
            if (t_mark) a.timers[id] += t_ - t_mark;                        \
            t_mark = t_;                                                   \
        }                                                                  \
    } while (0)
    extern __shared__ __align__(16) double smem[];
    const long long n = a.n;
    // columns in use: the host's k, or the device-side count an asynchronous
    // refresh left (W / AW / L are then compacted to that many columns)
    const int kmax = a.k;
    const int k = a.kdev ? (int)min((long long)kmax, max(0LL, *a.kdev)) : kmax;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int xt = (int)min(n, (long long)DCG_QT) + 2;
    double* s_g = smem;                                  // GEMV region (strategy dependent)
    double* s_L = s_g + gemv_region_doubles(STRAT, n, a.rbf.dim, a.rbf.nteam);   // k*k
    double* s_rd = s_L + kmax * kmax;                    // DCG_MAX_K  1 / L_jj
    double* s_c = s_rd + DCG_MAX_K;                      // 1 + DCG_MAX_K reduced slots
    double* s_mu = s_c + DCG_MAX_K + 2;                  // DCG_MAX_K
    double* s_tmp = s_mu + DCG_MAX_K;                    // 64 scratch
    double* s_scr = s_tmp + 64;                          // DCG_NT reduction scratch

    const long long r0 = part_begin(n, G, blockIdx.x);
    const long long r1 = part_begin(n, G, blockIdx.x + 1);
    const bool deflate = k > 0;
    const int nslots = 1 + k;
    const double* __restrict__ K = a.K;
    const double* s = a.s;
    const double shift = a.shift;

    unsigned int ring_seq = 0;
    constexpr bool kSym = STRAT == STRAT_SYM || STRAT == STRAT_SYMPK;
    constexpr bool kPk = STRAT == STRAT_SYMPK;
    int pending = 0;   // packed: tiles of the next pass already in flight
    // symmetric strategy: pass-2 rows are weighted by their partial count
    // (sym_row_begin), not the vector-phase rows [r0, r1); pass-2 outputs are
    // therefore read by other CTAs after a grid barrier, through L2.
    long long q0 = r0, q1 = r1;
    if constexpr (kSym) {
        sym_ring_init(s_g, n, kPk, a.symtbl);
        q0 = sym_row_begin(n, G, blockIdx.x);
        q1 = sym_row_begin(n, G, blockIdx.x + 1);
    }
    if constexpr (STRAT == STRAT_RBF) {
        rm_init(s_g, a.rbf);
        q0 = sym_row_begin(n, G, blockIdx.x);
        q1 = sym_row_begin(n, G, blockIdx.x + 1);
    }
    // t = K (s (.) v) for the own rows [r0, r1); epi(i, t_i) per row.  The
    // symmetric strategy contains one extra grid barrier between its passes.
    // The matrix-free strategy computes whole 64-row chunks (c = b, b + G, ...),
    // again read by other CTAs only after a grid barrier.
    auto gemv = [&](const double* v, auto&& epi) {
        if constexpr (STRAT == STRAT_RBF) {
            // symmetric half-evaluation of the regenerated tiles (FP64 tensor
            // pipe, rbfmma.cuh) + the shared pass 2 over the team ranges
            rbf_mma_pass1(a.rbf, v, s, a.colpart, a.rowpart, s_g);
            PHASE(0);
            GSYNC();
            PHASE(1);
            sym_pass2(n, a.colpart, a.rowpart, q0, q1, rm_table(s_g), G * a.rbf.nteam,
                      rm_pass2_scratch(s_g, a.rbf.dp), epi);
            PHASE(2);
        } else if constexpr (kSym) {
            PHASE(15);
            unsigned long long tc0 = 0;
            if (a.timers && threadIdx.x == 0) tc0 = globaltimer_ns();
            if constexpr (kPk)
                sym_pass1<true, 1, true>(a.Kp, 0, n, v, s, a.colpart, a.rowpart, s_g, ring_seq, nullptr, 0, &pending,
                                         true);
            else
                sym_pass1(K, a.ldk, n, v, s, a.colpart, a.rowpart, s_g, ring_seq);
            if (a.timers && threadIdx.x == 0) a.timers[16 + blockIdx.x] += globaltimer_ns() - tc0;
            PHASE(0);
            GSYNC();
            PHASE(1);
            if (a.timers && threadIdx.x == 0) tc0 = globaltimer_ns();
            sym_pass2<true>(n, a.colpart, a.rowpart, q0, q1, sym_range_table(s_g), G, s_scr, epi);
            if (a.timers && threadIdx.x == 0) a.timers[16 + gridDim.x + blockIdx.x] += globaltimer_ns() - tc0;
            PHASE(2);
        } else {
            block_gemv<true>(K, a.ldk, n, v, s, r0, r1, s_g, s_g + xt, epi);
        }
    };

    for (int i = tid; i < k * k; i += blockDim.x) s_L[i] = a.L[i];
    cta_sync();
    for (int j = tid; j < k; j += blockDim.x) s_rd[j] = 1.0 / s_L[j * k + j];
    cta_sync();

    // ---- own-row helpers ------------------------------------------------------
    // W / AW rows are read-only for the launch and re-read every iteration by
    // the same CTA; 16-byte loads when the rows allow it.
    const bool vec2 = ((k & 1) == 0) && (((reinterpret_cast<uintptr_t>(a.W) | reinterpret_cast<uintptr_t>(a.AW)) & 15) == 0);
    int swk = 1;   // power of two >= k: (row group, j) thread mapping of the basis partials
    while (swk < k) swk <<= 1;
    // sum_j M[i][j] v[j] for one row, by one thread (v in shared memory).
    auto row_dot = [&](const double* M, long long i, const double* v) {
        const double* row = M + i * k;
        double t = 0.0;
        if (vec2) {
#pragma unroll 4
            for (int j = 0; j < k; j += 2) {
                const double2 m = __ldg(reinterpret_cast<const double2*>(row + j));
                t = fma(m.x, v[j], t);
                t = fma(m.y, v[j + 1], t);
            }
        } else {
            for (int j = 0; j < k; ++j) t = fma(__ldg(row + j), v[j], t);
        }
        return t;
    };
    // Publish this CTA's partials: slot 0 = sum_i q_i^2 with q_i = sqval(i)
    // (thread-per-row; sqval may log, or write u_i itself: `sync_mid` then
    // orders those writes before the reads of u below), slots 1+j = sum_i
    // M[i][j] u[i] (thread (row group, j), coalesced rows of M).  Fixed
    // combination order.
    auto own_partials = [&](auto sqval, const double* u, const double* M, double* partials, bool sync_mid = false) {
        double sq = 0.0;
        for (long long i = r0 + tid; i < r1; i += DCG_NT) {
            const double q = sqval(i);
            sq = add_rn(sq, mul_rn(q, q));
        }
        if (sync_mid && M) cta_sync();
        double c = 0.0;
        if (M) {
            const int j = tid & (swk - 1), grp = tid / swk, ngrp = DCG_NT / swk;
            if (j < k) {
#pragma unroll 4
                for (long long i = r0 + grp; i < r1; i += ngrp) c = fma(__ldg(M + i * k + j), ld_cg(u + i), c);
            }
            if (swk < 32)
                for (int o = swk; o < 32; o <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        sq = warp_sum(sq);
        if (lane == 0) s_tmp[warp] = sq;
        if (M) {
            if (swk <= 32) {
                if (lane < swk) s_scr[warp * 32 + lane] = c;
            } else {
                s_scr[tid] = c;
            }
        }
        cta_sync();
        double* const mine = partials + (long long)blockIdx.x * a.ps;
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < DCG_NW; ++w) t += s_tmp[w];
            mine[0] = t;
        }
        if (M && tid < k) {
            double t = 0.0;
            if (swk <= 32) {
                for (int w = 0; w < DCG_NW; ++w) t += s_scr[w * 32 + tid];
            } else {
                for (int g = 0; g < DCG_NT / swk; ++g) t += s_scr[g * swk + tid];
            }
            mine[1 + tid] = t;
        }
    };

    // ---------------- prologue: norm_b and the warm-start correction ----------
    // deflated_cg_solve: r_prev = b - A x_prev ; x0 = x_prev + W chol_solve(L, W' r_prev)
    if (a.warm && deflate) {
        if (a.ax0) {
            // A x_prev came from a product enqueued before the launch (it
            // overlaps the Ritz pencil in the pipelined Newton step)
            for (long long i = r0 + tid; i < r1; i += DCG_NT) a.r[i] = sub_rn(a.b[i], ld_cg(a.ax0 + i));
            cta_sync();
        } else {
            gemv(a.x0, [&](long long i, double t) {
                const double ax = s ? add_rn(mul_rn(shift, a.x0[i]), mul_rn(s[i], t))
                                    : add_rn(mul_rn(shift, a.x0[i]), t);
                a.r[i] = sub_rn(a.b[i], ax);
            });
            if constexpr (STRAT != STRAT_ROWS) GSYNC(); else cta_sync();
        }
        // slot0 = b'b, slots 1.. = W' r_prev
        own_partials([&](long long i) { return a.b[i]; }, a.r, a.W, a.partials);
    } else {
        own_partials([&](long long i) { return a.b[i]; }, nullptr, nullptr, a.partials);
    }
    GSYNC();
    reduce_partials(a.partials, G, a.ps, (a.warm && deflate) ? nslots : 1, s_c, s_scr);
    const double norm_b = sqrt(s_c[0]);
    if (norm_b == 0.0) {
        // solvers.py:142-147: x = 0 (not x0), history [0.0], log.r = [0]
        for (long long i = r0 + tid; i < r1; i += blockDim.x) {
            a.x[i] = 0.0;
            if (a.logR) a.logR[i] = 0.0;
        }
        if constexpr (kPk) sym_ring_drain(s_g, ring_seq, pending);
        if (blockIdx.x == 0 && tid == 0) {
            a.history[0] = 0.0;
            put_status(a.st, DCG_OK, k, 0, 0, 0, 0.0, 0.0);   // 0 iterations, 0 stored
        }
        return;
    }
    if (a.warm && deflate) {
        solve_mu(s_L, s_rd, k, s_c + 1, s_mu);
        for (long long i = r0 + tid; i < r1; i += DCG_NT) a.x[i] = add_rn(a.x0[i], row_dot(a.W, i, s_mu));
    } else {
        for (long long i = r0 + tid; i < r1; i += DCG_NT) a.x[i] = a.x0[i];
    }
    GSYNC();

    // ---------------- r0 = b - A x0 ; mu ; p0 ------------------------------------
    if (a.warm && deflate) {
        // x0 = x_prev + W c, so A x0 = A x_prev + (A W) c with the basis' own
        // A W (refresh_basis, recycle.py:90, for this A): r0 = r_prev - (AW) c
        // (solvers.py:237-238 then 150 form b - A x0 with one more product;
        // the two are equal up to rounding, and W' r0 = 0 holds to rounding)
        for (long long i = r0 + tid; i < r1; i += DCG_NT) a.r[i] = sub_rn(ld_cg(a.r + i), row_dot(a.AW, i, s_mu));
        cta_sync();
    } else if (a.ax0) {
        // plain CG warm-started at x0 = x_prev (cg_solve, solvers.py:207-219):
        // A x0 is the product computed ahead of the launch
        for (long long i = r0 + tid; i < r1; i += DCG_NT) a.r[i] = sub_rn(a.b[i], ld_cg(a.ax0 + i));
        cta_sync();
    } else {
        gemv(a.x, [&](long long i, double t) {
            const double xi = ld_cg(a.x + i);
            const double ax = s ? add_rn(mul_rn(shift, xi), mul_rn(s[i], t)) : add_rn(mul_rn(shift, xi), t);
            a.r[i] = sub_rn(a.b[i], ax);
        });
        if constexpr (STRAT != STRAT_ROWS) GSYNC(); else cta_sync();
    }
    own_partials([&](long long i) { return ld_cg(a.r + i); }, a.r, deflate ? a.AW : nullptr, a.partials);
    GSYNC();
    reduce_partials(a.partials, G, a.ps, nslots, s_c, s_scr);
    double rr = s_c[0];
    if (deflate) solve_mu(s_L, s_rd, k, s_c + 1, s_mu);
    double rel = sqrt(rr) / norm_b;
    long long it = 0;
    const long long ell = a.ell;
    bool cont = (rel > a.tol) && (it < a.max_iters);
    // p0 (+ log r0, p0, mu0)
    for (long long i = r0 + tid; i < r1; i += DCG_NT) {
        const double ri = ld_cg(a.r + i);
        const double pi = deflate ? sub_rn(ri, row_dot(a.W, i, s_mu)) : ri;
        a.p[i] = pi;
        if (a.logR) a.logR[i] = ri;
        if (cont && it < ell) a.logP[i] = pi;
    }
    if (blockIdx.x == 0) {
        if (tid == 0) a.history[0] = rel;
        if (deflate && cont && it < ell && tid < k) a.logMu[tid] = s_mu[tid];   // stride kmax
    }
    GSYNC();

    // ---------------- main loop ------------------------------------------------
    PHASE(13);   // prologue
    while (cont) {
        // phase G: Ap, partial p'Ap
        double dpart = 0.0;
        gemv(a.p, [&](long long i, double t) {
            const double pi = ld_cg(a.p + i);
            const double api = s ? add_rn(mul_rn(shift, pi), mul_rn(s[i], t)) : add_rn(mul_rn(shift, pi), t);
            a.ap[i] = api;
            dpart = fma(pi, api, dpart);
        });
        // p'Ap goes to the second partials buffer: no grid barrier separates this
        // read from the r'r publish below, so they must not share slots.
        double* const dparts = a.partials + (long long)G * a.ps;
        PHASE(2);
        dpart = block_sum(dpart, s_tmp);
        if (tid == 0) dparts[(long long)blockIdx.x * a.ps] = dpart;
        PHASE(3);
        GSYNC();
        PHASE(4);
        reduce_partials(dparts, G, a.ps, 1, s_c, s_scr);
        PHASE(5);
        const double d = s_c[0];
        if (d <= 0.0) {   // solvers.py:170-172 (NaN falls through, as in numpy)
            if constexpr (kPk) sym_ring_drain(s_g, ring_seq, pending);
            if (blockIdx.x == 0 && tid == 0) {
                put_status(a.st, DCG_E_BREAKDOWN, k, it, it, 0, 0.0, 0.0);
            }
            return;
        }
        const double alpha = rr / d;
        ++it;
        const bool recompute = (a.recompute > 0) && (it % a.recompute == 0);
        const bool log_r = (it - 1) < ell;
        if (recompute) {
            for (long long i = r0 + tid; i < r1; i += blockDim.x)
                a.x[i] = add_rn(a.x[i], mul_rn(alpha, a.p[i]));
            GSYNC();
            gemv(a.x, [&](long long i, double t) {
                const double xi = ld_cg(a.x + i);
                const double ax = s ? add_rn(mul_rn(shift, xi), mul_rn(s[i], t)) : add_rn(mul_rn(shift, xi), t);
                a.r[i] = sub_rn(a.b[i], ax);
            });
            if constexpr (STRAT != STRAT_ROWS) GSYNC();
            cta_sync();
            PHASE(6);
            own_partials(
                [&](long long i) {
                    const double ri = ld_cg(a.r + i);
                    if (log_r) a.logR[it * n + i] = ri;
                    return ri;
                },
                a.r, deflate ? a.AW : nullptr, a.partials);
        } else {
            PHASE(6);
            // x += alpha p and r -= alpha Ap on the own rows, inside the r'r loop
            own_partials(
                [&](long long i) {
                    const double pi = a.p[i];
                    a.x[i] = add_rn(a.x[i], mul_rn(alpha, pi));
                    const double ri = sub_rn(ld_cg(a.r + i), mul_rn(alpha, ld_cg(a.ap + i)));
                    a.r[i] = ri;
                    if (log_r) a.logR[it * n + i] = ri;
                    return ri;
                },
                a.r, deflate ? a.AW : nullptr, a.partials, true);
        }
        PHASE(7);
        GSYNC();
        PHASE(8);
        reduce_partials(a.partials, G, a.ps, nslots, s_c, s_scr);
        PHASE(9);
        const double rr_new = s_c[0];
        const double beta = rr_new / rr;
        rel = sqrt(rr_new) / norm_b;
        if (blockIdx.x == 0 && tid == 0) {
            a.history[it] = rel;
            if (log_r) {
                a.logD[it - 1] = d;
                a.logAlpha[it - 1] = alpha;
                a.logBeta[it - 1] = beta;
            }
        }
        if (deflate) solve_mu(s_L, s_rd, k, s_c + 1, s_mu);
        PHASE(10);
        cont = (rel > a.tol) && (it < a.max_iters);
        const bool log_p = cont && it < ell;
        for (long long i = r0 + tid; i < r1; i += DCG_NT) {
            const double ri = ld_cg(a.r + i);
            const double pi = deflate ? sub_rn(add_rn(mul_rn(beta, a.p[i]), ri), row_dot(a.W, i, s_mu))   // beta*p + r - W mu
                                      : add_rn(ri, mul_rn(beta, a.p[i]));                                  // r + beta*p
            a.p[i] = pi;
            if (log_p) a.logP[it * n + i] = pi;
        }
        if (log_p && deflate && blockIdx.x == 0 && tid < k) a.logMu[it * kmax + tid] = s_mu[tid];
        rr = rr_new;
        PHASE(11);
        GSYNC();
        PHASE(12);
    }
    if constexpr (kPk) sym_ring_drain(s_g, ring_seq, pending);
    if (blockIdx.x == 0 && tid == 0) put_status(a.st, DCG_OK, k, 0, it, (it < ell) ? it : ell, rel, norm_b);
}

// The persistent kernel: the solve, then the last CTA out hands the barrier
// words back at zero (dcg_sync_exit) for the next launch.
template <int STRAT>
__global__ void __launch_bounds__(DCG_NT, 1) dcg_solve_kernel(SolveArgs a) {
    solve_body<STRAT>(a);
    if (threadIdx.x == 0) dcg_sync_exit(a.bar, gridDim.x);
}

}  // namespace

size_t dcg_solve_smem_bytes(long long n, int k, int strat, int dim, int nteam) {
    return sizeof(double) * (size_t)(gemv_region_doubles(strat, n, dim, nteam) + k * k + DCG_MAX_K + DCG_MAX_K + 2 +
                                     DCG_MAX_K + 64 + DCG_NT);
}

size_t dcg_rbf_mma_operand_doubles(long long n, int dim);
int dcg_rbf_mma_teams(const dcg_context* ctx, int dim, size_t other_bytes);
RbfMma dcg_rbf_mma_params(const dcg_operator* op, double* operands, int nteam);
int dcg_rbf_mma_prep(const dcg_context* ctx, cudaStream_t st, const RbfMma& p);

// per-phase device timers of the last dcg_solve run with DCG_PHASE_TIMERS set
static unsigned long long* g_phase_timers = nullptr;

// Developer diagnostic: the 16 phase accumulators (ns, CTA 0) of the last
// solve run with DCG_PHASE_TIMERS=1 (slot order as printed on stderr: pass1,
// gsync_mv, pass2+epi, ...).  DCG_E_CONFIG if none was recorded.
extern "C" __attribute__((visibility("default"))) int dcg_debug_phase_timers(unsigned long long* out16) {
    if (!g_phase_timers || !out16) return DCG_E_CONFIG;
    DCG_CUDA(cudaMemcpy(out16, g_phase_timers, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return DCG_OK;
}
// ... and the per-CTA pass-1 / pass-2 accumulators (slots 16 .. 16 + 2 G)
extern "C" __attribute__((visibility("default"))) int dcg_debug_phase_timers_all(unsigned long long* out, int nslots) {
    if (!g_phase_timers || !out || nslots < 0 || nslots > 1024) return DCG_E_CONFIG;
    DCG_CUDA(cudaMemcpy(out, g_phase_timers, (size_t)nslots * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return DCG_OK;
}

static int solve_impl(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_b,
                      const double* d_x0, const dcg_basis* basis, const dcg_solver_config* cfg, double* d_x,
                      dcg_krylov_log* log, double* d_history, dcg_solve_info* out, long long* info,
                      const long long* d_kuse, void* d_status, const double* d_ax0 = nullptr) {
    if (!ctx || !op || !cfg || !d_b || !d_x0 || !d_x || !d_history) return DCG_E_CONFIG;
    if (info) *info = 0;
    const long long n = op->n;
    if (op->kind != DCG_OP_DENSE && op->kind != DCG_OP_DENSE_SYM && op->kind != DCG_OP_RBF) return DCG_E_UNSUPPORTED;
    const bool sym = op->kind == DCG_OP_DENSE_SYM && ((reinterpret_cast<uintptr_t>(d_x0) | reinterpret_cast<uintptr_t>(op->d_s)) & 15) == 0;
    const int strat = op->kind == DCG_OP_RBF ? STRAT_RBF : (sym ? (op->d_kp ? STRAT_SYMPK : STRAT_SYM) : STRAT_ROWS);
    if (strat != STRAT_RBF && strat != STRAT_SYMPK && !op->d_k) return DCG_E_CONFIG;   // packed-only storage
    if (op->row0 != 0 || op->rows != n) return DCG_E_UNSUPPORTED;   // sharded solves: host loop
    if (strat == STRAT_RBF) {
        if (!op->d_x || op->dim < 1) return DCG_E_CONFIG;
        if (op->dim > DCG_RBF_MAX_DIM) return DCG_E_UNSUPPORTED;
    } else if (op->ldk < n || (op->ldk & 1) || (reinterpret_cast<uintptr_t>(op->d_k) & 15)) {
        return DCG_E_CONFIG;
    }
    if (!(cfg->tol > 0.0) || cfg->ell < 0 || cfg->recompute_residual_every < 0) return DCG_E_CONFIG;
    const int k = basis ? (int)basis->k : 0;
    if (k < 0) return DCG_E_CONFIG;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    if (k > 0 && (!basis->d_w || !basis->d_aw || !basis->d_chol)) return DCG_E_CONFIG;
    const long long ell = log ? log->ell : 0;
    if (cfg->ell > 0 && (!log || ell < cfg->ell || !log->d_p || !log->d_r || !log->d_d ||
                         !log->d_alpha || !log->d_beta || (k > 0 && !log->d_mu)))
        return DCG_E_CONFIG;
    const long long max_iters = cfg->max_iters > 0 ? cfg->max_iters : 10 * n;

    const int G = ctx->solve_blocks;
    const int ps = ((1 + k) + 1) & ~1;
    const size_t vec = sizeof(double) * (size_t)((n + 31) & ~31LL);
    const size_t tiles = (strat != STRAT_ROWS) ? (size_t)sym_ntiles(n) : 0;
    const size_t operands = strat == STRAT_RBF ? sizeof(double) * dcg_rbf_mma_operand_doubles(n, (int)op->dim) + 256 : 0;
    const size_t need = 3 * vec + 2 * sizeof(double) * (size_t)G * ps + 1024 + 2 * sizeof(double) * tiles * DCG_TB +
                        operands;
    int rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    char* w = static_cast<char*>(ctx->ws);
    SolveArgs a;
    memset(&a, 0, sizeof(a));
    a.K = op->d_k;
    a.symtbl = nullptr;
    a.Kp = strat == STRAT_SYMPK ? op->d_kp : nullptr;
    a.ldk = op->ldk;
    a.n = n;
    a.s = op->d_s;
    a.shift = op->shift;
    a.b = d_b;
    a.x0 = d_x0;
    a.ax0 = d_ax0;
    a.x = d_x;
    a.k = k;
    a.kdev = k ? d_kuse : nullptr;
    a.W = k ? basis->d_w : nullptr;
    a.AW = k ? basis->d_aw : nullptr;
    a.L = k ? basis->d_chol : nullptr;
    a.warm = k > 0;
    a.tol = cfg->tol;
    a.max_iters = max_iters;
    a.ell = cfg->ell;
    a.recompute = cfg->recompute_residual_every;
    a.logP = log ? log->d_p : nullptr;
    a.logR = log ? log->d_r : nullptr;
    a.logD = log ? log->d_d : nullptr;
    a.logAlpha = log ? log->d_alpha : nullptr;
    a.logBeta = log ? log->d_beta : nullptr;
    a.logMu = log ? log->d_mu : nullptr;
    a.history = d_history;
    a.r = reinterpret_cast<double*>(w);
    a.p = reinterpret_cast<double*>(w + vec);
    a.ap = reinterpret_cast<double*>(w + 2 * vec);
    a.partials = reinterpret_cast<double*>(w + 3 * vec);
    a.ps = ps;
    {
        // status block and barrier words on their own 256-byte line, then the tile partials
        const size_t st_off = (3 * vec + 2 * sizeof(double) * (size_t)G * ps + 255) & ~size_t(255);
        a.st = reinterpret_cast<DevStatus*>(w + st_off);
        a.colpart = reinterpret_cast<double*>(w + st_off + 256);
        a.rowpart = a.colpart + tiles * DCG_TB;
    }

    cudaStream_t st = as_stream(stream);
    const int nteam = strat == STRAT_RBF ? dcg_rbf_mma_teams(ctx, (int)op->dim,
                                                             dcg_solve_smem_bytes(n, k, strat, (int)op->dim, 0))
                                         : 1;
    const size_t smem = dcg_solve_smem_bytes(n, k, strat, (int)op->dim, nteam);
    const void* kfn = strat == STRAT_RBF     ? (const void*)dcg_solve_kernel<STRAT_RBF>
                      : strat == STRAT_SYMPK ? (const void*)dcg_solve_kernel<STRAT_SYMPK>
                      : strat == STRAT_SYM   ? (const void*)dcg_solve_kernel<STRAT_SYM>
                                             : (const void*)dcg_solve_kernel<STRAT_ROWS>;
    if (strat == STRAT_RBF) {
        double* opnd = reinterpret_cast<double*>(
            (reinterpret_cast<uintptr_t>(a.rowpart + tiles * DCG_TB) + 255) & ~uintptr_t(255));
        a.rbf = dcg_rbf_mma_params(op, opnd, nteam);
        rc = dcg_rbf_mma_prep(ctx, st, a.rbf);
        if (rc) return rc;
    } else {
        memset(&a.rbf, 0, sizeof(a.rbf));
    }
    if (strat == STRAT_SYM || strat == STRAT_SYMPK) {
        a.symtbl = dcg_sym_table(ctx, st, n, G);
        if (!a.symtbl) return DCG_E_CUDA;
    }
    if (strat == STRAT_RBF) DCG_SMEM_ATTR(dcg_solve_kernel<STRAT_RBF>, smem);
    else if (strat == STRAT_SYMPK) DCG_SMEM_ATTR(dcg_solve_kernel<STRAT_SYMPK>, smem);
    else if (strat == STRAT_SYM) DCG_SMEM_ATTR(dcg_solve_kernel<STRAT_SYM>, smem);
    else DCG_SMEM_ATTR(dcg_solve_kernel<STRAT_ROWS>, smem);
    // no memset before the launch: the barrier words are the context's
    // persistent line (returned to zero by the kernel), and the kernel writes
    // the whole status block -- in the asynchronous form straight into the
    // caller's block (no device-to-device copy behind the kernel)
    a.bar = dcg_sync_line(ctx, DCG_SW_SOLVE);
    if (d_status) a.st = static_cast<DevStatus*>(d_status);
    // DCG_PHASE_TIMERS=1: per-phase device time of CTA 0 printed per solve
    // (developer diagnostic; costs one predicated branch per phase otherwise).
    unsigned long long*& d_timers = g_phase_timers;
    const bool timers = getenv("DCG_PHASE_TIMERS") != nullptr;
    a.timers = nullptr;
    if (timers) {
        if (!d_timers) DCG_CUDA(cudaMalloc(&d_timers, 1024 * sizeof(unsigned long long)));
        DCG_CUDA(cudaMemsetAsync(d_timers, 0, 1024 * sizeof(unsigned long long), st));
        a.timers = d_timers;
    }
    void* args[] = {&a};
    if (!d_status) DCG_CUDA(cudaEventRecord(ctx->ev0, st));   // synchronous form: device_ms
    DCG_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(DCG_NT), args, smem, st));
    dcg_count_launch();
    if (d_status) return DCG_OK;   // asynchronous form: nothing waits here
    DCG_CUDA(cudaEventRecord(ctx->ev1, st));
    rc = dcg_host_reserve(ctx, sizeof(DevStatus));
    if (rc) return rc;
    DevStatus* hs = static_cast<DevStatus*>(ctx->host);
    DCG_CUDA(cudaMemcpyAsync(hs, a.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    DCG_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    if (timers) {
        unsigned long long h[16];
        DCG_CUDA(cudaMemcpy(h, d_timers, sizeof(h), cudaMemcpyDeviceToHost));
        const long long its = hs->count > 0 ? hs->count : 1;
        static const char* names[16] = {"pass1", "gsync_mv", "pass2+epi", "pAp_sum", "gsync_d", "reduce_d",
                                        "x_r_upd", "rr_partials", "gsync_rr", "reduce_rr", "mu_solve",
                                        "p_upd", "gsync_end", "prologue", "-", "gemv_entry"};
        fprintf(stderr, "phase_timers n=%lld k=%d its=%lld sym=%d (us per iteration; prologue total):", n, k,
                hs->count, (int)sym);
        for (int q = 0; q < 16; ++q)
            if (h[q]) fprintf(stderr, " %s=%.2f", names[q], q == 13 ? h[q] * 1e-3 : h[q] * 1e-3 / its);
        fprintf(stderr, "\n");
        if (sym) {
            unsigned long long hc[1024];
            DCG_CUDA(cudaMemcpy(hc, d_timers, sizeof(hc), cudaMemcpyDeviceToHost));
            for (int ph = 0; ph < 2; ++ph) {
                const unsigned long long* v = hc + 16 + ph * G;
                int imin = 0, imax = 0;
                double sum = 0;
                for (int b = 0; b < G; ++b) {
                    sum += v[b];
                    if (v[b] < v[imin]) imin = b;
                    if (v[b] > v[imax]) imax = b;
                }
                const double nmv = (double)(its + 2);
                fprintf(stderr, "  pass%d per-CTA us/matvec: min %.2f (cta %d) mean %.2f max %.2f (cta %d); first8:", ph + 1,
                        v[imin] * 1e-3 / nmv, imin, sum / G * 1e-3 / nmv, v[imax] * 1e-3 / nmv, imax);
                for (int b = 0; b < 8; ++b) fprintf(stderr, " %.1f", v[b] * 1e-3 / nmv);
                fprintf(stderr, " last4:");
                for (int b = G - 4; b < G; ++b) fprintf(stderr, " %.1f", v[b] * 1e-3 / nmv);
                fprintf(stderr, "\n");
            }
        }
    }
    if (hs->status != DCG_OK) {
        if (info) *info = hs->info;
        return hs->status;
    }
    if (out) {
        out->iterations = hs->count;
        out->stored = hs->aux;
        out->rel_residual = hs->value;
        out->norm_b = hs->value2;
        out->converged = hs->value <= cfg->tol ? 1 : 0;
        out->termination = out->converged ? 0 : 1;
        out->device_ms = ms;
    }
    return DCG_OK;
}

extern "C" int dcg_solve(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_b,
                         const double* d_x0, const dcg_basis* basis, const dcg_solver_config* cfg,
                         double* d_x, dcg_krylov_log* log, double* d_history, dcg_solve_info* out,
                         long long* info) {
    return solve_impl(ctx, stream, op, d_b, d_x0, basis, cfg, d_x, log, d_history, out, info, nullptr, nullptr);
}

// Enqueue-only form (no host synchronisation).  d_kuse (optional, device):
// the basis columns in use, as left by dcg_refresh_basis_async; the basis'
// k is the layout maximum.  d_status (64 bytes, device) receives the status
// block: int32 status, int32 columns used, int64 info, int64 iterations,
// int64 stored log entries, f64 relative residual, f64 norm_b.  d_ax0
// (optional): A x0, computed ahead (the warm-start correction's first product).
extern "C" int dcg_solve_async(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_b,
                               const double* d_x0, const dcg_basis* basis, const dcg_solver_config* cfg,
                               double* d_x, dcg_krylov_log* log, double* d_history, const long long* d_kuse,
                               void* d_status, const double* d_ax0) {
    if (!d_status) return DCG_E_CONFIG;
    return solve_impl(ctx, stream, op, d_b, d_x0, basis, cfg, d_x, log, d_history, nullptr, nullptr, d_kuse,
                      d_status, d_ax0);
}
