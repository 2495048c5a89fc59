// Small dense linear algebra on one CTA (kernel K5 of SURVEY.md section 2).
//
// Everything here is at most DCG_MAX_T x DCG_MAX_T (the harmonic pencil is
// k_prev + m <= k + ell).  The reference runs these as scalar Cython loops
// (_core.pyx:47-94, 135-177) driven from linalg.py:74-191; the device versions
// keep the reference's thresholds and operation order where it is inherently
// serial (Cholesky pivots, forward substitution) with non-contracted fp64
// arithmetic, and parallelise only independent work:
//   - Cholesky: column j serial, rows i > j in parallel (same per-element sum order);
//   - triangular solves of many right-hand sides: one warp per column;
//   - the symmetric eigensolver is Jacobi with the reference's skip rule and
//     convergence test (linalg.py:139-165) but a parallel round-robin pair
//     ordering (T/2 disjoint rotations per step), so a sweep costs T-1 barrier
//     rounds instead of T(T-1)/2 sequential rotations.  Eigenpairs agree with
//     the cyclic order to rounding; spans, not signs, are what callers use.
#include "common.cuh"

#define SD_NT 512
// pencils up to this order keep all working matrices in shared memory (4 T^2 doubles)
#define DCG_PENCIL_SMEM_T 80
// the pencil runs one warp per Jacobi pair: 32 warps cover T <= 64
#define PENCIL_NT 1024

// ---------------------------------------------------------------------------
// Cholesky with the reference's pivot rule (acc <= pivot_tol fails at j).
// A, L: row-major with leading dimensions; L's upper triangle is zeroed.
// Returns -1 on success or the failing pivot index.  All CTA threads call.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int cta_cholesky(const double* A, int lda, int n, double pivot_tol, double* L, int ldl,
                            double* s_scal) {
    // Right-looking in place in L: after column t is final, every trailing
    // element (i, c), t < c <= i, subtracts L_it L_ct.  Each element therefore
    // sees its subtractions in ascending t, rounded separately - the same
    // arithmetic as the reference's left-looking dot products
    // (_core.pyx:47-66) - but a column costs three CTA barriers and one
    // parallel trailing update instead of a serial diagonal chain.
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e / n, c = e - (e / n) * n;
        L[i * ldl + c] = (c <= i) ? A[i * lda + c] : 0.0;
    }
    cta_sync();
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            const double acc = L[j * ldl + j];
            if (acc <= pivot_tol) {
                s_scal[0] = 1.0;
            } else {
                s_scal[0] = 0.0;
                L[j * ldl + j] = sqrt(acc);
            }
        }
        cta_sync();
        if (s_scal[0] != 0.0) {
            cta_sync();
            return j;
        }
        const double ljj = L[j * ldl + j];
        for (int i = j + 1 + tid; i < n; i += blockDim.x) L[i * ldl + j] = div_rn(L[i * ldl + j], ljj);
        cta_sync();
        for (int i = j + 1 + warp; i < n; i += nw) {
            const double lij = L[i * ldl + j];
            for (int c = j + 1 + lane; c <= i; c += 32)
                L[i * ldl + c] = sub_rn(L[i * ldl + c], mul_rn(lij, L[c * ldl + j]));
        }
        cta_sync();
    }
    return -1;
}

// 1e-14 * max(max(diag), 0)   (linalg.py:74-76), diag of A restricted to idx[0..n)
__device__ __forceinline__ double cta_pivot_tol(const double* A, int lda, const int* idx, int n, double* red) {
    double m = -INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ii = idx ? idx[i] : i;
        m = fmax(m, A[ii * lda + ii]);
    }
    m = block_max(m, red);
    if (n == 0) m = 0.0;
    return 1e-14 * fmax(m, 0.0);
}

// Warp-level forward substitution: y = L^-1 b for one right-hand side
// (b, y with strides), reference order per element (_core.pyx:69-80).
// Lanes own rows lane + 32u.
static __device__ __forceinline__ void warp_solve_lower(const double* L, int ldl, int n, const double* b, int bstride,
                                 double* y, int ystride) {
    const int lane = threadIdx.x & 31;
    double a[(DCG_MAX_T + 31) / 32];
#pragma unroll
    for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
        const int i = lane + 32 * u;
        a[u] = (i < n) ? b[i * bstride] : 0.0;
    }
    for (int j = 0; j < n; ++j) {
        const int uj = j >> 5;
        double accj = 0.0;
#pragma unroll
        for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u)
            if (u == uj) accj = __shfl_sync(0xffffffffu, a[u], j & 31);
        const double yj = div_rn(accj, L[j * ldl + j]);
#pragma unroll
        for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
            const int i = lane + 32 * u;
            if (i == j) a[u] = yj;
            else if (i > j && i < n) a[u] = sub_rn(a[u], mul_rn(L[i * ldl + j], yj));
        }
    }
#pragma unroll
    for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
        const int i = lane + 32 * u;
        if (i < n) y[i * ystride] = a[u];
    }
}

// Column-parallel forward substitution Y = L^-1 B (n x n): a thread per
// column, left-looking.  Element i takes the same operation sequence as the
// right-looking warp_solve_lower -- b_i - L_i0 y_0 - L_i1 y_1 - ... in that
// order, unfused, then one division -- so the results are bit-identical; the
// chain is per thread instead of a warp shuffle per step.  B(i, c) =
// B[i * brs + c * bcs], Y(i, c) = Y[i * yrs + c * ycs].
static __device__ __forceinline__ void cta_solve_lower_cols(const double* L, int n, const double* B, int brs, int bcs,
                                                            double* Y, int yrs, int ycs) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        for (int i = 0; i < n; ++i) {
            double a = B[i * brs + c * bcs];
            const double* li = L + i * n;
            for (int j = 0; j < i; ++j) a = sub_rn(a, mul_rn(li[j], Y[j * yrs + c * ycs]));
            Y[i * yrs + c * ycs] = div_rn(a, li[i]);
        }
    }
}

// Warp-level back substitution x = L^-T b (wavefront order).
static __device__ __forceinline__ void warp_solve_lower_trans(const double* L, int ldl, int n, const double* b, int bstride,
                                       double* x, int xstride) {
    const int lane = threadIdx.x & 31;
    double a[(DCG_MAX_T + 31) / 32];
#pragma unroll
    for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
        const int i = lane + 32 * u;
        a[u] = (i < n) ? b[i * bstride] : 0.0;
    }
    for (int j = n - 1; j >= 0; --j) {
        const int uj = j >> 5;
        double accj = 0.0;
#pragma unroll
        for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u)
            if (u == uj) accj = __shfl_sync(0xffffffffu, a[u], j & 31);
        const double xj = div_rn(accj, L[j * ldl + j]);
#pragma unroll
        for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
            const int i = lane + 32 * u;
            if (i == j) a[u] = xj;
            else if (i < j) a[u] = sub_rn(a[u], mul_rn(L[j * ldl + i], xj));
        }
    }
#pragma unroll
    for (int u = 0; u < (DCG_MAX_T + 31) / 32; ++u) {
        const int i = lane + 32 * u;
        if (i < n) x[i * xstride] = a[u];
    }
}

// ---------------------------------------------------------------------------
// Parallel-order Jacobi eigensolver on a symmetric T x T matrix A (row-major,
// leading dimension T, typically shared memory); V receives eigenvectors as
// columns (unsorted).  Returns 0, or the sweep budget on NoConvergence.
//
// Same method as linalg.sym_eigen / _core.jacobi_sweep (linalg.py:139-165,
// _core.pyx:135-177): convergence test off(A) <= rtol ||A||_F before every
// sweep, the skip rule |a_pp| + 100|a_pq| == |a_pp| (and for q) zeroes a_pq,
// t = sgn(tau) / (|tau| + sqrt(1 + tau^2)), c = 1 / sqrt(1 + t^2), s = t c.
// The rotations of a sweep are applied in the circle-method parallel order
// (T/2 disjoint pairs per round) instead of the row-cyclic order, and the
// rotation parameters come from hardware reciprocal / rsqrt approximations
// refined by two Newton steps (working precision): the solver is a chain of
// ~8 sweeps x (T - 1) dependent rounds, so each round's latency is what
// counts.  Every thread updates at most a couple of 2 x 2 blocks per round
// (a 32 x 16 grid over row pairs x column pairs), so the round is one short
// dependent chain per thread.
// ---------------------------------------------------------------------------
#define JAC_NT 512   // == the pencil / eigen kernels' CTA size
__device__ __forceinline__ void jac_sync() { cta_sync(); }
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

// Rotation (c, s, mode) of the pair in circle slot `slot` for `round` from
// the current matrix: mode 0 identity (padding player), 1 zero a_pq (skip
// rule), 2 rotate.  Deterministic: every thread that needs a slot's rotation
// computes the same bits.
__device__ __forceinline__ void jac_rotation(const double* A, int T, int Te, int slot, int round, int& p, int& q,
                                             int& mode, double& c, double& sn) {
    int pa = slot == 0 ? Te - 1 : slot - 1 + round;
    if (slot != 0 && pa >= Te - 1) pa -= Te - 1;
    int pb = Te - 2 - slot + round;
    if (pb >= Te - 1) pb -= Te - 1;
    p = min(pa, pb);
    q = max(pa, pb);
    c = 1.0;
    sn = 0.0;
    mode = 0;
    if (q >= T) return;
    const double apq = A[p * T + q];
    const double app = A[p * T + p], aqq = A[q * T + q];
    const double g = 100.0 * fabs(apq);
    if (add_rn(fabs(app), g) == fabs(app) && add_rn(fabs(aqq), g) == fabs(aqq)) {
        mode = 1;
    } else if (apq != 0.0) {
        const double tau = (aqq - app) * fast_rcp(2.0 * apq);
        const double at = fabs(tau);
        double t;
        if (at < 1e100) {
            const double w = fma(tau, tau, 1.0);
            t = fast_rcp(at + w * fast_rsqrt(w));
        } else {
            t = 0.5 * fast_rcp(at);
        }
        if (tau < 0.0) t = -t;
        c = fast_rsqrt(fma(t, t, 1.0));
        sn = t * c;
        mode = 2;
    }
}

// Double-buffered variant: a round reads A (current) and writes Anext, every
// thread recomputing the rotations of its own row and column pairs, so a
// round needs one CTA barrier instead of two and no rotation broadcast.
// Same rotations, same order of application as cta_jacobi; the result is
// left in A.  `Anext` holds T * T doubles of shared memory.
__device__ int cta_jacobi2(double* A, double* Anext, double* V, int T, int max_sweeps, double rtol, double* red) {
    const int tid = threadIdx.x;
    __shared__ int s_result2;
    for (int e = tid; e < T * T; e += blockDim.x) V[e] = (e / T == e % T) ? 1.0 : 0.0;
    double f2 = 0.0;
    for (int e = tid; e < T * T; e += blockDim.x) f2 = fma(A[e], A[e], f2);
    const double frob = sqrt(block_sum(f2, red));
    if (frob == 0.0) return 0;   // zeros and identity (linalg.py:153-154)
    const int Te = T + (T & 1);
    const int np = Te / 2;
    const int nblk = np * np;
    double* cur = A;
    double* nxt = Anext;
    auto offdiag = [&]() {
        double o2 = 0.0;
        for (int e = tid; e < T * T; e += blockDim.x) {
            const int i = e / T, j = e - (e / T) * T;
            if (i != j) o2 = fma(cur[e], cur[e], o2);
        }
        return sqrt(block_sum(o2, red));
    };
    bool converged = offdiag() <= rtol * frob;
    for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
        for (int round = 0; round < Te - 1; ++round) {
            for (int blk = tid; blk < nblk; blk += blockDim.x) {
                const int ba = blk / np, bb = blk - (blk / np) * np;
                int pa0, pa1, ma, pb0, pb1, mb;
                double ca, sa, cb, sb;
                jac_rotation(cur, T, Te, ba, round, pa0, pa1, ma, ca, sa);
                if (bb == ba) {
                    pb0 = pa0; pb1 = pa1; mb = ma; cb = ca; sb = sa;
                } else {
                    jac_rotation(cur, T, Te, bb, round, pb0, pb1, mb, cb, sb);
                }
                const bool ra1v = pa1 < T, cb1v = pb1 < T;
                double x00 = cur[pa0 * T + pb0];
                double x01 = cb1v ? cur[pa0 * T + pb1] : 0.0;
                double x10 = ra1v ? cur[pa1 * T + pb0] : 0.0;
                double x11 = (ra1v && cb1v) ? cur[pa1 * T + pb1] : 0.0;
                if (mb == 2) {
                    const double y00 = sub_rn(mul_rn(cb, x00), mul_rn(sb, x01));
                    const double y01 = add_rn(mul_rn(sb, x00), mul_rn(cb, x01));
                    const double y10 = sub_rn(mul_rn(cb, x10), mul_rn(sb, x11));
                    const double y11 = add_rn(mul_rn(sb, x10), mul_rn(cb, x11));
                    x00 = y00; x01 = y01; x10 = y10; x11 = y11;
                }
                if (ma == 2) {
                    const double y00 = sub_rn(mul_rn(ca, x00), mul_rn(sa, x10));
                    const double y10 = add_rn(mul_rn(sa, x00), mul_rn(ca, x10));
                    const double y01 = sub_rn(mul_rn(ca, x01), mul_rn(sa, x11));
                    const double y11 = add_rn(mul_rn(sa, x01), mul_rn(ca, x11));
                    x00 = y00; x01 = y01; x10 = y10; x11 = y11;
                }
                if (ba == bb && ma != 0) { x01 = 0.0; x10 = 0.0; }
                nxt[pa0 * T + pb0] = x00;
                if (cb1v) nxt[pa0 * T + pb1] = x01;
                if (ra1v) nxt[pa1 * T + pb0] = x10;
                if (ra1v && cb1v) nxt[pa1 * T + pb1] = x11;
                // V <- V R' for pair bb on rows ba and ba + np (in place: each
                // (row, pair) belongs to exactly one block thread)
                if (mb == 2) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int vi = ba + u * np;
                        if (vi < T) {
                            const double vp = V[vi * T + pb0], vq = V[vi * T + pb1];
                            V[vi * T + pb0] = sub_rn(mul_rn(cb, vp), mul_rn(sb, vq));
                            V[vi * T + pb1] = add_rn(mul_rn(sb, vp), mul_rn(cb, vq));
                        }
                    }
                }
            }
            cta_sync();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        converged = offdiag() <= rtol * frob;
    }
    if (cur != A)
        for (int e = tid; e < T * T; e += blockDim.x) A[e] = cur[e];
    if (tid == 0) s_result2 = converged ? 0 : max_sweeps;
    cta_sync();
    return s_result2;
}

__device__ int cta_jacobi(double* A, double* V, int T, int max_sweeps, double rtol, double* red,
                          double* s_c, double* s_s, int* s_mode) {
    const int tid = threadIdx.x;
    __shared__ int s_result;
    for (int e = tid; e < T * T; e += blockDim.x) V[e] = (e / T == e % T) ? 1.0 : 0.0;
    // frob = sqrt(sum a^2) of the input
    double f2 = 0.0;
    for (int e = tid; e < T * T; e += blockDim.x) f2 = fma(A[e], A[e], f2);
    const double frob = sqrt(block_sum(f2, red));
    if (frob == 0.0) return 0;   // zeros and identity (linalg.py:153-154)
    if (tid < JAC_NT) {
        const int Te = T + (T & 1);
        const int np = Te / 2;
        // per-round pair table: (p, q, mode) and (c, s), one 16-byte record each
        __shared__ int4 s_pi[DCG_MAX_T / 2 + 1];
        __shared__ double2 s_cs[DCG_MAX_T / 2 + 1];
        // fixed work assignment for the whole solve: block (ba, bb) of the
        // np x np grid of 2 x 2 blocks, and V entries (row vi, pair vb)
        const int nblk = np * np;
        auto offdiag = [&]() {
            double o2 = 0.0;
            for (int e = tid; e < T * T; e += JAC_NT) {
                const int i = e / T, j = e - (e / T) * T;
                if (i != j) o2 = fma(A[e], A[e], o2);
            }
            return sqrt(block_sum(o2, red));
        };
        bool converged = offdiag() <= rtol * frob;
        for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
            for (int round = 0; round < Te - 1; ++round) {
                if (tid < np) {
                    // circle method: position 0 holds player Te-1, the others rotate
                    const int pos_b = Te - 1 - tid;
                    int pa = tid == 0 ? Te - 1 : tid - 1 + round;
                    if (tid != 0 && pa >= Te - 1) pa -= Te - 1;
                    int pb = pos_b - 1 + round;
                    if (pb >= Te - 1) pb -= Te - 1;
                    const int p = min(pa, pb), q = max(pa, pb);
                    double c = 1.0, sn = 0.0;
                    int mode = 0;   // 0 identity, 1 zero a_pq, 2 rotate
                    if (q < T) {
                        const double apq = A[p * T + q];
                        const double app = A[p * T + p], aqq = A[q * T + q];
                        const double g = 100.0 * fabs(apq);
                        if (add_rn(fabs(app), g) == fabs(app) && add_rn(fabs(aqq), g) == fabs(aqq)) {
                            mode = 1;
                        } else if (apq != 0.0) {
                            const double tau = (aqq - app) * fast_rcp(2.0 * apq);
                            const double at = fabs(tau);
                            double t;
                            if (at < 1e100) {
                                const double w = fma(tau, tau, 1.0);
                                t = fast_rcp(at + w * fast_rsqrt(w));
                            } else {
                                t = 0.5 * fast_rcp(at);
                            }
                            if (tau < 0.0) t = -t;
                            c = fast_rsqrt(fma(t, t, 1.0));
                            sn = t * c;
                            mode = 2;
                        }
                    }
                    s_pi[tid] = make_int4(p, q, mode, 0);
                    s_cs[tid] = make_double2(c, sn);
                }
                jac_sync();
                // A <- R A R' on the 2 x 2 block (row pair ba, column pair bb)
                for (int blk = tid; blk < nblk; blk += JAC_NT) {
                    const int ba = blk / np, bb = blk - (blk / np) * np;
                    const int4 ia = s_pi[ba], ib = s_pi[bb];
                    const double2 ra = s_cs[ba], rb = s_cs[bb];
                    const bool ra1v = ia.y < T, cb1v = ib.y < T;
                    double x00 = A[ia.x * T + ib.x];
                    double x01 = cb1v ? A[ia.x * T + ib.y] : 0.0;
                    double x10 = ra1v ? A[ia.y * T + ib.x] : 0.0;
                    double x11 = (ra1v && cb1v) ? A[ia.y * T + ib.y] : 0.0;
                    if (ib.z == 2) {   // columns: a'_ip = c a_ip - s a_iq ; a'_iq = s a_ip + c a_iq
                        const double y00 = sub_rn(mul_rn(rb.x, x00), mul_rn(rb.y, x01));
                        const double y01 = add_rn(mul_rn(rb.y, x00), mul_rn(rb.x, x01));
                        const double y10 = sub_rn(mul_rn(rb.x, x10), mul_rn(rb.y, x11));
                        const double y11 = add_rn(mul_rn(rb.y, x10), mul_rn(rb.x, x11));
                        x00 = y00; x01 = y01; x10 = y10; x11 = y11;
                    }
                    if (ia.z == 2) {   // rows
                        const double y00 = sub_rn(mul_rn(ra.x, x00), mul_rn(ra.y, x10));
                        const double y10 = add_rn(mul_rn(ra.y, x00), mul_rn(ra.x, x10));
                        const double y01 = sub_rn(mul_rn(ra.x, x01), mul_rn(ra.y, x11));
                        const double y11 = add_rn(mul_rn(ra.y, x01), mul_rn(ra.x, x11));
                        x00 = y00; x01 = y01; x10 = y10; x11 = y11;
                    }
                    if (ba == bb && ia.z != 0) { x01 = 0.0; x10 = 0.0; }
                    A[ia.x * T + ib.x] = x00;
                    if (cb1v) A[ia.x * T + ib.y] = x01;
                    if (ra1v) A[ia.y * T + ib.x] = x10;
                    if (ra1v && cb1v) A[ia.y * T + ib.y] = x11;
                }
                // V <- V R' (row vi, pair vb)
                for (int e = tid; e < T * np; e += JAC_NT) {
                    const int vi = e / np, vb = e - (e / np) * np;
                    const int4 ib = s_pi[vb];
                    if (ib.z != 2) continue;
                    const double2 rb = s_cs[vb];
                    const double vp = V[vi * T + ib.x], vq = V[vi * T + ib.y];
                    V[vi * T + ib.x] = sub_rn(mul_rn(rb.x, vp), mul_rn(rb.y, vq));
                    V[vi * T + ib.y] = add_rn(mul_rn(rb.y, vp), mul_rn(rb.x, vq));
                }
                jac_sync();
            }
            converged = offdiag() <= rtol * frob;
        }
        if (tid == 0) s_result = converged ? 0 : max_sweeps;
    }
    cta_sync();
    return s_result;
}

// order[r] = index of the r-th smallest value, ties by index (stable argsort)
__device__ void cta_stable_argsort(const double* vals, int stride, int n, int* order) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double vi = vals[i * stride];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double vj = vals[j * stride];
            if (vj < vi || (vj == vi && j < i)) ++rank;
        }
        order[rank] = i;
    }
    cta_sync();
}

// ===========================================================================
// Gram factorisation with optional failing-pivot pruning.
// Graw: k x k (W'AW, unsymmetrised).  Outputs L (kk x kk, leading dim kk),
// active column list, status.  solvers.py:107-115 (no prune -> GramNotSpd),
// recycle.py:66-77 (prune; empty -> BasisDeficient(0)).
// ===========================================================================
__global__ void __launch_bounds__(SD_NT) gram_factor_kernel(const double* Graw, int k, int prune,
                                                            double* Gsym, double* L, int* active,
                                                            DevStatus* st) {
    __shared__ double red[40];
    __shared__ double s_scal[4];
    __shared__ int s_act[DCG_MAX_K];
    __shared__ int s_na;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e % k;
        Gsym[e] = mul_rn(0.5, add_rn(Graw[i * k + j], Graw[j * k + i]));
    }
    if (threadIdx.x < k) s_act[threadIdx.x] = threadIdx.x;
    if (threadIdx.x == 0) s_na = k;
    cta_sync();
    // compact sub-matrix lives in L's own storage region "sub" right after L (kk*kk)
    double* sub = L + k * k;
    while (true) {
        const int na = s_na;
        if (na == 0) {
            if (threadIdx.x == 0) { st->status = DCG_E_BASIS_DEFICIENT; st->info = 0; st->count = 0; }
            return;
        }
        for (int e = threadIdx.x; e < na * na; e += blockDim.x) {
            const int i = e / na, j = e % na;
            sub[e] = Gsym[s_act[i] * k + s_act[j]];
        }
        cta_sync();
        const double tol = cta_pivot_tol(sub, na, nullptr, na, red);
        const int fail = cta_cholesky(sub, na, na, tol, L, na, s_scal);
        if (fail < 0) {
            if (threadIdx.x == 0) { st->status = DCG_OK; st->info = 0; st->count = na; }
            if (threadIdx.x < na) active[threadIdx.x] = s_act[threadIdx.x];
            return;
        }
        if (!prune) {
            if (threadIdx.x == 0) { st->status = DCG_E_GRAM_NOT_SPD; st->info = fail; st->count = na; }
            return;
        }
        cta_sync();
        if (threadIdx.x == 0) {
            for (int i = fail; i < na - 1; ++i) s_act[i] = s_act[i + 1];
            s_na = na - 1;
        }
        cta_sync();
    }
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi for C = L^-1 G L^-T without forming C.
// With G = R R' (lower R) and X = (L^-1 R)', X'X = C; rotating pairs of X's
// columns with the rotation two-sided Jacobi would apply to C (computed from
// the pair's 2 x 2 Gram [x_p'x_p x_p'x_q; x_p'x_q x_q'x_q], same skip rule,
// same formulas) orthogonalises the columns: theta_c = ||x_c||^2, V holds the
// accumulated rotations.  A pair belongs to one warp (lanes own rows lane and
// lane + 32): the rotation never leaves the warp, so a round is one CTA
// barrier.  Convergence: off(X'X) <= rtol ||C||_F before every sweep
// (linalg.py:156-163).  X: column c at X + c * n (T <= 64); Vc column-major.
// ---------------------------------------------------------------------------
// developer diagnostics of the Ritz pencil (dcg_debug_pencil_profile):
// globaltimer stamps of its phases and the one-sided Jacobi sweep count
__device__ unsigned long long g_pencil_prof[16];
// the pencil's tridiagonal fast path (1) or always the cyclic Jacobi (0)
__device__ int g_pencil_fast = 1;
__device__ __forceinline__ void pencil_stamp(int i) {
    if (threadIdx.x == 0) g_pencil_prof[i] = globaltimer_ns();
}

__device__ __forceinline__ int cta_jacobi_onesided(double* X, double* Vc, int n, int max_sweeps, double rtol,
                                                   double* red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ int s_res1;
    for (int e = tid; e < n * n; e += blockDim.x) Vc[e] = (e / n == e - (e / n) * n) ? 1.0 : 0.0;
    const int i0 = lane, i1 = lane + 32;
    auto gram = [&](double* frob2) {
        // off^2 = sum_{p != q} (x_p'x_q)^2 ; frob^2 = sum_{p,q} (x_p'x_q)^2.
        // Warp per p, lanes over q >= p, each dot sequential over the rows.
        double off2 = 0.0, all2 = 0.0;
        for (int p = warp; p < n; p += nw) {
            const double* xp = X + p * n;
            for (int q = p + lane; q < n; q += 32) {
                const double* xq = X + q * n;
                double d = 0.0;
                for (int i = 0; i < n; ++i) d = fma(xp[i], xq[i], d);
                if (q == p) {
                    all2 = fma(d, d, all2);
                } else {
                    off2 = fma(2.0 * d, d, off2);
                    all2 = fma(2.0 * d, d, all2);
                }
            }
        }
        off2 = block_sum(off2, red);
        all2 = block_sum(all2, red);
        if (frob2) *frob2 = all2;
        return sqrt(off2);
    };
    double frob2 = 0.0;
    double off = gram(&frob2);
    const double frob = sqrt(frob2);
    if (frob == 0.0) return 0;
    bool converged = off <= rtol * frob;
    const int Te = n + (n & 1), np = Te / 2;
    int sweeps_done = 0;
    for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
        ++sweeps_done;
        for (int round = 0; round < Te - 1; ++round) {
            // each pair's warp forms the pair's 2 x 2 Gram, computes the
            // rotation (redundantly on its lanes: no broadcast) and rotates
            for (int slot = warp; slot < np; slot += nw) {
                int pa = slot == 0 ? Te - 1 : slot - 1 + round;
                if (slot != 0 && pa >= Te - 1) pa -= Te - 1;
                int pb = Te - 2 - slot + round;
                if (pb >= Te - 1) pb -= Te - 1;
                const int p = min(pa, pb), q = max(pa, pb);
                if (q >= n) continue;
                const double xp0 = i0 < n ? X[p * n + i0] : 0.0, xp1 = i1 < n ? X[p * n + i1] : 0.0;
                const double xq0 = i0 < n ? X[q * n + i0] : 0.0, xq1 = i1 < n ? X[q * n + i1] : 0.0;
                // V rows loaded with X's, ahead of the rotation chain
                const double vp0 = i0 < n ? Vc[p * n + i0] : 0.0, vq0 = i0 < n ? Vc[q * n + i0] : 0.0;
                const double vp1 = i1 < n ? Vc[p * n + i1] : 0.0, vq1 = i1 < n ? Vc[q * n + i1] : 0.0;
                double app = fma(xp1, xp1, xp0 * xp0);
                double aqq = fma(xq1, xq1, xq0 * xq0);
                double apq = fma(xp1, xq1, xp0 * xq0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    app += __shfl_xor_sync(0xffffffffu, app, o);
                    aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
                    apq += __shfl_xor_sync(0xffffffffu, apq, o);
                }
                const double g = 100.0 * fabs(apq);
                if (add_rn(fabs(app), g) == fabs(app) && add_rn(fabs(aqq), g) == fabs(aqq)) continue;
                if (apq == 0.0) continue;
                const double tau = (aqq - app) * fast_rcp(2.0 * apq);
                const double at = fabs(tau);
                double t;
                if (at < 1e100) {
                    const double w = fma(tau, tau, 1.0);
                    t = fast_rcp(at + w * fast_rsqrt(w));
                } else {
                    t = 0.5 * fast_rcp(at);
                }
                if (tau < 0.0) t = -t;
                const double c = fast_rsqrt(fma(t, t, 1.0));
                const double sn = t * c;
                if (i0 < n) {
                    X[p * n + i0] = sub_rn(mul_rn(c, xp0), mul_rn(sn, xq0));
                    X[q * n + i0] = add_rn(mul_rn(sn, xp0), mul_rn(c, xq0));
                    Vc[p * n + i0] = sub_rn(mul_rn(c, vp0), mul_rn(sn, vq0));
                    Vc[q * n + i0] = add_rn(mul_rn(sn, vp0), mul_rn(c, vq0));
                }
                if (i1 < n) {
                    X[p * n + i1] = sub_rn(mul_rn(c, xp1), mul_rn(sn, xq1));
                    X[q * n + i1] = add_rn(mul_rn(sn, xp1), mul_rn(c, xq1));
                    Vc[p * n + i1] = sub_rn(mul_rn(c, vp1), mul_rn(sn, vq1));
                    Vc[q * n + i1] = add_rn(mul_rn(sn, vp1), mul_rn(c, vq1));
                }
            }
            cta_sync();
        }
        off = gram(nullptr);
        converged = off <= rtol * frob;
    }
    if (tid == 0) s_res1 = converged ? 0 : max_sweeps;
    if (tid == 0) g_pencil_prof[7] = sweeps_done;
    cta_sync();
    return s_res1;
}

// ===========================================================================
// Fast path of the pencil's symmetric eigenproblem: C (n x n, n <= 64, shared,
// row-major, destroyed) -> the k eigenpairs selected (the k largest or
// smallest), eigenvalues ascending.  Householder tridiagonalisation (n - 2
// reflector steps, two CTA phases each), multisection of the tridiagonal's
// Sturm counts for the selected eigenvalues (a warp per eigenvalue, 32
// shifts per round), a twisted factorisation per eigenvalue for its vector
// (Parlett-Dhillon: forward and backward pivots, the twist at min |gamma|),
// back-transformation by the stored reflectors.  Replaces the cyclic Jacobi's
// ~210 dependent rotation rounds at n = 36.
// Returns 0 -- and the caller runs Jacobi -- when two selected eigenvalues,
// or the boundary pair, are closer than 1e-7 ||C|| (twisted vectors of a
// cluster would need reorthogonalisation) or a vector is not finite.  Writes
// V[:, j] (row-major n x n storage, column j) and lam[j], j < k.  All CTA
// threads call; smem scratch `ws` >= 6 n + 64 doubles.
// ===========================================================================
// 1 / q to ~1 ulp: the MUFU estimate and two Newton steps (Sturm pivots
// tolerate a relative perturbation of a few ulps; div_rn's latency does not)
__device__ __forceinline__ double rcp_nr(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ int pencil_tridiag_fast(double* C, int n, int k, int largest, double* V, int ldv, double* lam, double* ws) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ double s_sc[4];
    __shared__ int s_ok;
    double* d = ws;            // n
    double* e = d + n;         // n (e[i] couples i, i+1)
    double* tau = e + n;       // n
    double* e2 = tau + n;      // n: e2[i] = e[i-1]^2
    double* pb = e2 + n;       // n: p = t A22 v
    if (tid == 0) s_ok = 1;
    // ---- tridiagonalisation on the first TW threads (a named barrier: the
    // step is latency-bound, a 1024-thread barrier costs more than its work).
    // A[j+1:, j] -> alpha e_1; the reflector is kept in row j's upper part,
    // C[j, j+1:] (only its head differs from the row), contiguous for the
    // back-transformation.  Every warp
    // forms the reflector's scalars itself (a warp reduction over the column),
    // so a step is two phases: p = t A22 v (a thread per row, reading A22 by
    // columns -- it is symmetric -- so the lanes' loads are contiguous), then
    // the rank-2 update with w = p - (t/2)(p'v) v, formed symmetrically.
    constexpr int TW = 256;
    if (tid < TW) {
        for (int j = 0; j + 2 < n; ++j) {
            const int m = n - j - 1;
            // column j below the diagonal, read as row j right of it (the
            // updates keep C bitwise symmetric): contiguous, conflict-free
            const double* col = C + j * n + j + 1;     // col[i], i < m
            const double x0 = col[0];
            double ss = 0.0;
            for (int i = lane; i < m; i += 32) ss = fma(col[i], col[i], ss);
            ss = warp_sum(ss);
            const double nrm = sqrt(ss);
            const double alpha = x0 >= 0.0 ? -nrm : nrm;
            const double v0 = x0 - alpha;
            const double vtv = ss - x0 * x0 + v0 * v0;
            const double t = (nrm == 0.0 || vtv == 0.0) ? 0.0 : 2.0 / vtv;
            if (tid == 0) {
                tau[j] = t;
                e[j] = (t == 0.0) ? x0 : alpha;
                d[j] = C[j * n + j];
            }
            if (t != 0.0) {
                double* a22 = C + (j + 1) * n + (j + 1);
                // p: four threads per row (m <= 63 rows in one pass), columns
                // interleaved over the four, combined by two shuffles
                {
                    const int r = tid >> 2, h = tid & 3;
                    double s0 = 0.0, s1 = 0.0;
                    if (r < m) {
                        int c = h;
                        for (; c + 4 < m; c += 8) {
                            s0 = fma(a22[c * n + r], c == 0 ? v0 : col[c], s0);
                            s1 = fma(a22[(c + 4) * n + r], col[c + 4], s1);
                        }
                        if (c < m) s0 = fma(a22[c * n + r], c == 0 ? v0 : col[c], s0);
                    }
                    double sp = s0 + s1;
                    sp += __shfl_xor_sync(0xffffffffu, sp, 1);
                    sp += __shfl_xor_sync(0xffffffffu, sp, 2);
                    if (h == 0 && r < m) pb[r] = t * sp;
                }
                asm volatile("barrier.sync 1, 256;" ::: "memory");
                double pv = 0.0;
                for (int i = lane; i < m; i += 32) pv = fma(pb[i], i == 0 ? v0 : col[i], pv);
                const double K = 0.5 * t * warp_sum(pv);
                // rank-2 update: thread (tid >> 4, tid & 15) walks a 16-strided grid
                for (int r = tid >> 4; r < m; r += TW / 16) {
                    const double vr = r == 0 ? v0 : col[r];
                    const double wr = pb[r] - K * vr;
                    for (int c = tid & 15; c < m; c += 16) {
                        const double vc = c == 0 ? v0 : col[c];
                        const double wc = pb[c] - K * vc;
                        a22[r * n + c] = sub_rn(a22[r * n + c], add_rn(mul_rn(vr, wc), mul_rn(wr, vc)));
                    }
                }
            }
            asm volatile("barrier.sync 1, 256;" ::: "memory");
            // the reflector is row j's upper part with its head replaced
            if (tid == 0 && t != 0.0) C[j * n + j + 1] = v0;
        }
    }
    cta_sync();
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = C[(n - 2) * n + (n - 2)];
            e[n - 2] = C[(n - 1) * n + (n - 2)];
        }
        d[n - 1] = C[(n - 1) * n + (n - 1)];
        if (n == 1) e[0] = 0.0;
        e[n - 1] = 0.0;
        // Gershgorin interval and the norm scale
        double lo = 1e300, hi = -1e300, nrm = 0.0;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
            lo = fmin(lo, d[i] - r);
            hi = fmax(hi, d[i] + r);
            nrm = fmax(nrm, fabs(d[i]) + r);
            e2[i] = i > 0 ? e[i - 1] * e[i - 1] : 0.0;
        }
        s_sc[0] = lo;
        s_sc[1] = hi;
        s_sc[2] = nrm;
    }
    cta_sync();
    pencil_stamp(8);
    const double glo = s_sc[0], ghi = s_sc[1], tnrm = s_sc[2];
    const double pivmin = fmax(1e-200, 1e-30 * tnrm * tnrm);
    // Sturm count: #eigenvalues < sigma, as sign changes of the scaled
    // characteristic-polynomial sequence p_i = (d_i - sigma) p_{i-1} - e_{i-1}^2 p_{i-2}.
    // Its ratios are the LDL pivots q_i = p_i / p_{i-1} of the division form
    // with the same rounding per step (one fused product each), and the same
    // pivmin clamp (|q_i| < pivmin -> q_i = -pivmin); a step's latency is one
    // FMA instead of a division.  |p| is kept in [2^-200, 2^200].
    // The power-of-two rescaling is exact and the clamp is relative, so WHEN
    // it is applied changes no sign and no count (only the p values, by powers
    // of two): with the pivot floor at or above 2^-400 a step moves |p| by at
    // most 2^100 up or 2^-400 down (|p_i / p_i-1| <= 2 ||T|| + e^2 / pivmin,
    // >= pivmin), so checking every second step keeps every value normal; the
    // check then leaves the FP64 chain on every other step.
    const bool two_step = pivmin >= 0x1p-400 && tnrm <= 0x1p90;
    auto step = [&](int i, double sigma, double& p, double& pp, int& c) {
        double pn = fma(d[i] - sigma, p, -(e2[i] * pp));
        if (fabs(pn) < pivmin * fabs(p)) pn = -pivmin * p;
        c += (pn < 0.0) != (p < 0.0);
        pp = p;
        p = pn;
    };
    auto rescale = [&](double& p, double& pp) {
        const double ap = fabs(p);
        if (ap > 0x1p200) { p *= 0x1p-200; pp *= 0x1p-200; }
        else if (ap < 0x1p-200) { p *= 0x1p200; pp *= 0x1p200; }
    };
    auto count_below = [&](double sigma) {
        int c = 0;
        double pp = 1.0;
        double p = d[0] - sigma;
        if (fabs(p) < pivmin) p = -pivmin;
        c += p < 0.0;
        if (two_step) {
            int i = 1;
            for (; i + 1 < n; i += 2) {
                step(i, sigma, p, pp, c);
                step(i + 1, sigma, p, pp, c);
                rescale(p, pp);
            }
            if (i < n) step(i, sigma, p, pp, c);
        } else {
            for (int i = 1; i < n; ++i) {
                step(i, sigma, p, pp, c);
                rescale(p, pp);
            }
        }
        return c;
    };
    // ---- multisection: warp w finds eigenvalue idx (ascending) of the selection
    const int first = largest ? n - k : 0;
    double* lamall = pb;   // reuse: k + 1 entries (the selection and its boundary neighbour)
    const int nloc = k + ((largest ? first > 0 : first + k < n) ? 1 : 0);
    for (int w = warp; w < nloc; w += nw) {
        const int idx = (w < k) ? first + w : (largest ? first - 1 : first + k);
        double a = glo, b = ghi;
        for (int it = 0; it < 40; ++it) {
            const double width = b - a;
            if (!(width > 4e-16 * fmax(fabs(a), fabs(b)))) break;
            const double sig = a + width * (lane + 1) / 33.0;
            const long long c0 = clock64();
            const int cnt = count_below(sig);
            if (tid == 0) { g_pencil_prof[12] += clock64() - c0; g_pencil_prof[13] += 1; }
            // lanes whose shift is above the eigenvalue: cnt > idx
            const unsigned above = __ballot_sync(0xffffffffu, cnt > idx);
            const int lo_lane = above ? __ffs(above) - 2 : 31;   // last lane below (-1: a)
            const double na_ = lo_lane < 0 ? a : a + width * (lo_lane + 1) / 33.0;
            const double nb_ = above ? a + width * (lo_lane + 2) / 33.0 : b;
            a = na_;
            b = nb_;
        }
        if (lane == 0) lamall[w] = 0.5 * (a + b);
    }
    cta_sync();
    pencil_stamp(9);
    // cluster check on the selected eigenvalues and the boundary pair
    if (tid == 0) {
        double prev = 0.0;
        bool have = false;
        const double gap = 1e-7 * fmax(tnrm, 1e-300);
        double vals[DCG_MAX_T + 2];
        int nv = 0;
        if (nloc > k && largest) vals[nv++] = lamall[k];
        for (int j = 0; j < k; ++j) vals[nv++] = lamall[j];
        if (nloc > k && !largest) vals[nv++] = lamall[k];
        for (int j = 0; j < nv; ++j) {
            if (have && vals[j] - prev < gap) s_ok = 0;
            prev = vals[j];
            have = true;
        }
        for (int j = 0; j < k; ++j) lam[j] = lamall[j];
    }
    cta_sync();
    if (!s_ok) return 0;
    // ---- twisted factorisation, a warp per eigenvalue.  All lanes run the
    // pivot recurrences (uniform control flow); lane l keeps pivots l, l + 32:
    //   D+_i = (d_i - lam) - e_{i-1}^2 / D+_{i-1},  D-_i = (d_i - lam) - e_i^2 / D-_{i+1},
    //   gamma_i = D+_i + D-_i - (d_i - lam),  r = argmin |gamma_i|,
    //   z_r = 1, z_i = -e_i z_{i+1} / D+_i (i < r), z_i = -e_{i-1} z_{i-1} / D-_i (i > r).
    for (int w = warp; w < k; w += nw) {
        const double lm = lam[w];
        double dp0 = 0.0, dp1 = 0.0, dm0 = 0.0, dm1 = 0.0;
        double q = 1.0;
        for (int i = 0; i < n; ++i) {
            q = (i == 0) ? d[0] - lm : (d[i] - lm) - e2[i] * rcp_nr(q);
            if (fabs(q) < pivmin) q = q < 0.0 ? -pivmin : pivmin;
            if (i == lane) dp0 = q;
            if (i == lane + 32) dp1 = q;
        }
        for (int i = n - 1; i >= 0; --i) {
            q = (i == n - 1) ? d[i] - lm : (d[i] - lm) - e2[i + 1] * rcp_nr(q);
            if (fabs(q) < pivmin) q = q < 0.0 ? -pivmin : pivmin;
            if (i == lane) dm0 = q;
            if (i == lane + 32) dm1 = q;
        }
        // twist index: min |gamma|, ties to the lower index
        double g = 1e308;
        int gi = n;
        if (lane < n) { g = fabs(dp0 + dm0 - (d[lane] - lm)); gi = lane; }
        if (lane + 32 < n) {
            const double g1 = fabs(dp1 + dm1 - (d[lane + 32] - lm));
            if (g1 < g) { g = g1; gi = lane + 32; }
        }
        for (int o = 16; o; o >>= 1) {
            const double og = __shfl_xor_sync(0xffffffffu, g, o);
            const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
            if (og < g || (og == g && oi < gi)) { g = og; gi = oi; }
        }
        const int r = gi;
        // ratios into V's column w, then the products outward from the twist
        if (lane < n) V[lane * ldv + w] = lane < r ? -e[lane] / dp0 : (lane > r ? -e[lane - 1] / dm0 : 1.0);
        if (lane + 32 < n) {
            const int i = lane + 32;
            V[i * ldv + w] = i < r ? -e[i] / dp1 : (i > r ? -e[i - 1] / dm1 : 1.0);
        }
        __syncwarp();
        if (lane == 0) {
            double z = 1.0;
            for (int i = r - 1; i >= 0; --i) { z *= V[i * ldv + w]; V[i * ldv + w] = z; }
            z = 1.0;
            for (int i = r + 1; i < n; ++i) { z *= V[i * ldv + w]; V[i * ldv + w] = z; }
        }
        __syncwarp();
        double s2 = 0.0;
        for (int i = lane; i < n; i += 32) s2 = fma(V[i * ldv + w], V[i * ldv + w], s2);
        const double inv = 1.0 / sqrt(warp_sum(s2));
        if (!(inv > 0.0) || !isfinite(inv)) { if (lane == 0) s_ok = 0; }
        else for (int i = lane; i < n; i += 32) V[i * ldv + w] *= inv;
    }
    cta_sync();
    pencil_stamp(10);
    if (!s_ok) return 0;
    // ---- back-transformation: y <- H_0 ... H_{n-3} y (reflectors in reverse
    // order, read from the upper rows: contiguous); a warp per vector
    for (int w = warp; w < k; w += nw) {
        for (int j = n - 3; j >= 0; --j) {
            const double t = tau[j];
            if (t == 0.0) continue;
            const int m = n - j - 1;
            const double* v = C + j * n + j + 1;
            double* y = V + (j + 1) * ldv + w;
            double dot = 0.0;
            for (int i = lane; i < m; i += 32) dot = fma(v[i], y[i * ldv], dot);
            dot = t * warp_sum(dot);
            for (int i = lane; i < m; i += 32) y[i * ldv] -= dot * v[i];
            __syncwarp();
        }
    }
    cta_sync();
    pencil_stamp(11);
    if (tid == 0) g_pencil_prof[14] = 1;
    return 1;
}

// ===========================================================================
// Harmonic pencil: symmetrise F, G; prune F's failing-pivot columns; solve
// G u = theta F u (gen_sym_eigen, linalg.py:168-191); select k values.
// Global scratch `wk` holds 5 * T * T doubles.  Outputs: theta (k), U (na x k,
// row-major over the surviving columns), active list, status (count = na).
// ===========================================================================
// `plan` (when non-null) carries the pencil order T (= count) decided on the
// device by the extraction's zero-column scan, and its status: the kernel does
// nothing unless that status is DCG_OK, so the pipeline needs no host sync.
// STAGED (T <= DCG_PENCIL_SMEM_T, every pencil the solver forms): the working
// matrices' pointers derive from the shared array at compile time, so every
// access is a shared-memory instruction -- through a pointer that may be
// either, the compiler emits generic loads (longer latency on each link of
// the serial chains).
template <bool STAGED>
__device__ __forceinline__ void pencil_body(const double* Fraw, const double* Graw, int T, int k, int largest,
                                            int max_sweeps, double* wk, double* theta, double* U, int* active,
                                            DevStatus* st) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[40];
    __shared__ double s_scal[4];
    __shared__ double s_c[DCG_MAX_T / 2 + 1], s_s[DCG_MAX_T / 2 + 1];
    __shared__ int s_mode[DCG_MAX_T / 2 + 1 + DCG_MAX_T + 2];
    __shared__ int s_act[DCG_MAX_T];
    __shared__ int s_order[DCG_MAX_T];
    __shared__ int s_na;
    pencil_stamp(0);
    if (threadIdx.x == 0)
        for (int i = 7; i < 15; ++i) g_pencil_prof[i] = 0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nw = blockDim.x >> 5;
    // F, G (symmetrised, T x T) stay in the global scratch: they are only read
    // by parallel compaction loops.  The matrices the serial chains walk
    // (Cholesky, triangular solves, Jacobi) live in shared memory when they fit:
    // slots S0 = Fa then V, S1 = L, S2 = Ga then Y (in place), S3 = A.
    double* F = wk;
    double* G = F + T * T;
    constexpr bool staged = STAGED;
    double* L;
    double* Y;
    double* Fa;
    if constexpr (STAGED) {
        L = sm + T * T;
        Y = sm + 2 * T * T;
        Fa = sm;
    } else {
        L = G + T * T;
        Y = L + T * T;
        Fa = Y + T * T;
    }
    for (int e = tid; e < T * T; e += blockDim.x) {
        const int i = e / T, j = e % T;
        F[e] = mul_rn(0.5, add_rn(Fraw[i * T + j], Fraw[j * T + i]));
        G[e] = mul_rn(0.5, add_rn(Graw[i * T + j], Graw[j * T + i]));
    }
    if (tid < T) s_act[tid] = tid;
    if (tid == 0) s_na = T;
    cta_sync();
    int na;
    while (true) {
        na = s_na;
        if (na < k) {
            if (tid == 0) { st->status = DCG_E_BASIS_DEFICIENT; st->info = na; st->count = na; }
            return;
        }
        for (int e = tid; e < na * na; e += blockDim.x) {
            const int i = e / na, j = e % na;
            Fa[e] = F[s_act[i] * T + s_act[j]];
        }
        cta_sync();
        const double tol = cta_pivot_tol(Fa, na, nullptr, na, red);
        const int fail = cta_cholesky(Fa, na, na, tol, L, na, s_scal);
        if (fail < 0) break;
        cta_sync();
        if (tid == 0) {
            for (int i = fail; i < na - 1; ++i) s_act[i] = s_act[i + 1];
            s_na = na - 1;
        }
        cta_sync();
    }
    pencil_stamp(1);
    double* A;
    double* V;
    if constexpr (STAGED) {
        A = sm + 3 * T * T;
        V = sm;
    } else {
        A = sm;
        V = sm + T * T;
    }
    const int off = largest ? (na - k) : 0;
    // ---- fast path: C = L^-1 G L^-T, tridiagonal eigensolver for the k
    // selected pairs (pencil_tridiag_fast); Jacobi below when it declines
    bool fast = false;
    int ldv = na;
    if (staged && na >= 12 && na <= 64 && g_pencil_fast) {   // na >= 12: T*T >= 6 na + 64 scratch in S2
        __shared__ double s_lam[DCG_MAX_T];
        for (int e = tid; e < na * na; e += blockDim.x) {
            const int i = e / na, j = e % na;
            Fa[e] = G[s_act[i] * T + s_act[j]];
        }
        cta_sync();
        cta_solve_lower_cols(L, na, Fa, na, 1, Y, na, 1);
        cta_sync();
        cta_solve_lower_cols(L, na, Y, 1, na, A, na, 1);
        cta_sync();
        for (int e = tid; e < na * na; e += blockDim.x) {
            const int i = e / na, j = e % na;
            if (i < j) {
                const double v = mul_rn(0.5, add_rn(A[i * na + j], A[j * na + i]));
                A[i * na + j] = v;
                A[j * na + i] = v;
            }
        }
        cta_sync();
        pencil_stamp(2);
        // V's row stride padded to na + 1 when it fits: the column walks of
        // the twisted factorisation and the back-transformation then spread
        // over the banks
        ldv = (na + 1) * na <= T * T ? na + 1 : na;
        fast = pencil_tridiag_fast(A, na, k, largest, V, ldv, s_lam, Y) != 0;
        pencil_stamp(3);
        if (fast) {
            for (int j = tid; j < k; j += blockDim.x) {
                A[j * na + j] = s_lam[j];
                s_order[off + j] = j;
            }
            cta_sync();
        } else {
            ldv = na;
        }
    }
    bool onesided = false;
    int nc = 0;
    if (!fast) {
    if (staged && na <= 64) {
        // G (compact) -> S0, R = chol(G) -> S2, X = (L^-1 R)' in place in S2
        for (int e = tid; e < na * na; e += blockDim.x) {
            const int i = e / na, j = e % na;
            Fa[e] = G[s_act[i] * T + s_act[j]];
        }
        cta_sync();
        if (cta_cholesky(Fa, na, na, 0.0, Y, na, s_scal) < 0) {
            onesided = true;
            // B = L^-1 R, right-looking over rows (lower triangular B, row-major = X column-major)
            for (int j = 0; j < na; ++j) {
                for (int c = tid; c <= j; c += blockDim.x) Y[j * na + c] = div_rn(Y[j * na + c], L[j * na + j]);
                cta_sync();
                for (int i = j + 1 + warp; i < na; i += nw) {
                    const double lij = L[i * na + j];
                    for (int c = lane; c <= j; c += 32) Y[i * na + c] = sub_rn(Y[i * na + c], mul_rn(lij, Y[j * na + c]));
                }
                cta_sync();
            }
        }
        cta_sync();
    }
    if (onesided) {
        // Vc (column-major) in S3; afterwards theta on the diagonal of A := S2 and V row-major in S0
        double* Vc = A;
        pencil_stamp(2);
        // staged: X is S2 and Vc is S3 -- pointers formed from `sm` here so the
        // (inlined) rounds use shared-memory instructions, not generic ones
        nc = cta_jacobi_onesided(sm + 2 * T * T, sm + 3 * T * T, na, max_sweeps, 1e-14, red);
        pencil_stamp(3);
        if (nc == 0) {
            for (int c = warp; c < na; c += nw) {
                const double x0 = lane < na ? Y[c * na + lane] : 0.0, x1 = lane + 32 < na ? Y[c * na + lane + 32] : 0.0;
                const double th = warp_sum(fma(x1, x1, x0 * x0));
                __syncwarp();
                if (lane == 0) Y[c * na + c] = th;
            }
            for (int e = tid; e < na * na; e += blockDim.x) {
                const int i = e / na, c = e % na;
                V[i * na + c] = Vc[c * na + i];
            }
            cta_sync();
            A = Y;
        }
    } else {
    // compact Ga (solved in place into Y below)
    double* Ga = staged ? Y : Fa;
    for (int e = tid; e < na * na; e += blockDim.x) {
        const int i = e / na, j = e % na;
        Ga[e] = G[s_act[i] * T + s_act[j]];
    }
    cta_sync();
    // Y = L^-1 Ga  (solve_lower_matrix: column by column)
    for (int c = warp; c < na; c += nw) warp_solve_lower(L, na, na, Ga + c, na, Y + c, na);
    cta_sync();
    // C = L^-1 Y'  -> into shared A
    for (int c = warp; c < na; c += nw) warp_solve_lower(L, na, na, Y + c * na, 1, A + c, na);
    cta_sync();
    // symmetrise
    for (int e = tid; e < na * na; e += blockDim.x) {
        const int i = e / na, j = e % na;
        if (i < j) {
            const double v = mul_rn(0.5, add_rn(A[i * na + j], A[j * na + i]));
            A[i * na + j] = v;
            A[j * na + i] = v;
        }
    }
    cta_sync();
    // staged: the Ga / Y slot (S2) is free again and double-buffers the Jacobi
    nc = staged ? cta_jacobi2(A, Y, V, na, max_sweeps, 1e-14, red)
                : cta_jacobi(A, V, na, max_sweeps, 1e-14, red, s_c, s_s, s_mode);
    }
    }   // !fast
    if (nc) {
        if (tid == 0) { st->status = DCG_E_NO_CONVERGENCE; st->info = nc; st->count = na; }
        return;
    }
    if (!fast) cta_stable_argsort(A, na + 1, na, s_order);
    // selected eigen-pairs: u = L^-T w, normalised
    for (int j = warp; j < k; j += nw) {
        const int col = s_order[off + j];
        warp_solve_lower_trans(L, na, na, V + col, ldv, U + j, k);
        __syncwarp();
        double s2 = 0.0;
        for (int i = lane; i < na; i += 32) s2 = fma(U[i * k + j], U[i * k + j], s2);
        const double nrm = sqrt(warp_sum(s2));
        if (nrm > 0.0)
            for (int i = lane; i < na; i += 32) U[i * k + j] = div_rn(U[i * k + j], nrm);
        if (lane == 0) theta[j] = A[col * na + col];
    }
    if (tid < na) active[tid] = s_act[tid];
    if (tid == 0) { st->status = DCG_OK; st->info = 0; st->count = na; }
    pencil_stamp(4);
    if (tid == 0) g_pencil_prof[6] = na;
}

__global__ void __launch_bounds__(PENCIL_NT) ritz_pencil_kernel(const double* Fraw, const double* Graw, int T,
                                                            int k, int largest, int max_sweeps,
                                                            double* wk, double* theta, double* U,
                                                            int* active, DevStatus* st, const DevStatus* plan) {
    // `plan` (when non-null) carries the pencil order decided on the device
    if (plan) {
        if (plan->status != DCG_OK) return;
        T = (int)plan->count;
    }
    if (T <= DCG_PENCIL_SMEM_T) pencil_body<true>(Fraw, Graw, T, k, largest, max_sweeps, wk, theta, U, active, st);
    else pencil_body<false>(Fraw, Graw, T, k, largest, max_sweeps, wk, theta, U, active, st);
}

extern "C" __attribute__((visibility("default"))) int dcg_debug_set_pencil_fast(int on) {
    const int v = on ? 1 : 0;
    if (cudaMemcpyToSymbol(g_pencil_fast, &v, sizeof(int)) != cudaSuccess) return DCG_E_CUDA;
    return DCG_OK;
}

int dcg_ritz_pencil_launch(cudaStream_t st, const double* Fraw, const double* Graw, int T, int k, int largest,
                           int max_sweeps, double* wk, double* theta, double* U, int* active, DevStatus* ds,
                           const DevStatus* plan);
// developer entry (tools/pencil_bench.py): the Ritz pencil alone on device
// inputs -- Fraw, Graw (T x T), wk (5 T^2), theta (k), U (T x k), active (T),
// status (one DevStatus) -- enqueued on `stream`
extern "C" __attribute__((visibility("default"))) int dcg_debug_ritz_pencil(void* stream, const double* Fraw,
                                                                          const double* Graw, int T, int k,
                                                                          int largest, double* wk, double* theta,
                                                                          double* U, int* active, void* status) {
    if (T < 1 || T > DCG_MAX_T || k < 1 || k > T) return DCG_E_CONFIG;
    return dcg_ritz_pencil_launch(static_cast<cudaStream_t>(stream), Fraw, Graw, T, k, largest, 60, wk, theta, U,
                                  active, static_cast<DevStatus*>(status), nullptr);
}

extern "C" __attribute__((visibility("default"))) int dcg_debug_pencil_profile(long long* out8) {
    unsigned long long h[16];
    if (cudaMemcpyFromSymbol(h, g_pencil_prof, sizeof(h)) != cudaSuccess) return DCG_E_CUDA;
    for (int i = 0; i < 16; ++i) out8[i] = (long long)h[i];
    return DCG_OK;
}

// ===========================================================================
// Standalone eigensolvers (dcg_sym_eigen / dcg_gen_sym_eigen).
// ===========================================================================
__global__ void __launch_bounds__(SD_NT) sym_eigen_kernel(const double* Ain, int n, int max_sweeps, double rtol,
                                                          double* values, double* vectors, DevStatus* st) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[40];
    __shared__ double s_c[DCG_MAX_T / 2 + 1], s_s[DCG_MAX_T / 2 + 1];
    __shared__ int s_mode[DCG_MAX_T / 2 + 1 + DCG_MAX_T + 2];
    __shared__ int s_order[DCG_MAX_T];
    double* A = sm;
    double* V = sm + n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[e] = Ain[e];
    cta_sync();
    const int nc = cta_jacobi(A, V, n, max_sweeps, rtol, red, s_c, s_s, s_mode);
    if (nc) {
        if (threadIdx.x == 0) { st->status = DCG_E_NO_CONVERGENCE; st->info = nc; }
        return;
    }
    cta_sync();
    cta_stable_argsort(A, n + 1, n, s_order);
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, r = e % n;
        vectors[i * n + r] = V[i * n + s_order[r]];
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) values[r] = A[s_order[r] * (n + 1)];
    if (threadIdx.x == 0) st->status = DCG_OK;
}

__global__ void __launch_bounds__(SD_NT) gen_sym_eigen_kernel(const double* g, const double* f, int n,
                                                              int max_sweeps, double* wk, double* values,
                                                              double* vectors, DevStatus* st) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[40];
    __shared__ double s_scal[4];
    __shared__ double s_c[DCG_MAX_T / 2 + 1], s_s[DCG_MAX_T / 2 + 1];
    __shared__ int s_mode[DCG_MAX_T / 2 + 1 + DCG_MAX_T + 2];
    __shared__ int s_order[DCG_MAX_T];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    double* L = wk;
    double* Y = wk + n * n;
    const double tol = cta_pivot_tol(f, n, nullptr, n, red);
    const int fail = cta_cholesky(f, n, n, tol, L, n, s_scal);
    if (fail >= 0) {
        if (tid == 0) { st->status = DCG_E_NOT_PD; st->info = fail; }
        return;
    }
    for (int c = warp; c < n; c += nw) warp_solve_lower(L, n, n, g + c, n, Y + c, n);
    cta_sync();
    double* A = sm;
    double* V = sm + n * n;
    for (int c = warp; c < n; c += nw) warp_solve_lower(L, n, n, Y + c * n, 1, A + c, n);
    cta_sync();
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e % n;
        if (i < j) {
            const double v = mul_rn(0.5, add_rn(A[i * n + j], A[j * n + i]));
            A[i * n + j] = v;
            A[j * n + i] = v;
        }
    }
    cta_sync();
    const int nc = cta_jacobi(A, V, n, max_sweeps, 1e-14, red, s_c, s_s, s_mode);
    if (nc) {
        if (tid == 0) { st->status = DCG_E_NO_CONVERGENCE; st->info = nc; }
        return;
    }
    cta_stable_argsort(A, n + 1, n, s_order);
    for (int j = warp; j < n; j += nw) {
        const int col = s_order[j];
        warp_solve_lower_trans(L, n, n, V + col, n, vectors + j, n);
        __syncwarp();
        double s2 = 0.0;
        for (int i = lane; i < n; i += 32) s2 = fma(vectors[i * n + j], vectors[i * n + j], s2);
        const double nrm = sqrt(warp_sum(s2));
        if (nrm > 0.0)
            for (int i = lane; i < n; i += 32) vectors[i * n + j] = div_rn(vectors[i * n + j], nrm);
        if (lane == 0) values[j] = A[col * (n + 1)];
    }
    if (tid == 0) st->status = DCG_OK;
}

// ===========================================================================
// L0 twins with the reference's exact operation order.
// ===========================================================================
__global__ void __launch_bounds__(SD_NT) k_cholesky_kernel(const double* a, int n, double tol, double* l,
                                                           DevStatus* st) {
    __shared__ double s_scal[4];
    const int fail = cta_cholesky(a, n, n, tol, l, n, s_scal);
    if (threadIdx.x == 0) st->info = fail;
}

__global__ void k_solve_lower_kernel(const double* l, int n, const double* b, double* y) {
    // single thread: exact reference order (_core.pyx:69-80)
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < n; ++i) {
        double acc = b[i];
        for (int j = 0; j < i; ++j) acc = sub_rn(acc, mul_rn(l[(long long)i * n + j], y[j]));
        y[i] = div_rn(acc, l[(long long)i * n + i]);
    }
}

__global__ void k_solve_lower_trans_kernel(const double* l, int n, const double* b, double* x) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = n - 1; i >= 0; --i) {
        double acc = b[i];
        for (int j = i + 1; j < n; ++j) acc = sub_rn(acc, mul_rn(l[(long long)j * n + i], x[j]));
        x[i] = div_rn(acc, l[(long long)i * n + i]);
    }
}

// One cyclic Jacobi sweep in the reference's exact order (_core.pyx:135-177);
// the three inner loops run in parallel over i.
__global__ void __launch_bounds__(SD_NT) k_jacobi_sweep_kernel(double* a, double* v, int n, DevStatus* st) {
    __shared__ double s_cs[2];
    __shared__ int s_mode;
    long long rotations = 0;
    for (int p = 0; p < n - 1; ++p) {
        for (int q = p + 1; q < n; ++q) {
            if (threadIdx.x == 0) {
                const double apq = a[p * n + q];
                const double g = 100.0 * fabs(apq);
                const double app = a[p * n + p], aqq = a[q * n + q];
                if (add_rn(fabs(app), g) == fabs(app) && add_rn(fabs(aqq), g) == fabs(aqq)) {
                    a[p * n + q] = 0.0;
                    a[q * n + p] = 0.0;
                    s_mode = 0;
                } else if (apq == 0.0) {
                    s_mode = 0;
                } else {
                    const double tau = div_rn(sub_rn(aqq, app), mul_rn(2.0, apq));
                    double t;
                    if (tau >= 0.0) t = div_rn(1.0, add_rn(tau, sqrt(add_rn(1.0, mul_rn(tau, tau)))));
                    else t = div_rn(-1.0, add_rn(-tau, sqrt(add_rn(1.0, mul_rn(tau, tau)))));
                    const double c = div_rn(1.0, sqrt(add_rn(1.0, mul_rn(t, t))));
                    s_cs[0] = c;
                    s_cs[1] = mul_rn(t, c);
                    s_mode = 1;
                }
            }
            cta_sync();
            if (s_mode) {
                const double c = s_cs[0], s = s_cs[1];
                for (int i = threadIdx.x; i < n; i += blockDim.x) {
                    const double aip = a[i * n + p], aiq = a[i * n + q];
                    a[i * n + p] = sub_rn(mul_rn(c, aip), mul_rn(s, aiq));
                    a[i * n + q] = add_rn(mul_rn(s, aip), mul_rn(c, aiq));
                }
                cta_sync();
                for (int i = threadIdx.x; i < n; i += blockDim.x) {
                    const double aip = a[p * n + i], aiq = a[q * n + i];
                    a[p * n + i] = sub_rn(mul_rn(c, aip), mul_rn(s, aiq));
                    a[q * n + i] = add_rn(mul_rn(s, aip), mul_rn(c, aiq));
                }
                cta_sync();
                if (threadIdx.x == 0) {
                    a[p * n + q] = 0.0;
                    a[q * n + p] = 0.0;
                }
                for (int i = threadIdx.x; i < n; i += blockDim.x) {
                    const double vp = v[i * n + p], vq = v[i * n + q];
                    v[i * n + p] = sub_rn(mul_rn(c, vp), mul_rn(s, vq));
                    v[i * n + q] = add_rn(mul_rn(s, vp), mul_rn(c, vq));
                }
                ++rotations;
            }
            cta_sync();
        }
    }
    if (threadIdx.x == 0) st->count = rotations;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int dcg_gram_factor_launch(cudaStream_t st, const double* Graw, int k, int prune, double* Gsym, double* L,
                           int* active, DevStatus* ds) {
    gram_factor_kernel<<<1, SD_NT, 0, st>>>(Graw, k, prune, Gsym, L, active, ds);
    DCG_LAUNCHED();
    return DCG_OK;
}

size_t dcg_pencil_smem(int T) { return sizeof(double) * 2 * (size_t)T * T; }
// for any pencil order up to T (the device-driven extraction knows only a bound)
static size_t pencil_smem(int T) {
    const size_t staged = 4 * (size_t)(T < DCG_PENCIL_SMEM_T ? T : DCG_PENCIL_SMEM_T) * (T < DCG_PENCIL_SMEM_T ? T : DCG_PENCIL_SMEM_T);
    const size_t plain = 2 * (size_t)T * T;
    return sizeof(double) * (staged > plain ? staged : plain);
}

int dcg_ritz_pencil_launch(cudaStream_t st, const double* Fraw, const double* Graw, int T, int k, int largest,
                           int max_sweeps, double* wk, double* theta, double* U, int* active, DevStatus* ds,
                           const DevStatus* plan) {
    const size_t smem = pencil_smem(T);
    DCG_SMEM_ATTR(ritz_pencil_kernel, smem);
    ritz_pencil_kernel<<<1, PENCIL_NT, smem, st>>>(Fraw, Graw, T, k, largest, max_sweeps, wk, theta, U, active, ds,
                                                plan);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_sym_eigen_launch(cudaStream_t st, const double* A, int n, int max_sweeps, double rtol, double* values,
                         double* vectors, DevStatus* ds) {
    const size_t smem = dcg_pencil_smem(n);
    DCG_CUDA(cudaFuncSetAttribute(sym_eigen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    sym_eigen_kernel<<<1, SD_NT, smem, st>>>(A, n, max_sweeps, rtol, values, vectors, ds);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_gen_sym_eigen_launch(cudaStream_t st, const double* g, const double* f, int n, int max_sweeps, double* wk,
                             double* values, double* vectors, DevStatus* ds) {
    const size_t smem = dcg_pencil_smem(n);
    DCG_CUDA(cudaFuncSetAttribute(gen_sym_eigen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gen_sym_eigen_kernel<<<1, SD_NT, smem, st>>>(g, f, n, max_sweeps, wk, values, vectors, ds);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_k_cholesky_launch(cudaStream_t st, const double* a, int n, double tol, double* l, DevStatus* ds) {
    k_cholesky_kernel<<<1, SD_NT, 0, st>>>(a, n, tol, l, ds);
    DCG_LAUNCHED();
    return DCG_OK;
}
int dcg_k_solve_lower_launch(cudaStream_t st, const double* l, int n, const double* b, double* y) {
    k_solve_lower_kernel<<<1, 32, 0, st>>>(l, n, b, y);
    DCG_LAUNCHED();
    return DCG_OK;
}
int dcg_k_solve_lower_trans_launch(cudaStream_t st, const double* l, int n, const double* b, double* x) {
    k_solve_lower_trans_kernel<<<1, 32, 0, st>>>(l, n, b, x);
    DCG_LAUNCHED();
    return DCG_OK;
}
int dcg_k_jacobi_sweep_launch(cudaStream_t st, double* a, double* v, int n, DevStatus* ds) {
    k_jacobi_sweep_kernel<<<1, SD_NT, 0, st>>>(a, v, n, ds);
    DCG_LAUNCHED();
    return DCG_OK;
}
