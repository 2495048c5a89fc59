// Matrix-free RBF operator, symmetric pass 1 on the FP64 tensor pipe
// (kernel K7 of SURVEY.md section 2; config 5).
//
//   K_ij = var exp(-|x_i - x_j|^2 / (2 l^2))  (i != j),   K_ii = var + jitter
//
// is regenerated tile by tile in every product.  Per element the exponent is
//   e_ij = b_i + b_j + x~_i . x~_j,   b_i = -|x_i|^2 / (2 l^2),   x~ = x sqrt(2 / (2 l^2))
// The signal variance is folded into the vector: K v' = E (var v') with
// E_ij = exp(e_ij) and E_ii = (var + jitter) / var.
// (the |x_i|^2 + |x_j|^2 - 2 x_i.x_j form; the cancellation error is ~eps |x|^2
// absolute in the exponent, ~1e-16 relative in K), so the d-term contraction is
// an (64 x d) x (d x 64) matrix product per tile: mma.sync.m8n8k4.f64 (DMMA),
// whose accumulators start at b_i + b_j.  DMMA and DFMA share the FP64 pipe
// (tools/fp64_peak.cu: 37 vs 34 TFLOP/s, a DMMA+DFMA mix takes the sum of the
// two times), so the contraction still costs d FMAs per element; what DMMA
// removes is the issue and operand-load overhead of the FMA form.
// The exponential is table-based: e = k ln2 / 2048 + r, |r| <= ln2 / 4096,
//   exp(e) = 2^(k >> 11) * T[k & 2047] * (1 + p(r)),   T[j] = 2^(j / 2048),
// with p the degree-3 Taylor polynomial of expm1 (truncation < 3.5e-17), k from
// the 1.5 * 2^52 rounding trick, r from one FMA: 7 FP64 instructions per
// element.  The clamp
// that keeps intermediates normal (e >= -700) is compiled only into the path
// taken when the data's largest norm allows an exponent below -690.  With the
// two accumulations (row sums and column sums) an element costs ~d + 10 FP64
// pipe operations, against ~130 issued instructions of the FMA-form kernel.
//
// Work decomposition: the lower-triangle 64 x 64 tile sequence of the stored
// strategy (symgemv.cuh) is split into ranges per *team* -- 8 warps (256
// threads) -- so a 512-thread CTA runs two independent teams with their own
// named barriers.  Warp w of a team owns the tile's columns 8w..8w+7 and all
// 64 rows: 8 DMMA accumulator tiles, 16 elements per lane.  Operands arrive
// by TMA-style bulk copies (cp.async.bulk + mbarrier complete_tx) from a
// fragment-major copy of x~ (rbf_prep_kernel), so a lane's A / B fragments of
// two k-steps are one conflict-free 16-byte shared load; the next J tile is
// in flight while the current one is computed.  Partials use exactly the
// stored strategy's layout (colpart per tile, rowpart per tile-row segment),
// so sym_pass2 reduces them (with the team range table).
#pragma once
#include "common.cuh"
#include "symgemv.cuh"

#ifndef RM_GB
#define RM_GB 4                  // accumulator blocks per DMMA / exponential group (of 8 per warp tile)
#endif
#define RM_TB 64                 // tile side
#define RM_TW 8                  // warps per team
#define RM_TT (RM_TW * 32)       // threads per team
#define RM_MAX_TEAMS (DCG_NT / RM_TT)

// fragment-major operand layout (per 64-row tile, dp = dim padded to 8):
// element (row 8 rb + r, coordinate 8 ch + 4 e + q) at ((rb * nch + ch) * 32 + 4 r + q) * 2 + e
__host__ __device__ __forceinline__ int rm_dpad(int dim) { return (dim + 7) & ~7; }
__host__ __device__ __forceinline__ long long rm_npad(long long n) { return (n + RM_TB - 1) / RM_TB * RM_TB; }
__host__ __device__ __forceinline__ long long rm_frag_index(long long i, int t, int dp) {
    const long long T = i / RM_TB;
    const int il = (int)(i - T * RM_TB), rb = il >> 3, r = il & 7;
    const int ch = t >> 3, e = (t >> 2) & 1, q = t & 3;
    return T * RM_TB * dp + ((long long)(rb * (dp >> 3) + ch) * 32 + 4 * r + q) * 2 + e;
}

struct RbfMma {
    const double* X;     // n x dim row-major (the operator's points)
    double* xf;          // npad x dp fragment-major x~ (prep output)
    double* xb;          // npad: b_i (0 beyond n); xb[npad] = max |x_i|^2 (bits, atomicMax)
    long long n;
    int dim, dp;
    double var, inv2, diag;   // diag = (var + jitter) / var (the E_ii above)
    int nteam;           // teams per CTA (1 or 2)
    long long t_lo, t_hi;   // lower-triangle tiles covered by this launch (a rank's share when sharded)
};

// xf / xb from X (one launch per product or solve; X is read once)
static __global__ void rbf_prep_kernel(RbfMma p) {
    const long long npad = rm_npad(p.n);
    const double sc = sqrt(2.0 * p.inv2);
    const long long total = npad * p.dp;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / p.dp;
        const int t = (int)(e - i * p.dp);
        const double v = (i < p.n && t < p.dim) ? mul_rn(__ldg(p.X + i * p.dim + t), sc) : 0.0;
        p.xf[rm_frag_index(i, t, p.dp)] = v;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npad;
         i += (long long)gridDim.x * blockDim.x) {
        double a = 0.0;
        if (i < p.n)
            for (int t = 0; t < p.dim; ++t) {
                const double x = __ldg(p.X + i * p.dim + t);
                a = fma(x, x, a);
            }
        p.xb[i] = -a * p.inv2;
        // nonnegative doubles order like their bit patterns: a deterministic max
        atomicMax(reinterpret_cast<unsigned long long*>(p.xb + npad), (unsigned long long)__double_as_longlong(a));
    }
}

// ---- shared-memory layout ----------------------------------------------------
// CTA header (doubles): exp table (RM_TAB), mbarriers (4 per team), team sequence
// words, range table (RM_MAX_TEAMS x 255 + 1 longs); then per team: XI frags
// (64 dp), XJ frags x2, I pairs {b, v'} (128), J pairs x2 (256), row-flush
// buffer (8 x 64).
#define RM_TAB 2048
#define RM_HDR 2576
__host__ __device__ __forceinline__ long long rm_team_doubles(int dp) { return 3LL * RM_TB * dp + 128 + 256 + RM_TW * RM_TB; }
__host__ __device__ __forceinline__ long long rm_smem_doubles(int dim, int nteam) {
    return RM_HDR + nteam * rm_team_doubles(rm_dpad(dim));
}
struct RmTeamSmem {
    double* xi;
    double* xj;      // 2 buffers of 64 dp
    double* pi;      // 64 x {b, v'}
    double* pj;      // 2 x 64 x {b, v'}
    double* red;     // 8 x 64
};
__device__ __forceinline__ RmTeamSmem rm_team_smem(double* smem, int dp, int team) {
    RmTeamSmem t;
    double* b = smem + RM_HDR + team * rm_team_doubles(dp);
    t.xi = b;
    t.xj = b + RM_TB * dp;
    t.pi = b + 3 * RM_TB * dp;
    t.pj = t.pi + 128;
    t.red = t.pj + 256;
    return t;
}
__device__ __forceinline__ double* rm_tab(double* smem) { return smem; }
__device__ __forceinline__ unsigned long long* rm_bars(double* smem, int team) {
    return reinterpret_cast<unsigned long long*>(smem + RM_TAB) + 4 * team;
}
__device__ __forceinline__ unsigned* rm_seq(double* smem, int team) {
    return reinterpret_cast<unsigned*>(smem + RM_TAB + 4 * RM_MAX_TEAMS) + 2 * team;
}
__device__ __forceinline__ long long* rm_table(double* smem) {
    return reinterpret_cast<long long*>(smem + RM_TAB + 4 * RM_MAX_TEAMS + RM_MAX_TEAMS);
}
static_assert(RM_TAB + 4 * RM_MAX_TEAMS + RM_MAX_TEAMS + RM_MAX_TEAMS * DCG_SYM_MAX_CTAS + 1 <= RM_HDR, "rbfmma header");
// the pass-2 reduction scratch (512 doubles, generic-proxy only): team 0's flush buffer
__device__ __forceinline__ double* rm_pass2_scratch(double* smem, int dp) { return rm_team_smem(smem, dp, 0).red; }

// ---- primitives --------------------------------------------------------------
__device__ __forceinline__ void rm_team_sync(int team) {
    asm volatile("barrier.sync %0, %1;" ::"r"(1 + team), "r"(RM_TT) : "memory");
}
__device__ __forceinline__ void rm_dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned rm_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void rm_bar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rm_saddr(bar)));
}
// one elected thread: expect `bytes` on `bar` and start the bulk copy gsrc -> sdst
__device__ __forceinline__ void rm_bulk_load(double* sdst, const double* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rm_saddr(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rm_saddr(sdst)),
        "l"(gsrc), "r"(bytes), "r"(rm_saddr(bar))
        : "memory");
}
__device__ __forceinline__ void rm_bar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RM_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RM_WAIT;\n"
        "}\n" ::"r"(rm_saddr(bar)),
        "r"(parity)
        : "memory");
}

// exp(x), table T[j] = 2^(j / 2048) in shared memory: k = rint(2048 x / ln 2)
// via the 1.5 * 2^52 shift, r = x - k ln2/2048 (|r| <= ln2/4096: one FMA with
// the rounded constant, whose relative error 3.3e-17 puts |x| * 3.3e-17 on
// the result -- below an ulp for the entries that carry the sums), expm1(r)
// by its degree-3 Taylor polynomial (truncation r^4/24 < 3.5e-17), result
// T[k & 2047] (1 + expm1 r) scaled by 2^(k >> 11) in the exponent field: 7
// FP64 operations (the 256-entry, degree-4, two-constant form took 9).  The
// exponent-field scaling needs a normal result: CLAMP bounds x below by -700
// (e^-700 ~ 1e-304 then stands in for smaller values), compiled only into the
// path for data that can reach it.
template <bool CLAMP>
__device__ __forceinline__ double rm_exp(double x, const double* tab) {
    if constexpr (CLAMP) x = fmax(x, -700.0);
    const double t = fma(x, 2954.639443740597, 6755399441055744.0);
    const double kf = t - 6755399441055744.0;
    const double r = fma(kf, -0.0003384507717577858, x);
    const int ki = __double2loint(t);
    const double q = fma(r, 1.6666666666666667e-01, 0.5);
    const double r2 = r * r;
    const double pm = fma(q, r2, r);
    const double tj = tab[ki & (RM_TAB - 1)];
    const double res = fma(tj, pm, tj);
    return __hiloint2double(__double2hiint(res) + (ki >> 11) * 1048576, __double2loint(res));
}

// Once per launch (all CTA threads): exp table, mbarriers, team range table.
// Ends with a CTA barrier.
__device__ __forceinline__ void rm_init(double* smem, const RbfMma& p) {
    double* tab = rm_tab(smem);
    for (int j = threadIdx.x; j < RM_TAB; j += blockDim.x) tab[j] = exp2((double)j / RM_TAB);
    if (threadIdx.x < (unsigned)RM_MAX_TEAMS) {
        unsigned long long* b = rm_bars(smem, threadIdx.x);
        rm_bar_init(b);
        rm_bar_init(b + 1);
        rm_bar_init(b + 2);
        unsigned* sq = rm_seq(smem, threadIdx.x);
        sq[0] = sq[1] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    long long* tbl = rm_table(smem);
    const int R = gridDim.x * p.nteam;
    for (int b = threadIdx.x; b <= R; b += blockDim.x) tbl[b] = sym_tile_begin_range(p.n, p.t_lo, p.t_hi, R, b);
    cta_sync();
}

__device__ __forceinline__ double2 rm_pair(const RbfMma& p, const double* v, const double* s, long long j) {
    if (j >= p.n) return make_double2(0.0, 0.0);
    const double vv = ld_cg(v + j);
    return make_double2(__ldg(p.xb + j), mul_rn(p.var, s ? mul_rn(__ldg(s + j), vv) : vv));
}

// One tile for warp w: E values of rows 8 rb + r, columns 8 w + 2 q + {0, 1};
// row sums into rowp[rb], column sums over the warp's rows into col0 / col1.
// DMMAs are issued in an order where consecutive ones use different
// accumulators (4 blocks per half), so the dependent k-steps do not stall.
template <bool DIAG, bool CLAMP>
__device__ __forceinline__ void rm_tile(const RmTeamSmem& S, const double* xj, int nch, int w, int lane, double2 pJ0,
                                        double2 pJ1, const double* tab, double diag, double rowp[8], double& col0,
                                        double& col1) {
    const int r = lane >> 2, q = lane & 3;
    double c[8][2];
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) {
        const double bI = S.pi[2 * (8 * rb + r)];
        c[rb][0] = bI + pJ0.x;
        c[rb][1] = bI + pJ1.x;
    }
    const double2* xi2 = reinterpret_cast<const double2*>(S.xi);
    const double2* xj2 = reinterpret_cast<const double2*>(xj);
    // Two halves of four accumulator blocks: the exponentials of one half have
    // the other half's DMMAs to overlap with (same operation order per element
    // and per sum as the all-DMMAs-first form).
#pragma unroll
    for (int h = 0; h < 8 / RM_GB; ++h) {
        for (int ch = 0; ch < nch; ++ch) {
            const double2 bf = xj2[(w * nch + ch) * 32 + lane];
            double2 af[RM_GB];
#pragma unroll
            for (int u = 0; u < RM_GB; ++u) af[u] = xi2[((RM_GB * h + u) * nch + ch) * 32 + lane];
#pragma unroll
            for (int u = 0; u < RM_GB; ++u) rm_dmma(c[RM_GB * h + u][0], c[RM_GB * h + u][1], af[u].x, bf.x);
#pragma unroll
            for (int u = 0; u < RM_GB; ++u) rm_dmma(c[RM_GB * h + u][0], c[RM_GB * h + u][1], af[u].y, bf.y);
        }
#pragma unroll
        for (int rb = RM_GB * h; rb < RM_GB * h + RM_GB; ++rb) {
            double k0 = rm_exp<CLAMP>(c[rb][0], tab);
            double k1 = rm_exp<CLAMP>(c[rb][1], tab);
            if constexpr (DIAG) {
                if (rb == w) {
                    if (r == 2 * q) k0 = diag;
                    if (r == 2 * q + 1) k1 = diag;
                }
            }
            rowp[rb] = fma(k0, pJ0.y, rowp[rb]);
            rowp[rb] = fma(k1, pJ1.y, rowp[rb]);
            const double vI = S.pi[2 * (8 * rb + r) + 1];
            col0 = fma(k0, vI, col0);
            col1 = fma(k1, vI, col1);
        }
    }
}

// Pass 1 of t = K (s (.) v): colpart / rowpart as in sym_pass1.  All CTA
// threads call; teams >= p.nteam idle.  No CTA barrier inside (team barriers only).
static __device__ void rbf_mma_pass1(const RbfMma& p, const double* v, const double* s, double* colpart, double* rowpart,
                              double* smem) {
    const int team = threadIdx.x / RM_TT;
    if (team >= p.nteam) return;
    const int tt = threadIdx.x - team * RM_TT, lane = tt & 31, w = tt >> 5;
    const int dp = p.dp, nch = dp >> 3;
    const long long n = p.n;
    const RmTeamSmem S = rm_team_smem(smem, dp, team);
    const double* tab = rm_tab(smem);
    unsigned long long* bars = rm_bars(smem, team);   // [0], [1]: XJ buffers, [2]: XI
    unsigned* seq = rm_seq(smem, team);
    const long long* tbl = rm_table(smem);
    const int range = blockIdx.x * p.nteam + team;
    const long long t0 = tbl[range], t1 = tbl[range + 1];
    if (t0 >= t1) return;
    const int ntiles = (int)(t1 - t0);
    const unsigned tile_bytes = (unsigned)(RM_TB * dp * sizeof(double));
    unsigned jseq = seq[0], iseq = seq[1];
    long long I = sym_tile_row(t0);
    long long J = t0 - sym_tile_row_base(I);
    const int r = lane >> 2, q = lane & 3;
    // the exponent can only reach -690 if 4 max|x|^2 / (2 l^2) can
    const double maxn2 = ld_cg(p.xb + rm_npad(n));   // written by rbf_prep_kernel
    const bool clamp = !(4.0 * maxn2 * p.inv2 <= 690.0);

    // prologue: XI(I), XJ(J) in flight; I / J pairs
    rm_team_sync(team);   // previous pass's readers of these buffers are done
    if (tt == 0) {
        rm_bulk_load(S.xi, p.xf + I * RM_TB * dp, tile_bytes, bars + 2);
        rm_bulk_load(S.xj + (jseq & 1) * RM_TB * dp, p.xf + J * RM_TB * dp, tile_bytes, bars + (jseq & 1));
    }
    if (tt < RM_TB) {
        reinterpret_cast<double2*>(S.pi)[tt] = rm_pair(p, v, s, I * RM_TB + tt);
        reinterpret_cast<double2*>(S.pj + (jseq & 1) * 128)[tt] = rm_pair(p, v, s, J * RM_TB + tt);
    }
    rm_bar_wait(bars + 2, iseq & 1);
    ++iseq;
    rm_team_sync(team);

    double rowp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) rowp[u] = 0.0;
    long long seg_start = t0;
    for (int lt = 0; lt < ntiles; ++lt) {
        const int buf = jseq & 1;
        // next tile: bulk copy into the other buffer (free: everyone passed the
        // barrier that ended the previous tile) and its pairs into registers
        long long In = I, Jn = J + 1;
        if (Jn > In) { ++In; Jn = 0; }
        const bool more = lt + 1 < ntiles;
        double2 pn = make_double2(0.0, 0.0);
        if (more) {
            if (tt == 0) rm_bulk_load(S.xj + (buf ^ 1) * RM_TB * dp, p.xf + Jn * RM_TB * dp, tile_bytes, bars + (buf ^ 1));
            if (tt < RM_TB) pn = rm_pair(p, v, s, Jn * RM_TB + tt);
        }
        rm_bar_wait(bars + buf, (jseq >> 1) & 1);
        ++jseq;

        // ---- the tile: 8 accumulator blocks (rows 8 rb + r, cols 8 w + 2 q + e)
        const double* xj = S.xj + buf * RM_TB * dp;
        const double2* pj2 = reinterpret_cast<const double2*>(S.pj + buf * 128);
        const double2 pJ0 = pj2[8 * w + 2 * q], pJ1 = pj2[8 * w + 2 * q + 1];
        const bool diag_tile = (J == I);
        double col0 = 0.0, col1 = 0.0;
        if (diag_tile) {
            if (clamp) rm_tile<true, true>(S, xj, nch, w, lane, pJ0, pJ1, tab, p.diag, rowp, col0, col1);
            else rm_tile<true, false>(S, xj, nch, w, lane, pJ0, pJ1, tab, p.diag, rowp, col0, col1);
        } else {
            if (clamp) rm_tile<false, true>(S, xj, nch, w, lane, pJ0, pJ1, tab, p.diag, rowp, col0, col1);
            else rm_tile<false, false>(S, xj, nch, w, lane, pJ0, pJ1, tab, p.diag, rowp, col0, col1);
        }
        if (!diag_tile) {
            // column sums over the 64 rows: the 8 lanes of equal q (xor 4, 8, 16)
            const bool hi = lane & 16;
            double cv = (hi ? col1 : col0) + __shfl_xor_sync(0xffffffffu, hi ? col0 : col1, 16);
            cv += __shfl_xor_sync(0xffffffffu, cv, 8);
            cv += __shfl_xor_sync(0xffffffffu, cv, 4);
            if ((lane & 12) == 0) colpart[(t0 + lt) * RM_TB + 8 * w + 2 * q + (hi ? 1 : 0)] = cv;
        }
        const bool seg_end = diag_tile || !more;
        if (seg_end) {
            // rows 8 rb + r: the quad's lanes (xor 1, 2), then the 8 warps in a fixed order
            const bool h2 = lane & 2;
            double s4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                s4[u] = (h2 ? rowp[u + 4] : rowp[u]) + __shfl_xor_sync(0xffffffffu, h2 ? rowp[u] : rowp[u + 4], 2);
            const bool h1 = lane & 1;
            double s2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u)
                s2[u] = (h1 ? s4[u + 2] : s4[u]) + __shfl_xor_sync(0xffffffffu, h1 ? s4[u] : s4[u + 2], 1);
            // lane holds rows 8 (4 h2 + 2 h1 + u) + r, u = 0, 1
#pragma unroll
            for (int u = 0; u < 2; ++u) S.red[w * RM_TB + 8 * (4 * h2 + 2 * h1 + u) + r] = s2[u];
            rm_team_sync(team);
            if (tt < RM_TB) {
                double a = 0.0;
#pragma unroll
                for (int u = 0; u < RM_TW; ++u) a += S.red[u * RM_TB + tt];
                rowpart[seg_start * RM_TB + tt] = a;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) rowp[u] = 0.0;
            seg_start = t0 + lt + 1;
        }
        if (more && tt < RM_TB) reinterpret_cast<double2*>(S.pj + (buf ^ 1) * 128)[tt] = pn;
        rm_team_sync(team);   // tile done: buffers of this tile and the flush buffer are free
        if (more && In != I) {
            // new tile row: restage XI and the I pairs
            if (tt == 0) rm_bulk_load(S.xi, p.xf + In * RM_TB * dp, tile_bytes, bars + 2);
            if (tt < RM_TB) reinterpret_cast<double2*>(S.pi)[tt] = rm_pair(p, v, s, In * RM_TB + tt);
            rm_bar_wait(bars + 2, iseq & 1);
            ++iseq;
            rm_team_sync(team);
        }
        I = In;
        J = Jn;
    }
    if (tt == 0) {
        seq[0] = jseq;
        seq[1] = iseq;
    }
}

// ---------------------------------------------------------------------------
// Row-owned products on the FP64 tensor pipe: Y = shift X_rows + s_out (.)
// K (s_in (.) X) for a row slab [row0, row0 + rows) of the operator, X n x kk
// (kk = 8 NB; NB = 0: a single vector).  A 256-thread CTA owns 64-row blocks
// and sweeps every 64-column tile: warp w owns the block's rows 8w..8w+7 and
// all 64 columns of a tile (8 accumulator blocks cb), so
//   * the distance contraction's A fragments (its 8 rows of x~) stay in
//     registers for the whole sweep, B fragments come from the staged tile;
//   * the product E V_J uses E straight from the accumulators: with the k
//     index of k-step e mapped to column 8 cb + 2 q + e, lane (r, q)'s
//     accumulator element e IS the A fragment, and V_J's rows are read in
//     the same order -- no transpose, no shared-memory round trip;
//   * a warp's output rows are complete inside the warp: no column
//     partials (the symmetric pass's per-tile partials would be 64 x kk per
//     tile here) and no cross-warp reduction.
// Used for row slabs (sharded operators) and for the
// multi-vector product of refresh_basis (recycle.py:90).  Costs ~d + 12 + kk
// FP64-pipe operations per element over all n x rows pairs.  Operands: the
// fragment-major x~ and b of rbf_prep_kernel, vs = var s_in (.) X (n_pad x
// kk, zero-padded) or, for NB = 0, var s_in (.) v (n_pad).
// ---------------------------------------------------------------------------
#define RR_NT 256

__device__ __forceinline__ void rr_cp16(void* sdst, const void* gsrc, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(rm_saddr(sdst)), "l"(gsrc), "r"(bytes));
}
__device__ __forceinline__ void rr_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void rr_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int NB>
__host__ __device__ __forceinline__ long long rr_smem_doubles(int dp) {
    const int kk = NB ? 8 * NB : 1;
    const int kks = NB ? kk + 2 : 1;   // padded V row stride (conflict-free B fragment reads)
    return RM_TAB + RM_TB * dp + 2LL * RM_TB * dp + 2LL * RM_TB * kks + 2 * RM_TB + RM_TB + 64;
}

template <int NB>
__global__ void __launch_bounds__(RR_NT, 1)
    rbf_mma_rows_kernel(RbfMma p, long long row0, long long rows, const double* __restrict__ vs,
                        const double* __restrict__ s_out, double shift, const double* __restrict__ x_rows,
                        double* __restrict__ Y, int kout, const dcg_shard_state* gate) {
    if (gate && gate->done) return;   // sharded solve: iterations enqueued past convergence
    constexpr int KK = NB ? 8 * NB : 1;
    constexpr int KKS = NB ? KK + 2 : 1;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int r = lane >> 2, q = lane & 3;
    const int dp = p.dp, nch = dp >> 3;
    const long long n = p.n;
    double* tab = sm;
    double* xi = tab + RM_TAB;                 // 64 x dp (fragment-major, rows of the block)
    double* xj = xi + RM_TB * dp;              // 2 x 64 x dp
    double* vj = xj + 2 * RM_TB * dp;          // 2 x 64 x KKS
    double* bj = vj + 2 * RM_TB * KKS;         // 2 x 64
    double* bi = bj + 2 * RM_TB;               // 64
    for (int j = tid; j < RM_TAB; j += RR_NT) tab[j] = exp2((double)j / RM_TAB);
    const long long ntj = (n + RM_TB - 1) / RM_TB;
    const long long nblk = (rows + RM_TB - 1) / RM_TB;
    // stage tile J (x~ fragments, b, V rows) into buffer `buf` with cp.async
    auto stage = [&](long long J, int buf) {
        const double* src = p.xf + J * RM_TB * dp;
        double* dst = xj + buf * RM_TB * dp;
        for (int c = tid; c < RM_TB * dp / 2; c += RR_NT) rr_cp16(dst + 2 * c, src + 2 * c, 16);
        if (tid < RM_TB / 2) rr_cp16(bj + buf * RM_TB + 2 * tid, p.xb + J * RM_TB + 2 * tid, 16);
        if constexpr (NB) {
            double* vd = vj + buf * RM_TB * KKS;
            const double* vsrc = vs + J * RM_TB * KK;
            for (int c = tid; c < RM_TB * KK / 2; c += RR_NT) {
                const int rr = c / (KK / 2), cc = (c - rr * (KK / 2)) * 2;
                rr_cp16(vd + rr * KKS + cc, vsrc + rr * KK + cc, 16);
            }
        } else {
            if (tid < RM_TB / 2) rr_cp16(vj + buf * RM_TB + 2 * tid, vs + J * RM_TB + 2 * tid, 16);
        }
        rr_commit();
    };
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long i0 = row0 + blk * RM_TB;   // first global row of the block
        cta_sync();   // previous block's readers are done with xi / the buffers
        // the block's own rows (global rows i0.. - not tile-aligned for slabs):
        // fragment-major x~ of rows i0 + 8 w + r, built here from X
        {
            const double sc = sqrt(2.0 * p.inv2);
            for (int e = tid; e < RM_TB * dp; e += RR_NT) {
                const int il = e / dp, t = e - il * dp;
                const long long g = i0 + il;
                const double v = (g < row0 + rows && g < n && t < p.dim) ? mul_rn(__ldg(p.X + g * p.dim + t), sc) : 0.0;
                xi[rm_frag_index(il, t, dp)] = v;
            }
            if (tid < RM_TB) {
                const long long g = i0 + tid;
                bi[tid] = (g < row0 + rows && g < n) ? __ldg(p.xb + g) : 0.0;
            }
        }
        stage(0, 0);
        cta_sync();
        const double bI = bi[8 * w + r];
        double acc[NB ? NB : 1][2];
#pragma unroll
        for (int nb = 0; nb < (NB ? NB : 1); ++nb) acc[nb][0] = acc[nb][1] = 0.0;
        for (long long J = 0; J < ntj; ++J) {
            const int buf = (int)(J & 1);
            rr_wait_all();
            cta_sync();   // tile J landed for everyone; everyone is done with tile J - 1
            if (J + 1 < ntj) stage(J + 1, buf ^ 1);
            const double2* xi2 = reinterpret_cast<const double2*>(xi);
            const double2* xj2 = reinterpret_cast<const double2*>(xj + buf * RM_TB * dp);
            const double* bJ = bj + buf * RM_TB;
            double c[8][2];
#pragma unroll
            for (int cb = 0; cb < 8; ++cb) {
                c[cb][0] = bI + bJ[8 * cb + 2 * q];
                c[cb][1] = bI + bJ[8 * cb + 2 * q + 1];
            }
            for (int ch = 0; ch < nch; ++ch) {
                const double2 af = xi2[(w * nch + ch) * 32 + lane];
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) {
                    const double2 bf = xj2[(cb * nch + ch) * 32 + lane];
                    rm_dmma(c[cb][0], c[cb][1], af.x, bf.x);
                    rm_dmma(c[cb][0], c[cb][1], af.y, bf.y);
                }
            }
            // elements: row i0 + 8 w + r, column 64 J + 8 cb + 2 q + e
            const long long dd = i0 + 8 * w + r - 64 * J;   // diagonal at local column dd
            const bool diag_tile = (i0 + 8 * w + 7 >= 64 * J) && (i0 + 8 * w <= 64 * J + 63);
            const double* vJ = vj + buf * RM_TB * KKS;
#pragma unroll
            for (int cb = 0; cb < 8; ++cb) {
                double e0 = rm_exp<true>(c[cb][0], tab), e1 = rm_exp<true>(c[cb][1], tab);
                if (diag_tile) {
                    if (dd == 8 * cb + 2 * q) e0 = p.diag;
                    if (dd == 8 * cb + 2 * q + 1) e1 = p.diag;
                }
                if constexpr (NB == 0) {
                    acc[0][0] = fma(e0, vJ[8 * cb + 2 * q], acc[0][0]);
                    acc[0][1] = fma(e1, vJ[8 * cb + 2 * q + 1], acc[0][1]);
                } else {
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) {
                        rm_dmma(acc[nb][0], acc[nb][1], e0, vJ[(8 * cb + 2 * q) * KKS + 8 * nb + r]);
                        rm_dmma(acc[nb][0], acc[nb][1], e1, vJ[(8 * cb + 2 * q + 1) * KKS + 8 * nb + r]);
                    }
                }
            }
        }
        // epilogue: the warp's 8 rows
        if constexpr (NB == 0) {
            double t = acc[0][0] + acc[0][1];
            t += __shfl_xor_sync(0xffffffffu, t, 1);
            t += __shfl_xor_sync(0xffffffffu, t, 2);
            const long long g = i0 + 8 * w + r;
            if (q == 0 && g < row0 + rows) {
                const long long li = g - row0;
                double val = s_out ? mul_rn(s_out[li], t) : t;
                if (shift != 0.0) val = add_rn(mul_rn(shift, x_rows[li]), val);
                Y[li] = val;
            }
        } else {
            // C fragment: row 8 w + r, columns 8 nb + 2 q + {0, 1}
            const long long g = i0 + 8 * w + r;
            if (g < row0 + rows) {
                const long long li = g - row0;
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * nb + 2 * q + e;
                        if (col < kout) {
                            double val = s_out ? mul_rn(s_out[li], acc[nb][e]) : acc[nb][e];
                            if (shift != 0.0) val = add_rn(mul_rn(shift, x_rows[li * kout + col]), val);
                            Y[li * kout + col] = val;
                        }
                    }
            }
        }
    }
}

// vs = var s_in (.) X, zero-padded to n_pad x kk (kk >= k); k = 0 means a vector
static __global__ void rr_scale_kernel(const double* X, int k, int kk, const double* s_in, double var, long long n,
                                       long long npad, double* vs) {
    const long long total = npad * (k ? kk : 1);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = k ? e / kk : e;
        const int c = k ? (int)(e - i * kk) : 0;
        double v = 0.0;
        if (i < n && c < (k ? k : 1)) {
            const double x = k ? X[i * k + c] : X[i];
            v = mul_rn(var, s_in ? mul_rn(s_in[i], x) : x);
        }
        vs[e] = v;
    }
}
