// Operator application and block products.
//
//   gemv_kernel      y = shift v + s_out (.) K (s_in (.) v)   (K1, standalone)
//   dmma_gemm_kernel Y = K V on FP64 tensor cores            (K3, A.W refresh, recycle.py:90)
//   xty_kernel       C = X' Y tall-skinny products           (K4, W'AW, F, G; solvers.py:109,
//                                                              recycle.py:71,133-136)
//   gemm_lr_kernel   C = A B with the reference's i-k-j order (K4, Z.U; _core.pyx:31-44)
#include "common.cuh"
#include <algorithm>
#include "gemv.cuh"
#include "symgemv.cuh"


// =============================================================================
// K1 standalone GEMV: one CTA per contiguous row range (grid = #SM).
// =============================================================================
__global__ void __launch_bounds__(DCG_NT, 1)
    gemv_kernel(const double* __restrict__ K, long long ldk, long long n, long long rows,
                const double* v, const double* s_in, const double* s_out, double shift,
                const double* v_rows, double* y) {
    extern __shared__ __align__(16) double smem[];
    const int xt = (int)min(n, (long long)DCG_QT) + 2;
    double* s_x = smem;
    double* s_red = s_x + xt;
    const long long r0 = part_begin(rows, gridDim.x, blockIdx.x);
    const long long r1 = part_begin(rows, gridDim.x, blockIdx.x + 1);
    block_gemv<false>(K, ldk, n, v, s_in, r0, r1, s_x, s_red, [&](long long i, double t) {
        double val = s_out ? mul_rn(s_out[i], t) : t;
        if (shift != 0.0) val = add_rn(mul_rn(shift, v_rows[i]), val);
        y[i] = val;
    });
}

static size_t gemv_smem(long long n) {
    const long long xt = (n < DCG_QT ? n : DCG_QT) + 2;
    return sizeof(double) * (size_t)(xt + DCG_NW * DCG_RB);
}

int dcg_gemv_launch(dcg_context* ctx, cudaStream_t st, const double* K, long long ldk, long long n,
                    long long rows, const double* v, const double* s_in, const double* s_out,
                    double shift, const double* v_rows, double* y) {
    if (rows <= 0) return DCG_OK;
    if ((ldk & 1) || (reinterpret_cast<uintptr_t>(K) & 15)) return DCG_E_CONFIG;
    const size_t smem = gemv_smem(n);
    DCG_CUDA(cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    long long blocks = ctx->sm_count;
    if (blocks > rows) blocks = rows;
    gemv_kernel<<<(unsigned)blocks, DCG_NT, smem, st>>>(K, ldk, n, rows, v, s_in, s_out, shift, v_rows, y);
    DCG_LAUNCHED();
    return DCG_OK;
}

// =============================================================================
// K1 over the lower triangle of a symmetric K (symgemv.cuh): pass 1 streams
// the tiles, pass 2 combines the per-tile partials.  Both launches use the
// same grid, which fixes the tile partition.
// =============================================================================
// Packed copy (dcg_pack_sym): one CTA per 64 x 64 lower-triangle tile; each
// thread moves 16-byte chunks (r, q) from the row-major rows into the tile's
// swizzled slot, zero beyond n.
__global__ void __launch_bounds__(256) pack_sym_kernel(const double* __restrict__ K, long long ldk, long long n,
                                                       double* __restrict__ kp) {
    const long long t = blockIdx.x;
    const long long I = sym_tile_row(t), J = t - sym_tile_row_base(I);
    double* dst = kp + t * DCG_SYM_TILE_DOUBLES;
    for (int c = threadIdx.x; c < DCG_SYM_TILE_DOUBLES / 2; c += blockDim.x) {
        const int r = c >> 5, q = c & 31;
        const long long gi = I * DCG_TB + r, gj = J * DCG_TB + 2 * q;
        double2 val = make_double2(0.0, 0.0);
        if (gi < n) {
            const double* src = K + gi * ldk + gj;
            if (gj + 1 < n) val = __ldg(reinterpret_cast<const double2*>(src));
            else if (gj < n) val.x = __ldg(src);
        }
        *reinterpret_cast<double2*>(dst + sym_swz(r, 2 * q)) = val;
    }
}

extern "C" long long dcg_packed_sym_doubles(long long n) { return n > 0 ? sym_packed_doubles(n) : 0; }

extern "C" int dcg_pack_sym(dcg_context* ctx, void* stream, const double* d_k, long long ldk, long long n,
                            double* d_kp) {
    if (!ctx || n < 0 || ldk < n || (ldk & 1) || !aligned16(d_k) || !aligned16(d_kp)) return DCG_E_CONFIG;
    if (n == 0) return DCG_OK;
    const long long ntt = sym_ntiles(n);
    if (ntt > 0x7fffffffLL) return DCG_E_UNSUPPORTED;
    pack_sym_kernel<<<(unsigned)ntt, 256, 0, as_stream(stream)>>>(d_k, ldk, n, d_kp);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Both passes in one cooperative launch (grid barrier between them): no
// second launch, and pass 2's partial reads follow pass 1 without a gap.
template <bool PK>
__global__ void __launch_bounds__(DCG_NT, 1)
    sym_apply_coop_kernel(const double* __restrict__ K, long long ldk, long long n, const double* v,
                          const double* s_in, const double* s_out, double shift, double* colpart, double* rowpart,
                          double* y, unsigned int* bar, unsigned long long* ts, const long long* gtbl) {
    extern __shared__ __align__(16) double smem[];
#define APPLY_TS(i) \
    if (ts && threadIdx.x == 0) ts[blockIdx.x * 5 + (i)] = globaltimer_ns()
    APPLY_TS(0);
    sym_ring_init(smem, n, PK, gtbl);
    APPLY_TS(1);
    unsigned int seq = 0;
    sym_pass1<false, 1, PK>(K, ldk, n, v, s_in, colpart, rowpart, smem, seq);
    APPLY_TS(2);
    dcg_grid_barrier(bar, gridDim.x);
    APPLY_TS(3);
    const long long q0 = sym_row_begin(n, gridDim.x, blockIdx.x);
    const long long q1 = sym_row_begin(n, gridDim.x, blockIdx.x + 1);
    sym_pass2<true>(n, colpart, rowpart, q0, q1, sym_range_table(smem), gridDim.x, smem, [&](long long i, double t) {
        double val = s_out ? mul_rn(s_out[i], t) : t;
        if (shift != 0.0) val = add_rn(mul_rn(shift, v[i]), val);
        y[i] = val;
    });
    APPLY_TS(4);
#undef APPLY_TS
    if (threadIdx.x == 0) dcg_sync_exit(bar, gridDim.x);
}

// DCG_APPLY_TIMERS=1 (developer diagnostic): per-CTA globaltimer stamps of the
// last standalone symmetric product (start, after the ring set-up, after pass
// 1, after the grid barrier, end), 5 per CTA.
static unsigned long long* g_apply_ts = nullptr;
extern "C" __attribute__((visibility("default"))) int dcg_debug_apply_timers(unsigned long long* out, int nslots) {
    if (!g_apply_ts || !out || nslots < 0 || nslots > 5 * 256) return DCG_E_CONFIG;
    DCG_CUDA(cudaMemcpy(out, g_apply_ts, (size_t)nslots * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return DCG_OK;
}

__global__ void __launch_bounds__(DCG_NT, 1)
    sym_pass2_kernel(long long n, int R, const double* colpart, const double* rowpart, const double* v,
                     const double* s_out, double shift, double* y) {
    __shared__ long long tbl[2 * DCG_SYM_MAX_CTAS + 1];
    __shared__ double red[DCG_NT];
    sym_fill_range_table(tbl, n, R);
    const long long q0 = sym_row_begin(n, gridDim.x, blockIdx.x);
    const long long q1 = sym_row_begin(n, gridDim.x, blockIdx.x + 1);
    sym_pass2<true>(n, colpart, rowpart, q0, q1, tbl, R, red, [&](long long i, double t) {
        double val = s_out ? mul_rn(s_out[i], t) : t;
        if (shift != 0.0) val = add_rn(mul_rn(shift, v[i]), val);
        y[i] = val;
    });
}

size_t dcg_sym_apply_scratch_doubles(long long n) { return 2 * (size_t)sym_ntiles(n) * DCG_TB + 32; }

// y = shift v + s_out (.) K (s_in (.) v) with K exactly symmetric (n x n, unsharded).
// Kp (optional): the packed tiles of K (dcg_pack_sym), read instead of K.
int dcg_sym_apply(dcg_context* ctx, cudaStream_t st, const double* K, const double* Kp, long long ldk, long long n,
                  const double* v, const double* s_in, const double* s_out, double shift, double* y,
                  double* scratch) {
    if (n <= 0) return DCG_OK;
    // One SM is left to the single-CTA Ritz pencil that the def-CG sequence
    // runs concurrently on the side stream (the K-products of the Newton
    // update overlap it): the pass-1 CTAs ask for the whole opt-in shared
    // memory, so none of them can share the pencil's SM, and they are one
    // fewer than the SMs.  A CTA sharing the pencil's SM had stretched both
    // (pencil 220 -> 360 us, pass 1 73 -> 117 us).
    size_t smem = sizeof(double) * (size_t)sym_smem_doubles();
    if (ctx->smem_optin > smem) smem = ctx->smem_optin;
    const long long ntt = sym_ntiles(n);
    double* colpart = scratch;
    double* rowpart = scratch + ntt * DCG_TB;
    const int navail = ctx->sm_count > 1 ? ctx->sm_count - 1 : 1;
    const int G = navail < DCG_SYM_MAX_CTAS ? navail : DCG_SYM_MAX_CTAS;
    // one cooperative launch: pass 1, grid barrier, pass 2 (the barrier word:
    // the context's persistent line, no memset)
    unsigned int* bar = dcg_sync_line(ctx, DCG_SW_APPLY);
    const void* kfn = Kp ? (const void*)sym_apply_coop_kernel<true> : (const void*)sym_apply_coop_kernel<false>;
    if (Kp) DCG_SMEM_ATTR(sym_apply_coop_kernel<true>, smem);
    else DCG_SMEM_ATTR(sym_apply_coop_kernel<false>, smem);
    const double* Ksrc = Kp ? Kp : K;
    const long long* gtbl = dcg_sym_table(ctx, st, n, G);
    if (!gtbl) return DCG_E_CUDA;
    unsigned long long* ts = nullptr;
    if (getenv("DCG_APPLY_TIMERS")) {
        if (!g_apply_ts) DCG_CUDA(cudaMalloc(&g_apply_ts, 5 * 256 * sizeof(unsigned long long)));
        ts = g_apply_ts;
    }
    void* args[] = {(void*)&Ksrc, (void*)&ldk, (void*)&n, (void*)&v, (void*)&s_in, (void*)&s_out, (void*)&shift,
                    (void*)&colpart, (void*)&rowpart, (void*)&y, (void*)&bar, (void*)&ts, (void*)&gtbl};
    DCG_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(DCG_NT), args, smem, st));
    dcg_count_launch();
    return DCG_OK;
}

// Two products over one pass of K's lower triangle (sym_pass1<NV = 2>):
//   y1 = shift1 v1 + s_out1 (.) K x1,   y2 = shift2 v2 + s_out2 (.) K x2
// x1, x2 are the (already input-scaled) operands, v1, v2 the shift vectors.
// Same tile partition, partial layout and pass-2 order as two dcg_sym_apply
// calls with (v, s_in) such that x = s_in (.) v: bitwise the same results.
template <bool PK>
__global__ void __launch_bounds__(DCG_NT, 1)
    sym_apply2_coop_kernel(const double* __restrict__ K, long long ldk, long long n, const double* x1,
                           const double* x2, const double* v1, const double* v2, const double* s_out1,
                           const double* s_out2, double shift1, double shift2, double* colpart, double* rowpart,
                           long long part2, double* y1, double* y2, unsigned int* bar, const long long* gtbl) {
    extern __shared__ __align__(16) double smem[];
    sym_ring_init(smem, n, PK, gtbl);
    unsigned int seq = 0;
    // (no L2 cache hints on the row-major copies of the standalone products: a
    // cp.async with a cache hint faulted here as an illegal instruction on sm_100a)
    sym_pass1<false, 2, PK>(K, ldk, n, x1, nullptr, colpart, rowpart, smem, seq, x2, part2);
    dcg_grid_barrier(bar, gridDim.x);
    const long long q0 = sym_row_begin(n, gridDim.x, blockIdx.x);
    const long long q1 = sym_row_begin(n, gridDim.x, blockIdx.x + 1);
    sym_pass2<true>(n, colpart, rowpart, q0, q1, sym_range_table(smem), gridDim.x, smem, [&](long long i, double t) {
        double val = s_out1 ? mul_rn(s_out1[i], t) : t;
        if (shift1 != 0.0) val = add_rn(mul_rn(shift1, v1[i]), val);
        y1[i] = val;
    });
    sym_pass2<true>(n, colpart + part2, rowpart + part2, q0, q1, sym_range_table(smem), gridDim.x, smem,
              [&](long long i, double t) {
                  double val = s_out2 ? mul_rn(s_out2[i], t) : t;
                  if (shift2 != 0.0) val = add_rn(mul_rn(shift2, v2[i]), val);
                  y2[i] = val;
              });
    if (threadIdx.x == 0) dcg_sync_exit(bar, gridDim.x);
}

size_t dcg_sym_apply2_scratch_doubles(long long n) { return 4 * (size_t)sym_ntiles(n) * DCG_TB + 32; }

int dcg_sym_apply2(dcg_context* ctx, cudaStream_t st, const double* K, const double* Kp, long long ldk, long long n,
                   const double* x1,
                   const double* x2, const double* v1, const double* v2, const double* s_out1, const double* s_out2,
                   double shift1, double shift2, double* y1, double* y2, double* scratch) {
    if (n <= 0) return DCG_OK;
    size_t smem = sizeof(double) * (size_t)sym_smem_doubles();
    if (ctx->smem_optin > smem) smem = ctx->smem_optin;
    const long long ntt = sym_ntiles(n);
    double* colpart = scratch;
    double* rowpart = scratch + ntt * DCG_TB;
    const long long part2 = 2 * ntt * DCG_TB;
    // the CTA count of dcg_sym_apply (same partition -> same partials)
    const int navail = ctx->sm_count > 1 ? ctx->sm_count - 1 : 1;
    const int G = navail < DCG_SYM_MAX_CTAS ? navail : DCG_SYM_MAX_CTAS;
    unsigned int* bar = dcg_sync_line(ctx, DCG_SW_APPLY2);
    const void* kfn = Kp ? (const void*)sym_apply2_coop_kernel<true> : (const void*)sym_apply2_coop_kernel<false>;
    if (Kp) DCG_SMEM_ATTR(sym_apply2_coop_kernel<true>, smem);
    else DCG_SMEM_ATTR(sym_apply2_coop_kernel<false>, smem);
    const double* Ksrc = Kp ? Kp : K;
    const long long* gtbl = dcg_sym_table(ctx, st, n, G);
    if (!gtbl) return DCG_E_CUDA;
    void* args[] = {(void*)&Ksrc,      (void*)&ldk,    (void*)&n,      (void*)&x1,      (void*)&x2,
                    (void*)&v1,     (void*)&v2,     (void*)&s_out1, (void*)&s_out2,  (void*)&shift1,
                    (void*)&shift2, (void*)&colpart, (void*)&rowpart, (void*)&part2, (void*)&y1,
                    (void*)&y2,     (void*)&bar,    (void*)&gtbl};
    DCG_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(DCG_NT), args, smem, st));
    dcg_count_launch();
    return DCG_OK;
}

// pass 2 alone (the matrix-free operator's symmetric pass 1 produces the same partials)
// (R = pass-1 ranges: G x teams)
int dcg_sym_pass2_launch(cudaStream_t st, int G, int R, long long n, const double* colpart, const double* rowpart,
                         const double* v, const double* s_out, double shift, double* y) {
    sym_pass2_kernel<<<G, DCG_NT, 0, st>>>(n, R, colpart, rowpart, v, s_out, shift, y);
    DCG_LAUNCHED();
    return DCG_OK;
}

// =============================================================================
// K3: Y(rows x k) = K(rows x n) V(n x k) with mma.sync.m8n8k4 FP64.
// CTA = 8 warps = 128 rows x all k columns; blockIdx.y splits the inner
// dimension (partials reduced in a fixed order by yscale_reduce_kernel).
// Operand tiles are staged with cp.async double buffering; the inner index is
// permuted inside each 8-chunk (thread loads a 16-byte pair for two MMAs),
// which leaves every dot product unchanged.
// =============================================================================
#define GM_BM 128                // 8 warps x 16 rows: each B fragment feeds two row tiles
#define GM_BK 32
#define GM_SA (GM_BK + 4)        // A row stride (doubles): conflict-free 16 B fragment loads

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gsrc),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NTILE>
__global__ void __launch_bounds__(256)
    dmma_gemm_kernel(const double* __restrict__ K, long long ldk, long long rows, long long n,
                     const double* __restrict__ V, int kcols, long long split_cols, double* P) {
    constexpr int KP = NTILE * 8;          // padded k
    constexpr int SB = KP + 4;             // B row stride
    extern __shared__ __align__(16) double sm[];
    double* sA = sm;                       // 2 x GM_BM x GM_SA
    double* sB = sA + 2 * GM_BM * GM_SA;   // 2 x GM_BK x SB
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const long long row0 = (long long)blockIdx.x * GM_BM;
    const long long cbeg = (long long)blockIdx.y * split_cols;
    long long cend = cbeg + split_cols;
    if (cend > n) cend = n;
    const int ntiles = (int)((cend - cbeg + GM_BK - 1) / GM_BK);

    auto load_tile = [&](int buf, long long c0) {
        double* a = sA + buf * GM_BM * GM_SA;
        // A: 64 rows x 32 cols = 1024 16-byte chunks
        for (int ch = tid; ch < GM_BM * (GM_BK / 2); ch += 256) {
            const int r = ch / (GM_BK / 2), cc = (ch % (GM_BK / 2)) * 2;
            const long long gr = row0 + r, gc = c0 + cc;
            int bytes = 0;
            const double* src = K;
            if (gr < rows && gc < cend) {
                bytes = (gc + 1 < cend) ? 16 : 8;
                src = K + gr * ldk + gc;
            }
            cp_async16(a + r * GM_SA + cc, src, bytes);
        }
        double* bsm = sB + buf * GM_BK * SB;
        // B: 32 rows x KP cols (kcols valid)
        for (int ch = tid; ch < GM_BK * (KP / 2); ch += 256) {
            const int r = ch / (KP / 2), cc = (ch % (KP / 2)) * 2;
            const long long gr = c0 + r;
            int bytes = 0;
            const double* src = V;
            if (gr < cend && cc < kcols) {
                bytes = (cc + 1 < kcols) ? 16 : 8;
                src = V + gr * kcols + cc;
            }
            // V rows are kcols long; 16-byte alignment needs kcols even (checked on host)
            cp_async16(bsm + r * SB + cc, src, bytes);
        }
    };

    double acc[2][NTILE][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < NTILE; ++j) acc[h][j][0] = acc[h][j][1] = 0.0;

    if (ntiles > 0) {
        load_tile(0, cbeg);
        cp_async_commit();
    }
    for (int tI = 0; tI < ntiles; ++tI) {
        const int buf = tI & 1;
        if (tI + 1 < ntiles) {
            load_tile(buf ^ 1, cbeg + (long long)(tI + 1) * GM_BK);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        cta_sync();
        const double* a = sA + buf * GM_BM * GM_SA + (warp * 16 + g) * GM_SA;
        const double* bsm = sB + buf * GM_BK * SB;
#pragma unroll
        for (int kk = 0; kk < GM_BK / 8; ++kk) {
            const double2 av0 = *reinterpret_cast<const double2*>(a + kk * 8 + 2 * t);
            const double2 av1 = *reinterpret_cast<const double2*>(a + 8 * GM_SA + kk * 8 + 2 * t);
            const double* b0 = bsm + (kk * 8 + 2 * t) * SB + g;
#pragma unroll
            for (int j = 0; j < NTILE; ++j) {
                const double bx = b0[j * 8], by = b0[SB + j * 8];
                dmma(acc[0][j][0], acc[0][j][1], av0.x, bx);
                dmma(acc[1][j][0], acc[1][j][1], av1.x, bx);
                dmma(acc[0][j][0], acc[0][j][1], av0.y, by);
                dmma(acc[1][j][0], acc[1][j][1], av1.y, by);
            }
        }
        cta_sync();
    }
    // D fragment: row = g, cols 2t, 2t+1 of each n-tile (two row tiles per warp)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const long long r = row0 + warp * 16 + 8 * h + g;
        if (r < rows) {
            double* out = P + ((long long)blockIdx.y * rows + r) * kcols;
#pragma unroll
            for (int j = 0; j < NTILE; ++j) {
                const int c = j * 8 + 2 * t;
                if (c < kcols) out[c] = acc[h][j][0];
                if (c + 1 < kcols) out[c + 1] = acc[h][j][1];
            }
        }
    }
}

// V = s (.) X  (row scaling of an n x k block)
__global__ void rowscale_kernel(const double* X, const double* s, long long n, int k, double* V) {
    const long long total = n * k;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / k;
        V[e] = s ? mul_rn(s[i], X[e]) : X[e];
    }
}

// V (n x kk, kk >= k) = s (.) X with zero padding columns (s may be null)
__global__ void pad_scale_kernel(const double* X, int k, const double* s, long long n, int kk, double* V) {
    const long long total = n * kk;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / kk;
        const int c = (int)(e - i * kk);
        double v = 0.0;
        if (c < k) {
            v = X[i * k + c];
            if (s) v = mul_rn(s[i], v);
        }
        V[e] = v;
    }
}

// Y[i][j] = shift X[i][j] + s_out[i] * sum_split P[split][i][j]   (fixed split order)
__global__ void yscale_reduce_kernel(const double* P, int splits, long long rows, int k,
                                     const double* X_rows, const double* s_out, double shift,
                                     double* Y) {
    const long long total = rows * k;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        double acc = P[e];
        for (int sp = 1; sp < splits; ++sp) acc += P[(long long)sp * total + e];
        const long long i = e / k;
        double val = s_out ? mul_rn(s_out[i], acc) : acc;
        if (shift != 0.0) val = add_rn(mul_rn(shift, X_rows[e]), val);
        Y[e] = val;
    }
}

template <int NTILE>
static int launch_dmma(dcg_context* ctx, cudaStream_t st, const double* K, long long ldk,
                       long long rows, long long n, const double* V, int k, double* P,
                       int& splits_out) {
    constexpr int KP = NTILE * 8;
    const size_t smem = sizeof(double) * (size_t)(2 * GM_BM * GM_SA + 2 * GM_BK * (KP + 4));
    // attribute and occupancy once per instantiation and device: these host
    // calls sat between the refresh's launches
    static std::atomic<long long> occ_cache[DCG_MAX_DEVICES];
    int per_sm = 0;
    DCG_SMEM_ATTR(dmma_gemm_kernel<NTILE>, smem);
    int rc_ = dcg_occupancy_cached(occ_cache, (const void*)dmma_gemm_kernel<NTILE>, 256, smem, &per_sm);
    if (rc_) return rc_;
    const long long row_tiles = (rows + GM_BM - 1) / GM_BM;
    const long long target = 2LL * (per_sm < 1 ? 1 : per_sm) * ctx->sm_count;   // ~2 waves
    long long splits = (target + row_tiles - 1) / row_tiles;
    const long long max_splits = (n + GM_BK - 1) / GM_BK;
    if (splits > max_splits) splits = max_splits;
    if (splits > 64) splits = 64;
    if (splits < 1) splits = 1;
    long long split_cols = (n + splits - 1) / splits;
    split_cols = (split_cols + GM_BK - 1) / GM_BK * GM_BK;
    splits = (n + split_cols - 1) / split_cols;
    splits_out = (int)splits;
    dim3 grid((unsigned)row_tiles, (unsigned)splits);
    dmma_gemm_kernel<NTILE><<<grid, 256, smem, st>>>(K, ldk, rows, n, V, k, split_cols, P);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Y = shift X_rows + s_out (.) K (s_in (.) X); X is n x k, Y rows x k.
size_t dcg_block_apply_scratch_doubles(long long n, long long rows, int k) {
    const long long kk = (k + 1) & ~1;
    return (size_t)(n * kk + 64 * rows * kk);
}

// `scratch` holds dcg_block_apply_scratch_doubles(n, rows, k) doubles.
int dcg_block_apply(dcg_context* ctx, cudaStream_t st, const double* K, long long ldk,
                    long long rows, long long n, const double* X, int k, const double* s_in,
                    const double* s_out, double shift, const double* X_rows, double* Y,
                    double* scratch) {
    if (k <= 0 || rows <= 0) return DCG_OK;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    if ((ldk & 1) || (reinterpret_cast<uintptr_t>(K) & 15)) return DCG_E_CONFIG;
    const int kk = (k + 1) & ~1;   // even width for 16-byte staging of V
    const size_t vbytes = sizeof(double) * (size_t)(n * kk);
    int rc = DCG_OK;
    double* V = scratch;
    double* P = V + n * kk;
    (void)vbytes;
    // V = s_in (.) X, padded to an even column count, in one pass (X itself
    // when it needs neither: V is only read)
    const double* Vin = V;
    if (kk != k || s_in || (reinterpret_cast<uintptr_t>(X) & 15)) {
        pad_scale_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(X, k, s_in, n, kk, V);
        DCG_LAUNCHED();
    } else {
        Vin = X;
    }
    int splits = 1;
    const int ntile = (kk + 7) / 8;
    switch (ntile) {
        case 1: rc = launch_dmma<1>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 2: rc = launch_dmma<2>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 3: rc = launch_dmma<3>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 4: rc = launch_dmma<4>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 5: rc = launch_dmma<5>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 6: rc = launch_dmma<6>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        case 7: rc = launch_dmma<7>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
        default: rc = launch_dmma<8>(ctx, st, K, ldk, rows, n, Vin, kk, P, splits); break;
    }
    if (rc) return rc;
    if (kk == k) {
        yscale_reduce_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(P, splits, rows, k, X_rows, s_out, shift, Y);
        DCG_LAUNCHED();
    } else {
        // reduce into the padded layout of V (no longer needed), then compact
        yscale_reduce_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(P, splits, rows, kk, nullptr, s_out, 0.0, V);
        DCG_LAUNCHED();
        DCG_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * k, V, sizeof(double) * kk, sizeof(double) * k, rows,
                                   cudaMemcpyDeviceToDevice, st));
        if (shift != 0.0) {
            // Y += shift X_rows (separate pass keeps the reference's (s*t) + shift*x order)
            yscale_reduce_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(Y, 1, rows, k, X_rows, nullptr, shift, Y);
            DCG_LAUNCHED();
        }
    }
    return DCG_OK;
}

// =============================================================================
// K4: C(p x q) = X(n x p)' Y(n x q), tall-skinny, deterministic two-stage.
// CTA b sums its rows [r0, r1) in ascending order into a partial (one fused
// multiply-add per row and pair); the partials are summed in CTA order.  Both
// stages are one launch: the last CTA to finish (cta_last_arrival on the
// context's persistent counter) does the ordered sum.  The CTA stages its
// rows in chunks of `cr` (the whole range when it fits: one load round), so
// the per-pair sequence of operations -- and the result -- does not depend on
// the chunking.
// =============================================================================
#define XTY_AHEAD 32  // partial loads in flight per element of the final sum
template <int XTY_PPT>   // pairs per thread (1: p q <= 256, the usual W'AW / W'v)
__global__ void __launch_bounds__(256)
    xty_kernel(const double* __restrict__ X, long long ldx, const double* __restrict__ Y, long long ldy,
               long long n, int p, int q, int cr, double* part, double* C, unsigned int* counter) {
    extern __shared__ double xty_sm[];
    double* sx = xty_sm;                // cr x p
    double* sy = xty_sm + cr * p;       // cr x q
    const int tid = threadIdx.x;
    const long long r0 = part_begin(n, gridDim.x, blockIdx.x);
    const long long r1 = part_begin(n, gridDim.x, blockIdx.x + 1);
    const int pq = p * q;
    const int pair0 = blockIdx.y * (256 * XTY_PPT);
    double acc[XTY_PPT];
    int pa[XTY_PPT], pb[XTY_PPT];
#pragma unroll
    for (int u = 0; u < XTY_PPT; ++u) {
        acc[u] = 0.0;
        const int e = pair0 + u * 256 + tid;
        pa[u] = (e < pq) ? e / q : -1;
        pb[u] = (e < pq) ? e % q : 0;
    }
    for (long long rb = r0; rb < r1; rb += cr) {
        const int nr = (int)min((long long)cr, r1 - rb);
        cta_sync();
        if (ldx == p) {
            for (int e = tid; e < nr * p; e += 256) sx[e] = X[rb * p + e];
        } else {
            for (int e = tid; e < nr * p; e += 256) sx[e] = X[(rb + e / p) * ldx + e % p];
        }
        if (ldy == q) {
            for (int e = tid; e < nr * q; e += 256) sy[e] = Y[rb * q + e];
        } else {
            for (int e = tid; e < nr * q; e += 256) sy[e] = Y[(rb + e / q) * ldy + e % q];
        }
        cta_sync();
        for (int r = 0; r < nr; ++r) {
#pragma unroll
            for (int u = 0; u < XTY_PPT; ++u)
                if (pa[u] >= 0) acc[u] = fma(sx[r * p + pa[u]], sy[r * q + pb[u]], acc[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < XTY_PPT; ++u) {
        const int e = pair0 + u * 256 + tid;
        if (e < pq) part[(long long)blockIdx.x * pq + e] = acc[u];
    }
    if (!C) return;
    // ---- the last CTA: C = partials summed in CTA order (reduce_parts' order)
    if (!cta_last_arrival(counter, gridDim.x * gridDim.y)) return;
    const int nparts = gridDim.x;
    for (int e = tid; e < pq; e += 256) {
        double t = 0.0;
        int b = 0;
        for (; b + XTY_AHEAD <= nparts; b += XTY_AHEAD) {
            double v[XTY_AHEAD];
#pragma unroll
            for (int u = 0; u < XTY_AHEAD; ++u) v[u] = ld_cg(part + (long long)(b + u) * pq + e);
#pragma unroll
            for (int u = 0; u < XTY_AHEAD; ++u) t += v[u];
        }
        for (; b < nparts; ++b) t += ld_cg(part + (long long)b * pq + e);
        C[e] = t;
    }
}

// Partials summed in CTA order; eight loads are issued ahead of their adds
// (same order, same result: the loop had paid one L2 round trip per partial)
__global__ void reduce_parts_kernel(const double* part, int nparts, int m, double* out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        double acc = 0.0;
        int b = 0;
        for (; b + 8 <= nparts; b += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ld_cg(part + (long long)(b + u) * m + e);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
        for (; b < nparts; ++b) acc += ld_cg(part + (long long)b * m + e);
        out[e] = acc;
    }
}

int dcg_xty(dcg_context* ctx, cudaStream_t st, const double* X, long long ldx, const double* Y,
            long long ldy, long long n, int p, int q, double* C, double* scratch_parts) {
    if (p <= 0 || q <= 0) return DCG_OK;
    if (p > DCG_MAX_T || q > DCG_MAX_T) return DCG_E_UNSUPPORTED;
    int nb = ctx->sm_count;
    if (n < (long long)nb * 32) nb = (int)max(1LL, (n + 31) / 32);
    const int pq = p * q;
    dim3 grid(nb, (pq + 256 * 8 - 1) / (256 * 8));
    // rows staged per round: the CTA's whole range when it fits 64 KB
    const long long range = (n + nb - 1) / nb;
    const long long cap = max(32LL, (long long)(65536 / (sizeof(double) * (p + q))));
    const int cr = (int)max(1LL, min(range, cap));
    const size_t smem = sizeof(double) * (size_t)cr * (size_t)(p + q);
    // the last-arrival counter: the context's persistent line (reset by the last CTA)
    unsigned int* counter = dcg_sync_line(ctx, DCG_SW_XTY);
    if (pq <= 256) {
        DCG_SMEM_ATTR(xty_kernel<1>, smem);
        xty_kernel<1><<<dim3(nb, (pq + 255) / 256), 256, smem, st>>>(X, ldx, Y, ldy, n, p, q, cr, scratch_parts, C,
                                                                    counter);
    } else {
        DCG_SMEM_ATTR(xty_kernel<8>, smem);
        xty_kernel<8><<<grid, 256, smem, st>>>(X, ldx, Y, ldy, n, p, q, cr, scratch_parts, C, counter);
    }
    DCG_LAUNCHED();
    return DCG_OK;
}

size_t dcg_xty_scratch_doubles(dcg_context* ctx, int p, int q) { return (size_t)ctx->sm_count * p * q; }

// =============================================================================
// C(m x n) = A(m x kk) B(kk x n) in the reference's i-k-j accumulation order
// (each C[i][j] sums k ascending with separate multiply and add, _core.pyx:31-44).
// =============================================================================
__global__ void gemm_lr_kernel(const double* __restrict__ A, long long lda, const double* __restrict__ B,
                               long long ldb, double* C, long long ldc, long long m, long long kk,
                               long long n) {
    const long long total = m * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / n, j = e % n;
        double acc = 0.0;
        for (long long t = 0; t < kk; ++t) acc = add_rn(acc, mul_rn(A[i * lda + t], B[t * ldb + j]));
        C[i * ldc + j] = acc;
    }
}

int dcg_gemm_lr(dcg_context* ctx, cudaStream_t st, const double* A, long long lda, const double* B,
                long long ldb, double* C, long long ldc, long long m, long long kk, long long n) {
    if (m <= 0 || n <= 0) return DCG_OK;
    long long blocks = (m * n + 255) / 256;
    if (blocks > ctx->sm_count * 16LL) blocks = ctx->sm_count * 16LL;
    gemm_lr_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, lda, B, ldb, C, ldc, m, kk, n);
    DCG_LAUNCHED();
    return DCG_OK;
}
