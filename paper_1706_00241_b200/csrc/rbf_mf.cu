// Standalone matrix-free RBF products (K7, rbfmma.cuh): the operator apply
// y = shift v + s_out (.) K (s_in (.) v) and the multi-vector form
// Y = shift X_rows + s_out (.) K (s_in (.) X) used by refresh_basis
// (recycle.py:90: A W with A the Newton matrix).  Rows [row0, row0 + rows) of
// the operator (row slabs for the sharded solver); work is distributed in
// whole 64-row chunks.
#include "common.cuh"
#include "rbfmma.cuh"

namespace {

__global__ void __launch_bounds__(DCG_NT, 1)
    rbf_mma_pass1_kernel(RbfMma p, const double* v, const double* s_in, double* colpart, double* rowpart) {
    extern __shared__ __align__(16) double smem[];
    rm_init(smem, p);
    rbf_mma_pass1(p, v, s_in, colpart, rowpart, smem);
}


}  // namespace

int dcg_rbf_mf_check(const dcg_operator* op) {
    if (!op || op->kind != DCG_OP_RBF) return DCG_E_CONFIG;
    if (op->n < 0 || op->row0 < 0 || op->rows < 0 || op->row0 + op->rows > op->n) return DCG_E_CONFIG;
    if (!op->d_x || op->dim < 1) return DCG_E_CONFIG;
    if (op->dim > DCG_RBF_MAX_DIM) return DCG_E_UNSUPPORTED;
    return DCG_OK;
}


int dcg_sym_pass2_launch(cudaStream_t st, int G, int R, long long n, const double* colpart, const double* rowpart,
                         const double* v, const double* s_out, double shift, double* y);
size_t dcg_sym_apply_scratch_doubles(long long n);

// operands of the tensor-pipe pass 1 (rbfmma.cuh): fragment-major x~ and b
size_t dcg_rbf_mma_operand_doubles(long long n, int dim) {
    return (size_t)rm_npad(n) * rm_dpad(dim) + (size_t)rm_npad(n) + 2;
}

// teams per 512-thread CTA that fit next to `other_bytes` of shared memory
int dcg_rbf_mma_teams(const dcg_context* ctx, int dim, size_t other_bytes) {
    return sizeof(double) * (size_t)rm_smem_doubles(dim, 2) + other_bytes <= ctx->smem_optin ? 2 : 1;
}

RbfMma dcg_rbf_mma_params(const dcg_operator* op, double* operands, int nteam) {
    RbfMma p;
    p.X = op->d_x;
    p.n = op->n;
    p.dim = (int)op->dim;
    p.dp = rm_dpad(p.dim);
    p.xf = operands;
    p.xb = operands + rm_npad(op->n) * p.dp;
    p.var = op->var;
    p.inv2 = op->inv_two_ell2;
    p.diag = op->diag / op->var;
    p.nteam = nteam;
    p.t_lo = 0;
    p.t_hi = sym_ntiles(op->n);
    return p;
}

int dcg_rbf_mma_prep(const dcg_context* ctx, cudaStream_t st, const RbfMma& p) {
    DCG_CUDA(cudaMemsetAsync(p.xb + rm_npad(p.n), 0, sizeof(double), st));
    rbf_prep_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(p);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Row-owned tensor-pipe product Y = shift X_rows + s_out (.) K (s_in (.) X) for
// the operator's row slab (k = 0: X is a vector).  Operands in ctx->ws2.
template <int NB>
static int launch_rows(const dcg_context* ctx, cudaStream_t st, const RbfMma& p, long long row0, long long rows,
                       const double* vs, const double* s_out, double shift, const double* x_rows, double* Y, int kout,
                       const dcg_shard_state* gate) {
    const size_t smem = sizeof(double) * (size_t)rr_smem_doubles<NB>(p.dp);
    DCG_CUDA(cudaFuncSetAttribute(rbf_mma_rows_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    DCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rbf_mma_rows_kernel<NB>, RR_NT, smem));
    if (per_sm < 1) per_sm = 1;
    const long long nblk = (rows + RM_TB - 1) / RM_TB;
    long long grid = (long long)per_sm * ctx->sm_count;
    if (grid > nblk) grid = nblk;
    rbf_mma_rows_kernel<NB><<<(unsigned)grid, RR_NT, smem, st>>>(p, row0, rows, vs, s_out, shift, x_rows, Y, kout,
                                                                  gate);
    DCG_LAUNCHED();
    return DCG_OK;
}

int dcg_rbf_rows_product(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* X, int k,
                         const double* s_in, const double* s_out, double shift, double* Y,
                         const dcg_shard_state* gate) {
    const long long n = op->n, npad = rm_npad(n);
    const int kk = k ? (k + 7) / 8 * 8 : 0;
    const size_t opnd = dcg_rbf_mma_operand_doubles(n, (int)op->dim);
    const size_t vsz = (size_t)npad * (k ? kk : 1);
    int rc = dcg_ws2_reserve(ctx, sizeof(double) * (opnd + vsz) + 512);
    if (rc) return rc;
    double* operands = static_cast<double*>(ctx->ws2);
    double* vs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(operands + opnd) + 255) & ~uintptr_t(255));
    const RbfMma p = dcg_rbf_mma_params(op, operands, 1);
    rc = dcg_rbf_mma_prep(ctx, st, p);
    if (rc) return rc;
    rr_scale_kernel<<<ctx->sm_count * 4, 256, 0, st>>>(X, k, kk, s_in, op->var, n, npad, vs);
    DCG_LAUNCHED();
    const long long row0 = op->row0, rows = op->rows;
    const double* x_rows = X + row0 * (k ? k : 1);
    switch (kk / 8) {
        case 0: return launch_rows<0>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, 1, gate);
        case 1: return launch_rows<1>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 2: return launch_rows<2>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 3: return launch_rows<3>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 4: return launch_rows<4>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 5: return launch_rows<5>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 6: return launch_rows<6>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        case 7: return launch_rows<7>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
        default: return launch_rows<8>(ctx, st, p, row0, rows, vs, s_out, shift, x_rows, Y, k, gate);
    }
}

size_t dcg_rbf_mf_scratch_doubles(const dcg_operator* op) {
    return (op->row0 == 0 && op->rows == op->n)
               ? dcg_sym_apply_scratch_doubles(op->n) + dcg_rbf_mma_operand_doubles(op->n, (int)op->dim) + 32
               : 0;
}

int dcg_rbf_mf_apply(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* v, const double* s_in,
                     const double* s_out, double shift, double* y, double* scratch) {
    int rc = dcg_rbf_mf_check(op);
    if (rc) return rc;
    if (op->rows == 0) return DCG_OK;
    if (scratch && op->row0 == 0 && op->rows == op->n) {
        // unsharded: symmetric half-evaluation on the FP64 tensor pipe + the
        // stored strategy's pass 2
        const long long n = op->n;
        const int G = ctx->sm_count < DCG_SYM_MAX_CTAS ? ctx->sm_count : DCG_SYM_MAX_CTAS;
        const int nteam = dcg_rbf_mma_teams(ctx, (int)op->dim, 0);
        const size_t smem = sizeof(double) * (size_t)rm_smem_doubles((int)op->dim, nteam);
        DCG_CUDA(cudaFuncSetAttribute(rbf_mma_pass1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        double* colpart = scratch;
        double* rowpart = scratch + sym_ntiles(n) * DCG_TB;
        double* operands = reinterpret_cast<double*>(
            (reinterpret_cast<uintptr_t>(rowpart + sym_ntiles(n) * DCG_TB) + 255) & ~uintptr_t(255));
        const RbfMma p = dcg_rbf_mma_params(op, operands, nteam);
        rc = dcg_rbf_mma_prep(ctx, st, p);
        if (rc) return rc;
        rbf_mma_pass1_kernel<<<G, DCG_NT, smem, st>>>(p, v, s_in, colpart, rowpart);
        DCG_LAUNCHED();
        return dcg_sym_pass2_launch(st, G, G * nteam, n, colpart, rowpart, v, s_out, shift, y);
    }
    // row slab (sharded operator): the row-owned tensor-pipe form
    return dcg_rbf_rows_product(ctx, st, op, v, 0, s_in, s_out, shift, y, nullptr);
}

int dcg_rbf_mf_block(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* X, int k,
                     const double* s_in, const double* s_out, double shift, double* Y) {
    int rc = dcg_rbf_mf_check(op);
    if (rc) return rc;
    if (op->rows == 0 || k <= 0) return DCG_OK;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    return dcg_rbf_rows_product(ctx, st, op, X, k, s_in, s_out, shift, Y, nullptr);
}

namespace {

// A rank's share [t_lo, t_hi) of the lower-triangle tiles: pass 1 with the
// team table exported (block 0) for the local pass 2.  colpart / rowpart are
// indexed relative to t_lo.
__global__ void __launch_bounds__(DCG_NT, 1)
    rbf_mma_pass1_share_kernel(RbfMma p, const double* v, const double* s_in, double* colpart, double* rowpart,
                               long long* tbl_out, const dcg_shard_state* gate) {
    if (gate && gate->done) return;
    extern __shared__ __align__(16) double smem[];
    rm_init(smem, p);
    const int R = gridDim.x * p.nteam;
    if (blockIdx.x == 0)
        for (int b = threadIdx.x; b <= R; b += blockDim.x) tbl_out[b] = rm_table(smem)[b];
    rbf_mma_pass1(p, v, s_in, colpart - p.t_lo * RM_TB, rowpart - p.t_lo * RM_TB, smem);
}

// t_i (all n rows) from this share's partials: column partials of the tiles
// (I', I), I' > I, inside [t_lo, t_hi), and the row segments of tile row I
// that start inside it (at J = 0 or at a team range start).  Rows without
// contributions get 0.  A 256-thread CTA takes 32 consecutive rows at a time
// (lane = row: a warp's loads of one tile's partials are one 256-byte line);
// its 8 warps each sum every eighth tile of the column (sixteen loads in
// flight ahead of their in-order adds) and every eighth range start, and the
// eight sums are combined in warp order -- a fixed order, and the longest
// dependent chain is an eighth of the column (row 0 of a whole triangle at
// n = 5 10^4 has 781 partials: one thread per row took 83 us per product).
#define P2S_SUBS 8
__global__ void __launch_bounds__(32 * P2S_SUBS)
    sym_pass2_share_kernel(long long n, long long t_lo, long long t_hi, const long long* tbl, int R,
                           const double* colpart, const double* rowpart, double* t, const dcg_shard_state* gate) {
    if (gate && gate->done) return;
    __shared__ double red[P2S_SUBS][32];
    const long long NT = sym_ntiles_side(n);
    const int lane = threadIdx.x & 31, sub = threadIdx.x >> 5;
    const long long ngroups = (n + 31) / 32;
    for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const long long i = grp * 32 + lane;
        const long long I = (grp * 32) / RM_TB;          // uniform per group
        const int rl = (int)(i - I * RM_TB);             // < 64: the partial arrays hold whole tiles
        double acc = 0.0;
        // column partials: tile id base(I') + I in [t_lo, t_hi), I' > I
        long long Ip = I + 1;
        if (t_lo > I) {
            const long long need = t_lo - I;   // base(I') >= need
            long long c = sym_tile_row(need);
            if (sym_tile_row_base(c) < need) ++c;
            if (c > Ip) Ip = c;
        }
        Ip += sub;
        long long id = sym_tile_row_base(Ip) + I;
        while (Ip < NT && id < t_hi) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                v[u] = 0.0;
                if (Ip + P2S_SUBS * u < NT && id < t_hi) {
                    v[u] = ld_cg(colpart + (id - t_lo) * RM_TB + rl);
                    // base(r + 8) - base(r) = 8 r + 36
                    id += P2S_SUBS * (Ip + P2S_SUBS * u) + P2S_SUBS * (P2S_SUBS + 1) / 2;
                }
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc += v[u];
            Ip += 16 * P2S_SUBS;
        }
        // row segments of tile row I
        const long long base = sym_tile_row_base(I);
        if (sub == 0 && base >= t_lo && base < t_hi) acc += ld_cg(rowpart + (base - t_lo) * RM_TB + rl);
        for (int b = sub; b < R; b += P2S_SUBS) {   // team range starts inside the row (tbl[0] = t_lo may be one)
            const long long st = tbl[b];
            if (st > base && st <= base + I && st < t_hi && (b == 0 || st > tbl[b - 1]))
                acc += ld_cg(rowpart + (st - t_lo) * RM_TB + rl);
        }
        red[sub][lane] = acc;
        __syncthreads();
        if (sub == 0 && i < n) {
            double a = red[0][lane];
#pragma unroll
            for (int q = 1; q < P2S_SUBS; ++q) a += red[q][lane];
            t[i] = a;
        }
        __syncthreads();
    }
}

// Stored tile share: pass 1 of the packed-tile GEMV over the rank's tiles
// [t_lo, t_hi) (kp_share holds exactly those, tile t at t - t_lo), split over
// the CTAs with the same equal-cost rule, the range table exported (block 0)
// for the share's pass 2.  colpart / rowpart are indexed relative to t_lo.
// NV = 2: a second vector v2 (both unscaled, s_in unused) with its partials
// at colpart / rowpart + part2.
template <int NV>
__global__ void __launch_bounds__(DCG_NT, 1)
    stored_pass1_share_kernel(const double* kp_share, long long n, long long t_lo, long long t_hi, const double* v,
                              const double* s_in, double* colpart, double* rowpart, long long* tbl_out,
                              const dcg_shard_state* gate, const double* v2 = nullptr, long long part2 = 0) {
    if (gate && gate->done) return;
    extern __shared__ __align__(16) double smem[];
    sym_ring_init(smem, n, true);
    long long* tbl = sym_range_table(smem);
    const int G = gridDim.x;
    for (int b = threadIdx.x; b <= G; b += blockDim.x) tbl[b] = sym_tile_begin_range(n, t_lo, t_hi, G, b);
    cta_sync();
    if (blockIdx.x == 0)
        for (int b = threadIdx.x; b <= G; b += blockDim.x) tbl_out[b] = tbl[b];
    unsigned int seq = 0;
    sym_pass1<true, NV, true>(kp_share - t_lo * DCG_SYM_TILE_DOUBLES, 0, n, v, NV == 2 ? nullptr : s_in,
                              colpart - t_lo * DCG_TB, rowpart - t_lo * DCG_TB, smem, seq, v2, part2);
}

}  // namespace

// Sharded stored K (s (.) v) over a tile share: op->kind DCG_OP_DENSE_SYM,
// op->d_kp = this rank's packed tiles [t_lo, t_hi) (dcg_shard_tile_range:
// the same equal-cost split as the matrix-free share), op->d_s the full
// scale vector.  Writes the rank's partial t (all n rows) to d_t; the sum over
// ranks (one all-reduce of n doubles) is K (s (.) v).
extern "C" int dcg_shard_tiles_partial(dcg_context* ctx, void* stream, const dcg_operator* op, int rank, int world,
                                       const double* d_v, double* d_t, const dcg_shard_state* d_state) {
    if (!ctx || !op || !d_v || !d_t || world < 1 || rank < 0 || rank >= world) return DCG_E_CONFIG;
    if (op->kind != DCG_OP_DENSE_SYM || !op->d_kp || !aligned16(op->d_kp) || !aligned16(d_v) ||
        !aligned16(op->d_s))
        return DCG_E_CONFIG;
    const long long n = op->n;
    if (n == 0) return DCG_OK;
    cudaStream_t st = as_stream(stream);
    const long long t_lo = sym_tile_begin(n, world, rank), t_hi = sym_tile_begin(n, world, rank + 1);
    const long long nloc = t_hi - t_lo;
    const int G = ctx->sm_count < DCG_SYM_MAX_CTAS ? ctx->sm_count : DCG_SYM_MAX_CTAS;
    const size_t need = sizeof(double) * 2 * (size_t)(nloc > 0 ? nloc : 1) * DCG_TB +
                        sizeof(long long) * (DCG_SYM_MAX_CTAS + 2) + 1024;
    int rc = dcg_ws2_reserve(ctx, need);
    if (rc) return rc;
    double* colpart = static_cast<double*>(ctx->ws2);
    double* rowpart = colpart + (nloc > 0 ? nloc : 1) * DCG_TB;
    long long* tbl = reinterpret_cast<long long*>(rowpart + (nloc > 0 ? nloc : 1) * DCG_TB);
    if (nloc > 0) {
        const size_t smem = sizeof(double) * (size_t)sym_smem_doubles();
        DCG_SMEM_ATTR(stored_pass1_share_kernel<1>, smem);
        stored_pass1_share_kernel<1><<<G, DCG_NT, smem, st>>>(op->d_kp, n, t_lo, t_hi, d_v, op->d_s, colpart, rowpart,
                                                               tbl, d_state);
        DCG_LAUNCHED();
    }
    sym_pass2_share_kernel<<<ctx->sm_count * 4, 32 * P2S_SUBS, 0, st>>>(n, t_lo, t_hi, tbl, G, colpart, rowpart, d_t, d_state);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Two products over one pass of the rank's tile share: partials of K v1 and
// K v2 (both unscaled; op->d_s is not applied) for all n rows into d_t1, d_t2
// (the Newton system's K inner and the next solve's K (s (.) x_prev)).
extern "C" int dcg_shard_tiles_partial2(dcg_context* ctx, void* stream, const dcg_operator* op, int rank, int world,
                                        const double* d_v1, const double* d_v2, double* d_t1, double* d_t2) {
    if (!ctx || !op || !d_v1 || !d_v2 || !d_t1 || !d_t2 || world < 1 || rank < 0 || rank >= world) return DCG_E_CONFIG;
    if (op->kind != DCG_OP_DENSE_SYM || !op->d_kp || !aligned16(op->d_kp) || !aligned16(d_v1) || !aligned16(d_v2))
        return DCG_E_CONFIG;
    const long long n = op->n;
    if (n == 0) return DCG_OK;
    cudaStream_t st = as_stream(stream);
    const long long t_lo = sym_tile_begin(n, world, rank), t_hi = sym_tile_begin(n, world, rank + 1);
    const long long nloc = t_hi - t_lo, nl = nloc > 0 ? nloc : 1;
    const int G = ctx->sm_count < DCG_SYM_MAX_CTAS ? ctx->sm_count : DCG_SYM_MAX_CTAS;
    const size_t need = sizeof(double) * 4 * (size_t)nl * DCG_TB + sizeof(long long) * (DCG_SYM_MAX_CTAS + 2) + 1024;
    int rc = dcg_ws2_reserve(ctx, need);
    if (rc) return rc;
    double* colpart = static_cast<double*>(ctx->ws2);
    double* rowpart = colpart + nl * DCG_TB;
    const long long part2 = 2 * nl * DCG_TB;
    long long* tbl = reinterpret_cast<long long*>(colpart + 4 * nl * DCG_TB);
    if (nloc > 0) {
        const size_t smem = sizeof(double) * (size_t)sym_smem_doubles();
        DCG_SMEM_ATTR(stored_pass1_share_kernel<2>, smem);
        stored_pass1_share_kernel<2><<<G, DCG_NT, smem, st>>>(op->d_kp, n, t_lo, t_hi, d_v1, nullptr, colpart,
                                                               rowpart, tbl, nullptr, d_v2, part2);
        DCG_LAUNCHED();
    }
    sym_pass2_share_kernel<<<ctx->sm_count * 4, 32 * P2S_SUBS, 0, st>>>(n, t_lo, t_hi, tbl, G, colpart, rowpart, d_t1, nullptr);
    DCG_LAUNCHED();
    sym_pass2_share_kernel<<<ctx->sm_count * 4, 32 * P2S_SUBS, 0, st>>>(n, t_lo, t_hi, tbl, G, colpart + part2,
                                                              rowpart + part2, d_t2, nullptr);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Sharded matrix-free K (s (.) v), symmetric form: rank `rank` of `world`
// evaluates an equal-cost share of the lower-triangle tiles (each pair once,
// as in the unsharded operator) and writes its partial t (all n rows) to d_t;
// the sum over ranks (an all-reduce) is K (s (.) v).  Half the pairs of the
// row-slab form; the exchange is one n-vector all-reduce per product.
extern "C" int dcg_shard_rbf_sym_partial(dcg_context* ctx, void* stream, const dcg_operator* op, int rank, int world,
                                         const double* d_v, double* d_t, const dcg_shard_state* d_state) {
    if (!ctx || !d_v || !d_t || world < 1 || rank < 0 || rank >= world) return DCG_E_CONFIG;
    int rc = dcg_rbf_mf_check(op);
    if (rc) return rc;
    const long long n = op->n;
    if (n == 0) return DCG_OK;
    cudaStream_t st = as_stream(stream);
    const long long ntt = sym_ntiles(n);
    const long long t_lo = sym_tile_begin(n, world, rank), t_hi = sym_tile_begin(n, world, rank + 1);
    const long long nloc = t_hi - t_lo;
    const int G = ctx->sm_count < DCG_SYM_MAX_CTAS ? ctx->sm_count : DCG_SYM_MAX_CTAS;
    const int nteam = dcg_rbf_mma_teams(ctx, (int)op->dim, 0);
    const size_t opnd = dcg_rbf_mma_operand_doubles(n, (int)op->dim);
    const size_t need = sizeof(double) * (opnd + 2 * (size_t)(nloc > 0 ? nloc : 1) * RM_TB) +
                        sizeof(long long) * (2 * DCG_SYM_MAX_CTAS + 2) + 1024;
    rc = dcg_ws2_reserve(ctx, need);
    if (rc) return rc;
    double* operands = static_cast<double*>(ctx->ws2);
    double* colpart = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(operands + opnd) + 255) & ~uintptr_t(255));
    double* rowpart = colpart + (nloc > 0 ? nloc : 1) * RM_TB;
    long long* tbl = reinterpret_cast<long long*>(rowpart + (nloc > 0 ? nloc : 1) * RM_TB);
    RbfMma p = dcg_rbf_mma_params(op, operands, nteam);
    p.t_lo = t_lo;
    p.t_hi = t_hi;
    (void)ntt;
    rc = dcg_rbf_mma_prep(ctx, st, p);
    if (rc) return rc;
    const size_t smem = sizeof(double) * (size_t)rm_smem_doubles((int)op->dim, nteam);
    DCG_CUDA(cudaFuncSetAttribute(rbf_mma_pass1_share_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rbf_mma_pass1_share_kernel<<<G, DCG_NT, smem, st>>>(p, d_v, op->d_s, colpart, rowpart, tbl, d_state);
    DCG_LAUNCHED();
    sym_pass2_share_kernel<<<ctx->sm_count * 4, 32 * P2S_SUBS, 0, st>>>(n, t_lo, t_hi, tbl, G * nteam, colpart, rowpart, d_t,
                                                              d_state);
    DCG_LAUNCHED();
    return DCG_OK;
}

