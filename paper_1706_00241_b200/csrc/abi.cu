#include <stddef.h>
// C ABI entry points (include/defcg_b200.h): context, workspace, the L0
// kernel twins, operator application, basis refresh / Gram factorisation,
// harmonic-Ritz extraction, eigensolvers and the GPC glue.  Each entry point
// mirrors one reference function (cited per function) and maps its failure
// modes to the status codes of errors.py.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "symgemv.cuh"

#include <atomic>

thread_local cudaError_t dcg_last_cuda_error = cudaSuccess;
static std::atomic<long long> g_launches{0};

std::mutex& dcg_setup_mutex() {
    static std::mutex m;
    return m;
}

void dcg_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" long long dcg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// launchers implemented in the other translation units
int dcg_gemv_launch(dcg_context*, cudaStream_t, const double*, long long, long long, long long, const double*,
                    const double*, const double*, double, const double*, double*);
size_t dcg_sym_apply_scratch_doubles(long long n);
size_t dcg_sym_apply2_scratch_doubles(long long n);
int dcg_sym_apply2(dcg_context*, cudaStream_t, const double*, const double*, long long, long long, const double*,
                   const double*,
                   const double*, const double*, const double*, const double*, double, double, double*, double*,
                   double*);
int dcg_newton_prep2_launch(dcg_context*, cudaStream_t, long long, const double*, const double*, const double*,
                            const double*, double*, double*, double*);
int dcg_sym_apply(dcg_context*, cudaStream_t, const double*, const double*, long long, long long, const double*,
                  const double*, const double*, double, double*, double*);
size_t dcg_block_apply_scratch_doubles(long long n, long long rows, int k);
int dcg_block_apply(dcg_context*, cudaStream_t, const double*, long long, long long, long long, const double*, int,
                    const double*, const double*, double, const double*, double*, double*);
int dcg_xty(dcg_context*, cudaStream_t, const double*, long long, const double*, long long, long long, int, int,
            double*, double*);
size_t dcg_sym_block_scratch_doubles(long long n, int k);
bool dcg_sym_block_ok(int k);
int dcg_sym_block_apply(dcg_context*, cudaStream_t, const double*, long long, const double*, int, const double*,
                        const double*, double, double*, double*);

// The refresh's block product A W over the operator's storage: the packed
// lower-triangle tiles with the symmetric DMMA product (symblock.cu, half the
// bytes; k padded to 16 or 32 columns) when the operator has them and
// k <= 16 or 24 < k <= 32, else the row-major DMMA GEMM (for 16 < k <= 24 the
// padding to 32 columns costs what the halved bytes save: 1.95 vs 1.89 ms at
// n = 3e4, k = 24; at k = 32, n = 5e4: 5.35 vs 7.46 ms).
// DCG_NO_SYMBLOCK (developer A/B knob) forces the row-major product.
static bool use_sym_block(const dcg_operator* op, int k) {
    static const bool off = getenv("DCG_NO_SYMBLOCK") != nullptr;
    return !off && op->kind == DCG_OP_DENSE_SYM && op->d_kp && op->row0 == 0 && op->rows == op->n &&
           dcg_sym_block_ok(k) && (k <= 16 || k > 24);
}
extern "C" int dcg_block_uses_packed(int k) {
    static const bool off = getenv("DCG_NO_SYMBLOCK") != nullptr;
    return !off && dcg_sym_block_ok(k) && (k <= 16 || k > 24);
}
static size_t block_scratch_doubles(const dcg_operator* op, int k) {
    return use_sym_block(op, k) ? dcg_sym_block_scratch_doubles(op->n, k)
                                : dcg_block_apply_scratch_doubles(op->n, op->rows, k);
}
static int block_apply_op(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* X, int k,
                          const double* s_in, const double* s_out, double shift, const double* X_rows, double* Y,
                          double* scratch) {
    if (use_sym_block(op, k))
        return dcg_sym_block_apply(ctx, st, op->d_kp, op->n, X, k, s_in, s_out, shift, Y, scratch);
    if (!op->d_k) return DCG_E_CONFIG;   // a packed-only operator without its row-major storage
    return dcg_block_apply(ctx, st, op->d_k, op->ldk, op->rows, op->n, X, k, s_in, s_out, shift, X_rows, Y, scratch);
}
size_t dcg_xty_scratch_doubles(dcg_context* ctx, int p, int q);
int dcg_gemm_lr(dcg_context*, cudaStream_t, const double*, long long, const double*, long long, double*, long long,
                long long, long long, long long);
int dcg_gram_factor_launch(cudaStream_t, const double*, int, int, double*, double*, int*, DevStatus*);
size_t dcg_pencil_smem(int T);
int dcg_ritz_pencil_launch(cudaStream_t, const double*, const double*, int, int, int, int, double*, double*,
                           double*, int*, DevStatus*, const DevStatus*);
int dcg_sym_eigen_launch(cudaStream_t, const double*, int, int, double, double*, double*, DevStatus*);
int dcg_gen_sym_eigen_launch(cudaStream_t, const double*, const double*, int, int, double*, double*, double*,
                             DevStatus*);
int dcg_k_cholesky_launch(cudaStream_t, const double*, int, double, double*, DevStatus*);
int dcg_k_solve_lower_launch(cudaStream_t, const double*, int, const double*, double*);
int dcg_k_solve_lower_trans_launch(cudaStream_t, const double*, int, const double*, double*);
int dcg_k_jacobi_sweep_launch(cudaStream_t, double*, double*, int, DevStatus*);
int dcg_rbf_launch(cudaStream_t, const double*, long long, const double*, long long, long long, double, double,
                   double, int, long long, long long, double*, long long);
int dcg_derivs_launch(dcg_context*, cudaStream_t, long long, const double*, const double*, const double*, double*,
                      double*, double*, DevStatus*, double* llpsi = nullptr);
int dcg_newton_prep_launch(dcg_context*, cudaStream_t, long long, const double*, const double*, const double*,
                           double*, double*);
int dcg_newton_a_launch(dcg_context*, cudaStream_t, long long, const double*, const double*, const double*,
                        double*);

// ---------------------------------------------------------------------------
// context and workspace
// ---------------------------------------------------------------------------
extern "C" int dcg_version(void) { return DCG_ABI_VERSION; }

extern "C" const char* dcg_status_string(int status) {
    switch (status) {
        case DCG_OK: return "ok";
        case DCG_E_DIMENSION: return "dimension mismatch";
        case DCG_E_NOT_PD: return "non-positive pivot (not positive definite)";
        case DCG_E_BREAKDOWN: return "non-positive curvature p'Ap <= 0";
        case DCG_E_GRAM_NOT_SPD: return "W'AW not SPD";
        case DCG_E_BASIS_DEFICIENT: return "basis deficient";
        case DCG_E_NO_CONVERGENCE: return "Jacobi eigensolver did not converge";
        case DCG_E_ASYMMETRIC: return "matrix is not symmetric within tolerance";
        case DCG_E_CONFIG: return "invalid argument";
        case DCG_E_CUDA: return dcg_last_cuda_error != cudaSuccess ? cudaGetErrorString(dcg_last_cuda_error)
                                                                    : "CUDA error";
        case DCG_E_UNSUPPORTED: return "size outside compiled limits";
        default: return "unknown status";
    }
}

extern "C" int dcg_context_create(int device, dcg_context** out) {
    if (!out) return DCG_E_CONFIG;
    *out = nullptr;
    DCG_CUDA(cudaSetDevice(device));
    dcg_context* c = new dcg_context();
    memset(c, 0, sizeof(*c));
    c->device = device;
    cudaDeviceProp prop;
    DCG_CUDA(cudaGetDeviceProperties(&prop, device));
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    c->solve_blocks = prop.multiProcessorCount;   // one persistent CTA per SM
    DCG_CUDA(cudaEventCreate(&c->ev0));
    DCG_CUDA(cudaEventCreate(&c->ev1));
    DCG_CUDA(cudaMalloc(&c->d_sync, 128 * DCG_SW_NSLOTS));
    DCG_CUDA(cudaMemset(c->d_sync, 0, 128 * DCG_SW_NSLOTS));
    *out = c;
    return DCG_OK;
}

const long long* dcg_sym_table(dcg_context* ctx, cudaStream_t st, long long n, int G) {
    for (auto& e : ctx->symtbl)
        if (e.d && e.n == n && e.G == G) return e.d;
    auto& e = ctx->symtbl[ctx->symtbl_next];
    ctx->symtbl_next = (ctx->symtbl_next + 1) % 4;
    if (!e.d) {
        if (cudaMalloc(&e.d, sizeof(long long) * (DCG_SYM_MAX_CTAS + 2)) != cudaSuccess) return nullptr;
        if (cudaHostAlloc(&e.h, sizeof(long long) * (DCG_SYM_MAX_CTAS + 2), cudaHostAllocDefault) != cudaSuccess)
            return nullptr;
    } else {
        cudaStreamSynchronize(st);   // the staging copy of the entry being replaced may still be in flight
    }
    for (int b = 0; b <= G; ++b) e.h[b] = sym_tile_begin(n, G, b);
    if (cudaMemcpyAsync(e.d, e.h, sizeof(long long) * (G + 1), cudaMemcpyHostToDevice, st) != cudaSuccess)
        return nullptr;
    e.n = n;
    e.G = G;
    return e.d;
}

extern "C" int dcg_context_destroy(dcg_context* ctx) {
    if (!ctx) return DCG_OK;
    cudaDeviceSynchronize();
    for (auto& e : ctx->symtbl) {
        if (e.d) cudaFree(e.d);
        if (e.h) cudaFreeHost(e.h);
    }
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->ws2) cudaFree(ctx->ws2);
    if (ctx->host) cudaFreeHost(ctx->host);
    if (ctx->d_res) cudaFree(ctx->d_res);
    if (ctx->d_sync) cudaFree(ctx->d_sync);
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    delete ctx;
    return DCG_OK;
}

extern "C" int dcg_context_grid(dcg_context* ctx, int* blocks, int* sm_count) {
    if (!ctx) return DCG_E_CONFIG;
    if (blocks) *blocks = ctx->solve_blocks;
    if (sm_count) *sm_count = ctx->sm_count;
    return DCG_OK;
}

int dcg_ws_reserve(dcg_context* ctx, size_t bytes) {
    if (bytes <= ctx->ws_bytes) return DCG_OK;
    if (ctx->ws) {
        cudaDeviceSynchronize();   // outstanding work may still use the old buffer
        cudaFree(ctx->ws);
        ctx->ws = nullptr;
        ctx->ws_bytes = 0;
    }
    size_t want = bytes + bytes / 4 + (1 << 20);
    DCG_CUDA(cudaMalloc(&ctx->ws, want));
    ctx->ws_bytes = want;
    return DCG_OK;
}

int dcg_ws2_reserve(dcg_context* ctx, size_t bytes) {
    if (bytes <= ctx->ws2_bytes) return DCG_OK;
    if (ctx->ws2) {
        cudaDeviceSynchronize();
        cudaFree(ctx->ws2);
        ctx->ws2 = nullptr;
        ctx->ws2_bytes = 0;
    }
    size_t want = bytes + bytes / 4 + (1 << 20);
    DCG_CUDA(cudaMalloc(&ctx->ws2, want));
    ctx->ws2_bytes = want;
    return DCG_OK;
}

int dcg_host_reserve(dcg_context* ctx, size_t bytes) {
    if (bytes <= ctx->host_bytes) return DCG_OK;
    if (ctx->host) cudaFreeHost(ctx->host);
    if (ctx->d_res) cudaFree(ctx->d_res);
    ctx->host = nullptr;
    DCG_CUDA(cudaMallocHost(&ctx->host, bytes + 4096));
    ctx->host_bytes = bytes + 4096;
    return DCG_OK;
}

int dcg_read_status(dcg_context* ctx, cudaStream_t st, const DevStatus* dev, DevStatus* out) {
    int rc = dcg_host_reserve(ctx, sizeof(DevStatus));
    if (rc) return rc;
    DevStatus* hs = static_cast<DevStatus*>(ctx->host);
    DCG_CUDA(cudaMemcpyAsync(hs, dev, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    DCG_CUDA(cudaStreamSynchronize(st));
    *out = *hs;
    return DCG_OK;
}


// ---------------------------------------------------------------------------
// L0 twins
// ---------------------------------------------------------------------------
extern "C" int dcg_k_matvec(dcg_context* ctx, void* stream, const double* d_a, long long m, long long n,
                            long long lda, const double* d_x, double* d_y) {
    if (!ctx || m < 0 || n < 0 || lda < n) return DCG_E_CONFIG;
    if (m == 0) return DCG_OK;
    if ((lda & 1) || !aligned16(d_a)) return DCG_E_CONFIG;
    return dcg_gemv_launch(ctx, as_stream(stream), d_a, lda, n, m, d_x, nullptr, nullptr, 0.0, nullptr, d_y);
}

extern "C" int dcg_k_gemm(dcg_context* ctx, void* stream, const double* d_a, const double* d_b, double* d_c,
                          long long m, long long kk, long long n) {
    if (!ctx || m < 0 || kk < 0 || n < 0) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    if (kk == 0 && m * n > 0) {
        DCG_CUDA(cudaMemsetAsync(d_c, 0, sizeof(double) * m * n, st));
        return DCG_OK;
    }
    return dcg_gemm_lr(ctx, st, d_a, kk, d_b, n, d_c, n, m, kk, n);
}

extern "C" int dcg_k_cholesky(dcg_context* ctx, void* stream, const double* d_a, long long n, double pivot_tol,
                              double* d_l, long long* fail_index) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        if (fail_index) *fail_index = -1;
        return DCG_OK;
    }
    int rc = dcg_ws_reserve(ctx, sizeof(DevStatus));
    if (rc) return rc;
    DevStatus* ds = static_cast<DevStatus*>(ctx->ws);
    rc = dcg_k_cholesky_launch(st, d_a, (int)n, pivot_tol, d_l, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (fail_index) *fail_index = hs.info;
    return DCG_OK;
}

extern "C" int dcg_k_solve_lower(dcg_context* ctx, void* stream, const double* d_l, long long n, const double* d_b,
                                 double* d_y) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    if (n == 0) return DCG_OK;
    return dcg_k_solve_lower_launch(as_stream(stream), d_l, (int)n, d_b, d_y);
}

extern "C" int dcg_k_solve_lower_trans(dcg_context* ctx, void* stream, const double* d_l, long long n,
                                       const double* d_b, double* d_x) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    if (n == 0) return DCG_OK;
    return dcg_k_solve_lower_trans_launch(as_stream(stream), d_l, (int)n, d_b, d_x);
}

extern "C" int dcg_k_rbf_gram(dcg_context* ctx, void* stream, const double* d_x, long long n, long long dim,
                              double signal_var, double inv_two_ell2, double jitter, double* d_k, long long ldk,
                              long long row0, long long rows) {
    if (!ctx || n < 0 || dim < 0 || ldk < n || row0 < 0 || rows < 0 || row0 + rows > n) return DCG_E_CONFIG;
    return dcg_rbf_launch(as_stream(stream), d_x, n, d_x, n, dim, signal_var, inv_two_ell2, jitter, 1, row0, rows,
                          d_k, ldk);
}

int dcg_rbf_packed_launch(cudaStream_t, const double*, long long, long long, double, double, double, long long,
                          long long, double*);

extern "C" int dcg_shard_tile_range(long long n, int rank, int world, long long* t_lo, long long* t_hi) {
    if (n < 0 || world < 1 || rank < 0 || rank >= world || !t_lo || !t_hi) return DCG_E_CONFIG;
    *t_lo = n ? sym_tile_begin(n, world, rank) : 0;
    *t_hi = n ? sym_tile_begin(n, world, rank + 1) : 0;
    return DCG_OK;
}

extern "C" int dcg_k_rbf_gram_packed(dcg_context* ctx, void* stream, const double* d_x, long long n, long long dim,
                                     double signal_var, double inv_two_ell2, double jitter, long long t_lo,
                                     long long t_hi, double* d_kp) {
    if (!ctx || n < 0 || dim < 0 || t_lo < 0 || t_hi < t_lo || t_hi > sym_ntiles(n) || !aligned16(d_kp))
        return DCG_E_CONFIG;
    return dcg_rbf_packed_launch(as_stream(stream), d_x, n, dim, signal_var, inv_two_ell2, jitter, t_lo, t_hi, d_kp);
}

extern "C" int dcg_k_rbf_cross(dcg_context* ctx, void* stream, const double* d_xa, long long na, const double* d_xb,
                               long long nb, long long dim, double signal_var, double inv_two_ell2, double* d_k) {
    if (!ctx || na < 0 || nb < 0 || dim < 0) return DCG_E_CONFIG;
    return dcg_rbf_launch(as_stream(stream), d_xa, na, d_xb, nb, dim, signal_var, inv_two_ell2, 0.0, 0, 0, na, d_k,
                          nb);
}

extern "C" int dcg_k_jacobi_sweep(dcg_context* ctx, void* stream, double* d_a, double* d_v, long long n,
                                  long long* rotations) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        if (rotations) *rotations = 0;
        return DCG_OK;
    }
    int rc = dcg_ws_reserve(ctx, sizeof(DevStatus));
    if (rc) return rc;
    DevStatus* ds = static_cast<DevStatus*>(ctx->ws);
    rc = dcg_k_jacobi_sweep_launch(st, d_a, d_v, (int)n, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (rotations) *rotations = hs.count;
    return DCG_OK;
}

// ---------------------------------------------------------------------------
// L1: symmetry check and eigensolvers
// ---------------------------------------------------------------------------
#define SYM_T 32
__global__ void symcheck_kernel(const double* a, long long n, long long lda, unsigned long long* maxes) {
    __shared__ double t1[SYM_T][SYM_T + 1];
    __shared__ double t2[SYM_T][SYM_T + 1];
    const long long I = blockIdx.y, J = blockIdx.x;
    if (J < I) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int r = ty; r < SYM_T; r += 8) {
        const long long i1 = I * SYM_T + r, j1 = J * SYM_T + tx;
        t1[r][tx] = (i1 < n && j1 < n) ? a[i1 * lda + j1] : 0.0;
        const long long i2 = J * SYM_T + r, j2 = I * SYM_T + tx;
        t2[r][tx] = (i2 < n && j2 < n) ? a[i2 * lda + j2] : 0.0;
    }
    cta_sync();
    double dmax = 0.0, amax = 0.0;
    for (int r = ty; r < SYM_T; r += 8) {
        const double v = t1[r][tx];
        const double d = fabs(v - t2[tx][r]);
        dmax = (d > dmax || d != d) ? d : dmax;
        const double av = fabs(v), aw = fabs(t2[r][tx]);
        amax = (av > amax || av != av) ? av : amax;
        amax = (aw > amax || aw != aw) ? aw : amax;
    }
    // non-negative doubles (and NaN) order like their bit patterns
    atomicMax(&maxes[0], (unsigned long long)__double_as_longlong(dmax));
    atomicMax(&maxes[1], (unsigned long long)__double_as_longlong(amax));
}

extern "C" int dcg_check_symmetric(dcg_context* ctx, void* stream, const double* d_a, long long n, long long lda,
                                   double rtol, int* symmetric) {
    if (!ctx || !symmetric || n < 0 || lda < n) return DCG_E_CONFIG;
    *symmetric = 1;
    if (n == 0) return DCG_OK;
    cudaStream_t st = as_stream(stream);
    int rc = dcg_ws_reserve(ctx, 64);
    if (rc) return rc;
    unsigned long long* mx = static_cast<unsigned long long*>(ctx->ws);
    DCG_CUDA(cudaMemsetAsync(mx, 0, 16, st));
    const long long tiles = (n + SYM_T - 1) / SYM_T;
    symcheck_kernel<<<dim3((unsigned)tiles, (unsigned)tiles), 256, 0, st>>>(d_a, n, lda, mx);
    DCG_LAUNCHED();
    rc = dcg_host_reserve(ctx, 16);
    if (rc) return rc;
    unsigned long long* h = static_cast<unsigned long long*>(ctx->host);
    DCG_CUDA(cudaMemcpyAsync(h, mx, 16, cudaMemcpyDeviceToHost, st));
    DCG_CUDA(cudaStreamSynchronize(st));
    double dmax, amax;
    memcpy(&dmax, &h[0], 8);
    memcpy(&amax, &h[1], 8);
    const double scale = amax > 1e-300 ? amax : 1e-300;   // max(scale, 1e-300), linalg.py:53
    *symmetric = (dmax > rtol * scale) ? 0 : 1;
    return DCG_OK;
}

extern "C" int dcg_sym_eigen(dcg_context* ctx, void* stream, const double* d_a, long long n, long long max_sweeps,
                             double rtol, double* d_values, double* d_vectors, long long* info) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    if (info) *info = 0;
    if (n == 0) return DCG_OK;
    if (n > DCG_MAX_T) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    int rc = dcg_ws_reserve(ctx, 256);
    if (rc) return rc;
    DevStatus* ds = static_cast<DevStatus*>(ctx->ws);
    DCG_CUDA(cudaMemsetAsync(ds, 0, sizeof(DevStatus), st));
    rc = dcg_sym_eigen_launch(st, d_a, (int)n, (int)max_sweeps, rtol, d_values, d_vectors, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (hs.status != DCG_OK && info) *info = hs.info;
    return hs.status;
}

extern "C" int dcg_gen_sym_eigen(dcg_context* ctx, void* stream, const double* d_g, const double* d_f, long long n,
                                 long long max_sweeps, double* d_values, double* d_vectors, long long* info) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    if (info) *info = 0;
    if (n == 0) return DCG_OK;
    if (n > DCG_MAX_T) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    int rc = dcg_ws_reserve(ctx, al(sizeof(DevStatus)) + al(sizeof(double) * 2 * n * n));
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    DevStatus* ds = ar.take<DevStatus>(1);
    double* wk = ar.take<double>(2 * n * n);
    DCG_CUDA(cudaMemsetAsync(ds, 0, sizeof(DevStatus), st));
    rc = dcg_gen_sym_eigen_launch(st, d_g, d_f, (int)n, (int)max_sweeps, wk, d_values, d_vectors, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (hs.status != DCG_OK && info) *info = hs.info;
    return hs.status;
}

// ---------------------------------------------------------------------------
// L2: operator application
// ---------------------------------------------------------------------------
int dcg_rbf_mf_check(const dcg_operator* op);
int dcg_rbf_mf_apply(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* v, const double* s_in,
                     const double* s_out, double shift, double* y, double* scratch);
size_t dcg_rbf_mf_scratch_doubles(const dcg_operator* op);
int dcg_rbf_mf_block(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* X, int k,
                     const double* s_in, const double* s_out, double shift, double* Y);

static int check_dense_op(const dcg_operator* op) {
    if (!op) return DCG_E_CONFIG;
    if (op->kind == DCG_OP_RBF) return dcg_rbf_mf_check(op);
    if (op->kind != DCG_OP_DENSE && op->kind != DCG_OP_DENSE_SYM) return DCG_E_UNSUPPORTED;
    if (op->n < 0 || op->row0 < 0 || op->rows < 0 || op->row0 + op->rows > op->n) return DCG_E_CONFIG;
    if (op->ldk < op->n || (op->ldk & 1) || !aligned16(op->d_k)) return DCG_E_CONFIG;
    if (op->kind == DCG_OP_DENSE_SYM && (op->row0 != 0 || op->rows != op->n)) return DCG_E_CONFIG;
    return DCG_OK;
}

// y = shift v + s_out (.) K (s_in (.) v) over the operator's storage strategy;
// `scratch` holds apply_k_scratch(op) doubles (workspace reserved by the caller).
static size_t apply_k_scratch(const dcg_operator* op) {
    if (op->kind == DCG_OP_RBF) return dcg_rbf_mf_scratch_doubles(op);
    return op->kind == DCG_OP_DENSE_SYM ? dcg_sym_apply_scratch_doubles(op->n) : 0;
}
static int apply_k(dcg_context* ctx, cudaStream_t st, const dcg_operator* op, const double* v, const double* s_in,
                   const double* s_out, double shift, double* y, double* scratch) {
    if (op->kind == DCG_OP_RBF) return dcg_rbf_mf_apply(ctx, st, op, v, s_in, s_out, shift, y, scratch);
    // the lower-triangle strategy stages 16-byte slices of v and s_in
    if (op->kind == DCG_OP_DENSE_SYM && aligned16(v) && aligned16(s_in))
        return dcg_sym_apply(ctx, st, op->d_k, op->d_kp, op->ldk, op->n, v, s_in, s_out, shift, y, scratch);
    if (!op->d_k) return DCG_E_CONFIG;
    return dcg_gemv_launch(ctx, st, op->d_k, op->ldk, op->n, op->rows, v, s_in, s_out, shift, v + op->row0, y);
}

extern "C" int dcg_op_apply(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_x,
                            double* d_y) {
    if (!ctx) return DCG_E_CONFIG;
    int rc = check_dense_op(op);
    if (rc) return rc;
    const double* s_out = op->d_s ? op->d_s + op->row0 : nullptr;
    rc = dcg_ws_reserve(ctx, sizeof(double) * apply_k_scratch(op) + 256);
    if (rc) return rc;
    return apply_k(ctx, as_stream(stream), op, d_x, op->d_s, s_out, op->shift, d_y, static_cast<double*>(ctx->ws));
}

extern "C" int dcg_op_apply_block(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_x,
                                  long long k, double* d_y) {
    if (!ctx || k < 0) return DCG_E_CONFIG;
    int rc = check_dense_op(op);
    if (rc) return rc;
    if (k == 0) return DCG_OK;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    if (op->kind == DCG_OP_RBF)
        return dcg_rbf_mf_block(ctx, as_stream(stream), op, d_x, (int)k, op->d_s,
                                op->d_s ? op->d_s + op->row0 : nullptr, op->shift, d_y);
    rc = dcg_ws_reserve(ctx, sizeof(double) * block_scratch_doubles(op, (int)k) + 256);
    if (rc) return rc;
    const double* s_out = op->d_s ? op->d_s + op->row0 : nullptr;
    return block_apply_op(ctx, as_stream(stream), op, d_x, (int)k, op->d_s, s_out, op->shift, d_x + op->row0 * k, d_y,
                          static_cast<double*>(ctx->ws));
}

// ---------------------------------------------------------------------------
// Gram factor / basis refresh
// ---------------------------------------------------------------------------
__global__ void gather_cols_kernel(const double* src, long long n, int k, const int* cols, int kk, double* dst) {
    const long long total = n * kk;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / kk;
        const int c = (int)(e % kk);
        dst[e] = src[i * k + cols[c]];
    }
}

// Gram = W'AW -> (sym) -> Cholesky [-> prune].  Writes L (k_out x k_out) and
// the surviving column list (device ints) and returns k_out via *k_out.
static int gram_core(dcg_context* ctx, cudaStream_t st, const double* W, const double* AW, long long n, int k,
                     int prune, double* L_out, int* d_active, long long* k_out, long long* info, Arena& ar) {
    double* graw = ar.take<double>((size_t)k * k);
    double* gsym = ar.take<double>((size_t)k * k);
    double* lwork = ar.take<double>((size_t)2 * k * k);
    double* parts = ar.take<double>(dcg_xty_scratch_doubles(ctx, k, k));
    DevStatus* ds = ar.take<DevStatus>(1);
    DCG_CUDA(cudaMemsetAsync(ds, 0, sizeof(DevStatus), st));
    int rc = dcg_xty(ctx, st, W, k, AW, k, n, k, k, graw, parts);
    if (rc) return rc;
    rc = dcg_gram_factor_launch(st, graw, k, prune, gsym, lwork, d_active, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (hs.status != DCG_OK) {
        if (info) *info = hs.info;
        return hs.status;
    }
    const long long kk = hs.count;
    DCG_CUDA(cudaMemcpyAsync(L_out, lwork, sizeof(double) * kk * kk, cudaMemcpyDeviceToDevice, st));
    *k_out = kk;
    return DCG_OK;
}

static size_t gram_scratch_bytes(dcg_context* ctx, int k) {
    return al(sizeof(double) * k * k) * 2 + al(sizeof(double) * 2 * k * k) +
           al(sizeof(double) * dcg_xty_scratch_doubles(ctx, k, k)) + al(sizeof(DevStatus)) + al(sizeof(int) * 64) +
           4096;
}

// RecycleBasis.ensure_factored (solvers.py:107-115): no pruning, GramNotSpd.
extern "C" int dcg_gram_factor(dcg_context* ctx, void* stream, double* d_w, double* d_aw, long long n, long long k,
                               int prune, double* d_chol, long long* k_out, long long* info) {
    if (!ctx || n < 0 || k < 0) return DCG_E_CONFIG;
    if (info) *info = 0;
    if (k_out) *k_out = k;
    if (k == 0) return DCG_OK;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const size_t nk = sizeof(double) * n * k;
    int rc = dcg_ws_reserve(ctx, gram_scratch_bytes(ctx, (int)k) + (prune ? 2 * al(nk) : 0));
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    int* active = ar.take<int>(DCG_MAX_K);
    long long kk = k;
    rc = gram_core(ctx, st, d_w, d_aw, n, (int)k, prune, d_chol, active, &kk, info, ar);
    if (rc) return rc;
    if (prune && kk != k) {
        // compact W and AW in place through scratch copies
        double* wtmp = ar.take<double>(n * k);
        double* awtmp = ar.take<double>(n * k);
        DCG_CUDA(cudaMemcpyAsync(wtmp, d_w, nk, cudaMemcpyDeviceToDevice, st));
        DCG_CUDA(cudaMemcpyAsync(awtmp, d_aw, nk, cudaMemcpyDeviceToDevice, st));
        gather_cols_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(wtmp, n, (int)k, active, (int)kk, d_w);
        gather_cols_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(awtmp, n, (int)k, active, (int)kk, d_aw);
        DCG_LAUNCHED();
    }
    if (k_out) *k_out = kk;
    DCG_CUDA(cudaStreamSynchronize(st));
    return DCG_OK;
}

// refresh_basis (recycle.py:80-92): AW = A W, then pruning Gram factorisation.
// d_w_out / d_aw_out receive n x k_out compacted columns.
extern "C" int dcg_refresh_basis(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_w,
                                 long long k, double* d_w_out, double* d_aw_out, double* d_chol, long long* k_out,
                                 long long* info) {
    if (!ctx || k < 0) return DCG_E_CONFIG;
    if (info) *info = 0;
    int rc = check_dense_op(op);
    if (rc) return rc;
    if (op->row0 != 0 || op->rows != op->n) return DCG_E_UNSUPPORTED;
    const long long n = op->n;
    if (k_out) *k_out = k;
    if (k == 0) return DCG_OK;
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const size_t nk = sizeof(double) * n * k;
    const size_t need = al(sizeof(double) * block_scratch_doubles(op, (int)k)) + al(nk) +
                        gram_scratch_bytes(ctx, (int)k);
    rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* aw = ar.take<double>(n * k);
    int* active = ar.take<int>(DCG_MAX_K);
    double* scratch = ar.take<double>(block_scratch_doubles(op, (int)k));
    if (op->kind == DCG_OP_RBF)
        rc = dcg_rbf_mf_block(ctx, st, op, d_w, (int)k, op->d_s, op->d_s, op->shift, aw);
    else
        rc = block_apply_op(ctx, st, op, d_w, (int)k, op->d_s, op->d_s, op->shift, d_w, aw, scratch);
    if (rc) return rc;
    long long kk = k;
    rc = gram_core(ctx, st, d_w, aw, n, (int)k, 1, d_chol, active, &kk, info, ar);
    if (rc) return rc;
    if (kk == k) {
        DCG_CUDA(cudaMemcpyAsync(d_w_out, d_w, nk, cudaMemcpyDeviceToDevice, st));
        DCG_CUDA(cudaMemcpyAsync(d_aw_out, aw, nk, cudaMemcpyDeviceToDevice, st));
    } else {
        gather_cols_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(d_w, n, (int)k, active, (int)kk, d_w_out);
        gather_cols_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(aw, n, (int)k, active, (int)kk, d_aw_out);
        DCG_LAUNCHED();
    }
    if (k_out) *k_out = kk;
    DCG_CUDA(cudaStreamSynchronize(st));
    return DCG_OK;
}

// Device-side end of an asynchronous refresh: the surviving column count
// (0 when the extraction that produced W failed -- its result block says so --
// or when pruning empties the basis: recycle.py:178-179 then solves with
// plain CG), the gathered W / AW columns and the compact factor.
__global__ void refresh_finish_kernel(const DevStatus* ds, const long long* d_valid, const int* active, int k,
                                      long long n, const double* W, const double* AW, const double* Lc,
                                      double* w_out, double* aw_out, double* chol_out, long long* kout) {
    const bool ok = ds->status == DCG_OK && (!d_valid || d_valid[0] == DCG_OK);
    const int kk = ok ? (int)ds->count : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *kout = kk;
    if (kk == 0) return;
    const long long total = n * kk;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / kk;
        const int c = active[(int)(e - i * kk)];
        w_out[e] = W[i * k + c];
        aw_out[e] = AW[i * k + c];
    }
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)kk * kk;
         e += (long long)gridDim.x * blockDim.x)
        chol_out[e] = Lc[e];
}

// refresh_basis without host synchronisation: the column count stays on the
// device (*d_kout), for dcg_solve_async's d_kuse.  d_valid (optional) is the
// result block of the extraction that produced d_w.
extern "C" int dcg_refresh_basis_async(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_w,
                                       long long k, const long long* d_valid, double* d_w_out, double* d_aw_out,
                                       double* d_chol, long long* d_kout) {
    if (!ctx || k < 0 || !d_kout) return DCG_E_CONFIG;
    int rc = check_dense_op(op);
    if (rc) return rc;
    if (op->row0 != 0 || op->rows != op->n) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    if (k == 0) {
        DCG_CUDA(cudaMemsetAsync(d_kout, 0, sizeof(long long), st));
        return DCG_OK;
    }
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    const long long n = op->n;
    const size_t nk = sizeof(double) * n * k;
    const size_t need = al(sizeof(double) * block_scratch_doubles(op, (int)k)) + al(nk) +
                        gram_scratch_bytes(ctx, (int)k);
    rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* aw = ar.take<double>(n * k);
    int* active = ar.take<int>(DCG_MAX_K);
    double* scratch = ar.take<double>(block_scratch_doubles(op, (int)k));
    if (op->kind == DCG_OP_RBF)
        rc = dcg_rbf_mf_block(ctx, st, op, d_w, (int)k, op->d_s, op->d_s, op->shift, aw);
    else
        rc = block_apply_op(ctx, st, op, d_w, (int)k, op->d_s, op->d_s, op->shift, d_w, aw, scratch);
    if (rc) return rc;
    double* graw = ar.take<double>((size_t)k * k);
    double* gsym = ar.take<double>((size_t)k * k);
    double* lwork = ar.take<double>((size_t)2 * k * k);
    double* parts = ar.take<double>(dcg_xty_scratch_doubles(ctx, (int)k, (int)k));
    DevStatus* ds = ar.take<DevStatus>(1);   // written by every path of gram_factor (no memset)
    rc = dcg_xty(ctx, st, d_w, (int)k, aw, (int)k, n, (int)k, (int)k, graw, parts);
    if (rc) return rc;
    rc = dcg_gram_factor_launch(st, graw, (int)k, 1, gsym, lwork, active, ds);
    if (rc) return rc;
    refresh_finish_kernel<<<ctx->sm_count * 2, 256, 0, st>>>(ds, d_valid, active, (int)k, n, d_w, aw, lwork, d_w_out,
                                                             d_aw_out, d_chol, d_kout);
    DCG_LAUNCHED();
    return DCG_OK;
}

// P_W v = v - AW (W'AW)^-1 W' v   (solvers.py:242-256)
__global__ void project_kernel(long long n, int k, const double* L, const double* c, const double* v,
                               const double* AW, double* out) {
    __shared__ double y[DCG_MAX_K];
    if (threadIdx.x == 0 && blockIdx.x >= 0) {
        // forward / back substitution (k <= 64), reference order
        double t[DCG_MAX_K];
        for (int i = 0; i < k; ++i) {
            double acc = c[i];
            for (int j = 0; j < i; ++j) acc = sub_rn(acc, mul_rn(L[i * k + j], t[j]));
            t[i] = div_rn(acc, L[i * k + i]);
        }
        for (int i = k - 1; i >= 0; --i) {
            double acc = t[i];
            for (int j = i + 1; j < k; ++j) acc = sub_rn(acc, mul_rn(L[j * k + i], y[j]));
            y[i] = div_rn(acc, L[i * k + i]);
        }
    }
    cta_sync();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc = fma(AW[i * k + j], y[j], acc);
        out[i] = sub_rn(v[i], acc);
    }
}

extern "C" int dcg_deflation_project(dcg_context* ctx, void* stream, long long n, const dcg_basis* basis,
                                     const double* d_v, double* d_out) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    const long long k = basis ? basis->k : 0;
    if (k == 0) {
        if (n) DCG_CUDA(cudaMemcpyAsync(d_out, d_v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        return DCG_OK;
    }
    if (k > DCG_MAX_K) return DCG_E_UNSUPPORTED;
    int rc = dcg_ws_reserve(ctx, al(sizeof(double) * k) + al(sizeof(double) * dcg_xty_scratch_doubles(ctx, (int)k, 1)));
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* c = ar.take<double>(k);
    double* parts = ar.take<double>(dcg_xty_scratch_doubles(ctx, (int)k, 1));
    rc = dcg_xty(ctx, st, basis->d_w, k, d_v, 1, n, (int)k, 1, c, parts);
    if (rc) return rc;
    project_kernel<<<ctx->sm_count, 256, 0, st>>>(n, (int)k, basis->d_chol, c, d_v, basis->d_aw, d_out);
    DCG_LAUNCHED();
    return DCG_OK;
}

// ---------------------------------------------------------------------------
// L4: GPC glue
// ---------------------------------------------------------------------------
extern "C" int dcg_gpc_derivs(dcg_context* ctx, void* stream, long long n, const double* d_f, const double* d_y,
                              double* d_grad, double* d_h, double* loglik) {
    if (!ctx || n < 0) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2) + al(sizeof(DevStatus));
    int rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DevStatus* ds = ar.take<DevStatus>(1);
    rc = dcg_derivs_launch(ctx, st, n, d_f, d_y, nullptr, d_grad, d_h, part, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (loglik) *loglik = hs.value;
    return DCG_OK;
}

// Laplace-Newton start state (gpc.py:160-172, f = 0): f = a = 0, the
// likelihood derivatives at f = 0 and loglik, plus the count of labels that
// are not -1 / +1 (gpc.py:135-139) -- one launch pair and one host read.
extern "C" int dcg_gpc_init(dcg_context* ctx, void* stream, long long n, const double* d_y, double* d_f, double* d_a,
                            double* d_grad, double* d_h, double* loglik, long long* bad_labels) {
    if (!ctx || n < 0 || (n > 0 && (!d_y || !d_f || !d_a || !d_grad || !d_h))) return DCG_E_CONFIG;
    if (n == 0) {
        if (loglik) *loglik = 0.0;
        if (bad_labels) *bad_labels = 0;
        return DCG_OK;
    }
    cudaStream_t st = as_stream(stream);
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2) + al(sizeof(DevStatus));
    int rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DevStatus* ds = ar.take<DevStatus>(1);
    DCG_CUDA(cudaMemsetAsync(d_f, 0, sizeof(double) * (size_t)n, st));
    DCG_CUDA(cudaMemsetAsync(d_a, 0, sizeof(double) * (size_t)n, st));
    rc = dcg_derivs_launch(ctx, st, n, d_f, d_y, nullptr, d_grad, d_h, part, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (loglik) *loglik = hs.value;
    if (bad_labels) *bad_labels = hs.info;
    return DCG_OK;
}

// dcg_gpc_init without the host read: the 48-byte status block (int32 status,
// int64 info = labels not in {-1, +1} at byte 8, f64 loglik at byte 32) goes to
// d_status (device, 64 bytes); the caller copies it back when it needs it --
// after it has enqueued the first Newton system and solve.
extern "C" int dcg_gpc_init_async(dcg_context* ctx, void* stream, long long n, const double* d_y, double* d_f,
                                  double* d_a, double* d_grad, double* d_h, void* d_status) {
    if (!ctx || n <= 0 || !d_y || !d_f || !d_a || !d_grad || !d_h || !d_status) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2);
    int rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DCG_CUDA(cudaMemsetAsync(d_f, 0, sizeof(double) * (size_t)n, st));
    DCG_CUDA(cudaMemsetAsync(d_a, 0, sizeof(double) * (size_t)n, st));
    return dcg_derivs_launch(ctx, st, n, d_f, d_y, nullptr, d_grad, d_h, part, static_cast<DevStatus*>(d_status), nullptr);
}

extern "C" int dcg_gpc_objective(dcg_context* ctx, void* stream, long long n, const double* d_f, const double* d_y,
                                 const double* d_a, double* d_grad, double* d_h, double* loglik, double* psi) {
    if (!ctx || n < 0 || !d_f || !d_y || !d_a) return DCG_E_CONFIG;
    cudaStream_t st = as_stream(stream);
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2) + al(sizeof(DevStatus));
    int rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DevStatus* ds = ar.take<DevStatus>(1);
    rc = dcg_derivs_launch(ctx, st, n, d_f, d_y, d_a, d_grad, d_h, part, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (loglik) *loglik = hs.value;
    if (psi) *psi = hs.value2;
    return DCG_OK;
}

extern "C" int dcg_gpc_newton_system(dcg_context* ctx, void* stream, const dcg_operator* kop, const double* d_f,
                                     const double* d_grad, const double* d_h, double* d_s, double* d_inner,
                                     double* d_b) {
    if (!ctx) return DCG_E_CONFIG;
    int rc = check_dense_op(kop);
    if (rc) return rc;
    cudaStream_t st = as_stream(stream);
    const long long n = kop->n;
    rc = dcg_ws_reserve(ctx, sizeof(double) * apply_k_scratch(kop) + 256);
    if (rc) return rc;
    rc = dcg_newton_prep_launch(ctx, st, n, d_f, d_grad, d_h, d_s, d_inner);
    if (rc) return rc;
    // b = s (.) (K inner): K's own scaling/shift are ignored here (K is the kernel matrix)
    return apply_k(ctx, st, kop, d_inner, nullptr, d_s + kop->row0, 0.0, d_b, static_cast<double*>(ctx->ws));
}

// newton_system plus the next solve's first product, ax0 = A x_prev with
// A = I + S K S of the new system, from ONE pass over K's lower triangle when
// K is stored symmetric (sym_pass1<NV = 2>): b and ax0 are bitwise the results
// of the two separate products (newton_system's K inner, the operator's
// A x_prev), one K read fewer per Newton step.  Other operators: two products.
extern "C" int dcg_gpc_newton_system_ax0(dcg_context* ctx, void* stream, const dcg_operator* kop, const double* d_f,
                                         const double* d_grad, const double* d_h, const double* d_x_prev,
                                         double* d_s, double* d_inner, double* d_b, double* d_ax0) {
    if (!ctx || !d_x_prev || !d_ax0) return DCG_E_CONFIG;
    int rc = check_dense_op(kop);
    if (rc) return rc;
    cudaStream_t st = as_stream(stream);
    const long long n = kop->n;
    const bool fused = kop->kind == DCG_OP_DENSE_SYM && kop->row0 == 0 && kop->rows == n && aligned16(d_inner);
    const size_t scr = fused ? dcg_sym_apply2_scratch_doubles(n) : apply_k_scratch(kop);
    rc = dcg_ws_reserve(ctx, al(sizeof(double) * (size_t)n) + sizeof(double) * scr + 256);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* xs = ar.take<double>(n);
    double* scratch = ar.take<double>(scr);
    if (!fused) {
        rc = dcg_newton_prep_launch(ctx, st, n, d_f, d_grad, d_h, d_s, d_inner);
        if (rc) return rc;
        rc = apply_k(ctx, st, kop, d_inner, nullptr, d_s + kop->row0, 0.0, d_b, scratch);
        if (rc) return rc;
        return apply_k(ctx, st, kop, d_x_prev, d_s, d_s + kop->row0, 1.0, d_ax0, scratch);
    }
    rc = dcg_newton_prep2_launch(ctx, st, n, d_f, d_grad, d_h, d_x_prev, d_s, d_inner, xs);
    if (rc) return rc;
    return dcg_sym_apply2(ctx, st, kop->d_k, kop->d_kp, kop->ldk, n, d_inner, xs, nullptr, d_x_prev, d_s, d_s, 0.0, 1.0, d_b,
                          d_ax0, scratch);
}

// gpc newton_update without host synchronisation: (loglik, psi) go to d_llpsi
// (2 doubles on the device).  Full (unsharded) operators only.
extern "C" int dcg_gpc_newton_update_async(dcg_context* ctx, void* stream, const dcg_operator* kop,
                                           const double* d_inner, const double* d_s, const double* d_x,
                                           const double* d_y, double* d_a, double* d_f, double* d_grad, double* d_h,
                                           double* d_llpsi) {
    if (!ctx || !d_llpsi) return DCG_E_CONFIG;
    int rc = check_dense_op(kop);
    if (rc) return rc;
    if (kop->row0 != 0 || kop->rows != kop->n) return DCG_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    const long long n = kop->n;
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2) + al(sizeof(DevStatus)) +
                        al(sizeof(double) * apply_k_scratch(kop));
    rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DevStatus* ds = ar.take<DevStatus>(1);
    double* scratch = ar.take<double>(apply_k_scratch(kop));
    rc = dcg_newton_a_launch(ctx, st, n, d_inner, d_s, d_x, d_a);
    if (rc) return rc;
    rc = apply_k(ctx, st, kop, d_a, nullptr, nullptr, 0.0, d_f, scratch);
    if (rc) return rc;
    // the finalize kernel writes (loglik, psi) to d_llpsi itself
    return dcg_derivs_launch(ctx, st, n, d_f, d_y, d_a, d_grad, d_h, part, ds, d_llpsi);
}

extern "C" int dcg_gpc_newton_update(dcg_context* ctx, void* stream, const dcg_operator* kop, const double* d_inner,
                                     const double* d_s, const double* d_x, const double* d_y, double* d_a,
                                     double* d_f, double* d_grad, double* d_h, double* loglik, double* psi) {
    if (!ctx) return DCG_E_CONFIG;
    int rc = check_dense_op(kop);
    if (rc) return rc;
    cudaStream_t st = as_stream(stream);
    const long long n = kop->n;
    if (kop->row0 != 0 || kop->rows != kop->n) {
        // row slab (sharded Newton loop): a over all n entries, f for this
        // rank's rows only; the caller gathers f and calls dcg_gpc_objective
        rc = dcg_ws_reserve(ctx, sizeof(double) * apply_k_scratch(kop) + 256);
        if (rc) return rc;
        rc = dcg_newton_a_launch(ctx, st, n, d_inner, d_s, d_x, d_a);
        if (rc) return rc;
        return apply_k(ctx, st, kop, d_a, nullptr, nullptr, 0.0, d_f, static_cast<double*>(ctx->ws));
    }
    const size_t need = al(sizeof(double) * 3 * ctx->sm_count * 2) + al(sizeof(DevStatus)) +
                        al(sizeof(double) * apply_k_scratch(kop));
    rc = dcg_ws_reserve(ctx, need);
    if (rc) return rc;
    Arena ar{static_cast<char*>(ctx->ws), 0};
    double* part = ar.take<double>(6 * ctx->sm_count);
    DevStatus* ds = ar.take<DevStatus>(1);
    double* scratch = ar.take<double>(apply_k_scratch(kop));
    rc = dcg_newton_a_launch(ctx, st, n, d_inner, d_s, d_x, d_a);
    if (rc) return rc;
    rc = apply_k(ctx, st, kop, d_a, nullptr, nullptr, 0.0, d_f, scratch);
    if (rc) return rc;
    rc = dcg_derivs_launch(ctx, st, n, d_f, d_y, d_a, d_grad, d_h, part, ds);
    if (rc) return rc;
    DevStatus hs;
    rc = dcg_read_status(ctx, st, ds, &hs);
    if (rc) return rc;
    if (loglik) *loglik = hs.value;
    if (psi) *psi = hs.value2;
    return DCG_OK;
}
