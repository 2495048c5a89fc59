/*
 * defcg_b200.h — C ABI of the B200-native deflated-CG (def-CG) hot path.
 *
 * The reference (`defcg`, arXiv 1706.00241) is a single-process CPU package
 * whose only plugin point is the kernel backend selected by DEFCG_BACKEND
 * (/root/reference/pkg/src/defcg/_kernels/__init__.py:11-45).  That per-kernel
 * boundary is too fine for a GPU (the solver loop would ship the n x n matrix
 * every iteration, solvers.py:169), so this ABI exposes two layers:
 *
 *   L0  dcg_k_*      device twins of the eight backend kernels
 *                    (_kernels/_core.pyx:16-177), for unit parity;
 *   L1-L4            the solver API one level up (linalg.py, solvers.py,
 *                    recycle.py, gpc.py): operator apply, Gram factor with
 *                    pruning, the whole CG / def-CG loop as ONE persistent
 *                    kernel, harmonic-Ritz extraction, the small dense
 *                    eigensolvers, RBF Gram assembly and the GPC Newton glue.
 *
 * Conventions
 *   - Every pointer argument named d_* is DEVICE memory (cudaMalloc / torch).
 *     Matrices are row-major fp64 with an explicit leading dimension; vectors
 *     are contiguous fp64.  The library never frees caller memory.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Every entry point returns an int status (DCG_OK == 0).  Entry points
 *     whose outcome depends on device data (pivot failures, breakdown,
 *     convergence) synchronise `stream` before returning; their payload
 *     (pivot index, iteration, remaining columns, sweeps) is written to
 *     *info when info != NULL — the same payloads the reference exceptions
 *     carry (errors.py:8-93).
 *   - A dcg_context owns the device workspace and must be used from one host
 *     thread at a time.
 */
#ifndef DEFCG_B200_H
#define DEFCG_B200_H

#if defined(__GNUC__)
#define DCG_API __attribute__((visibility("default")))
#else
#define DCG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DCG_ABI_VERSION 1

/* ---- status codes: one per reference exception type (errors.py) ---------- */
enum dcg_status {
    DCG_OK = 0,
    DCG_E_DIMENSION = 1,        /* DimensionMismatch            errors.py:24 */
    DCG_E_NOT_PD = 2,           /* NotPositiveDefinite(pivot)   errors.py:28-33 */
    DCG_E_BREAKDOWN = 3,        /* BreakdownZeroCurvature(it)   errors.py:44-49 */
    DCG_E_GRAM_NOT_SPD = 4,     /* GramNotSpd                   errors.py:52-53 */
    DCG_E_BASIS_DEFICIENT = 5,  /* BasisDeficient(remaining)    errors.py:56-61 */
    DCG_E_NO_CONVERGENCE = 6,   /* NoConvergence(sweeps)        errors.py:36-41 */
    DCG_E_ASYMMETRIC = 7,       /* ValueError from require_symmetric, linalg.py:49-55 */
    DCG_E_CONFIG = 8,           /* ValueError from bad arguments / SolverConfig */
    DCG_E_CUDA = 9,             /* CUDA runtime failure (info = cudaError_t) */
    DCG_E_UNSUPPORTED = 10      /* size outside the compiled limits (k > DCG_MAX_K ...) */
};

#define DCG_MAX_K 64            /* deflation basis columns handled by the fused kernels */
#define DCG_MAX_T 112           /* harmonic pencil order k_prev + m handled on device   */
#define DCG_RBF_MAX_DIM 64      /* point dimension of the matrix-free RBF operator      */

/* ---- operator: A = shift * I + diag(s) * K * diag(s) --------------------- */
/* The reference always materialises A (gpc.py:178 builds K * outer(s,s) + I).
 * Here A stays implicit: the Newton system is (K, s = sqrt(h), shift = 1);
 * an explicit matrix is (K = A, s = NULL, shift = 0).  `row0/rows` select the
 * locally stored row slab for row-sharded operators (rows == n on one GPU). */
/* DCG_OP_DENSE_SYM: same dense storage, K exactly symmetric and unsharded: the
 * GEMV streams only the lower triangle (64 x 64 tiles), half the bytes.     */
/* DCG_OP_RBF: matrix-free RBF Gram (config 5): K is regenerated from the
 * points d_x on every product (never stored); elements are computed exactly
 * as dcg_k_rbf_gram computes them.                                           */
enum dcg_op_kind { DCG_OP_DENSE = 0, DCG_OP_RBF = 1, DCG_OP_DENSE_SYM = 2 };

typedef struct dcg_operator {
    int kind;                 /* dcg_op_kind                                     */
    long long n;              /* global order                                    */
    long long row0;           /* first global row held by this rank              */
    long long rows;           /* number of rows held (== n unsharded)            */
    const double* d_k;        /* DENSE: rows x ldk slab of K (row-major)         */
    long long ldk;            /* DENSE: leading dimension (>= n, even)           */
    const double* d_x;        /* RBF: n x dim points, row-major (all points)     */
    long long dim;            /* RBF: point dimension                            */
    double var;               /* RBF: signal variance                            */
    double inv_two_ell2;      /* RBF: 1 / (2 lengthscale^2)                      */
    double diag;              /* RBF: diagonal value (var + jitter)              */
    const double* d_s;        /* optional symmetric scaling s (n), NULL = ones   */
    double shift;             /* identity shift                                  */
    const double* d_kp;       /* DENSE_SYM, optional: K's lower-triangle 64 x 64 */
                              /* tiles packed by dcg_pack_sym (NULL = read d_k)  */
} dcg_operator;

/* ---- deflation basis (solvers.py:84-115 RecycleBasis) -------------------- */
typedef struct dcg_basis {
    long long k;              /* columns (0 = plain CG)                          */
    const double* d_w;        /* n x k row-major W                               */
    const double* d_aw;       /* n x k row-major AW                              */
    const double* d_chol;     /* k x k row-major lower Cholesky factor of W'AW   */
} dcg_basis;

/* ---- SolverConfig (solvers.py:28-51) ------------------------------------- */
typedef struct dcg_solver_config {
    double tol;
    long long max_iters;      /* <= 0 selects the reference default 10 n         */
    long long ell;
    long long recompute_residual_every;
} dcg_solver_config;

/* ---- KrylovLog (solvers.py:54-72), caller-owned device buffers ----------- */
typedef struct dcg_krylov_log {
    long long ell;            /* capacity in logged iterations                   */
    double* d_p;              /* ell x n      search directions p_0..p_{m-1}     */
    double* d_r;              /* (ell+1) x n  residuals r_0..r_m                 */
    double* d_d;              /* ell          p'Ap                               */
    double* d_alpha;          /* ell                                             */
    double* d_beta;           /* ell                                             */
    double* d_mu;             /* ell x k      deflation coefficients (k > 0)     */
} dcg_krylov_log;

/* ---- SolveReport (solvers.py:75-81) -------------------------------------- */
typedef struct dcg_solve_info {
    long long iterations;
    long long stored;         /* m = logged iterations                           */
    int converged;
    int termination;          /* 0 = "converged", 1 = "max_iters"               */
    double rel_residual;      /* final recurrence residual                       */
    double norm_b;
    double device_ms;         /* solve-kernel time measured with CUDA events     */
} dcg_solve_info;

/* ---- context ------------------------------------------------------------- */
typedef struct dcg_context dcg_context;

DCG_API int dcg_version(void);
DCG_API const char* dcg_status_string(int status);
DCG_API int dcg_context_create(int device, dcg_context** out);
DCG_API int dcg_context_destroy(dcg_context* ctx);
/* kernels this process has launched through the library (benchmark accounting) */
DCG_API long long dcg_launch_count(void);
/* number of CTAs of the persistent solve kernel (one per SM) */
DCG_API int dcg_context_grid(dcg_context* ctx, int* blocks, int* sm_count);

/* ---- L0: device twins of the backend kernels (_core.pyx) ----------------- */
/* y = A x                                          _core.pyx:16-28  matvec   */
DCG_API int dcg_k_matvec(dcg_context* ctx, void* stream, const double* d_a, long long m,
                 long long n, long long lda, const double* d_x, double* d_y);
/* C(m x n) = A(m x kk) B(kk x n), all row-major   _core.pyx:31-44  gemm     */
DCG_API int dcg_k_gemm(dcg_context* ctx, void* stream, const double* d_a, const double* d_b,
               double* d_c, long long m, long long kk, long long n);
/* lower L with pivot rule acc <= pivot_tol -> fail   _core.pyx:47-66        */
DCG_API int dcg_k_cholesky(dcg_context* ctx, void* stream, const double* d_a, long long n,
                   double pivot_tol, double* d_l, long long* fail_index);
/*                                                  _core.pyx:69-94          */
DCG_API int dcg_k_solve_lower(dcg_context* ctx, void* stream, const double* d_l, long long n,
                      const double* d_b, double* d_y);
DCG_API int dcg_k_solve_lower_trans(dcg_context* ctx, void* stream, const double* d_l,
                            long long n, const double* d_b, double* d_x);
/* rows [row0, row0+rows) of the RBF Gram            _core.pyx:97-114        */
DCG_API int dcg_k_rbf_gram(dcg_context* ctx, void* stream, const double* d_x, long long n,
                   long long dim, double signal_var, double inv_two_ell2, double jitter,
                   double* d_k, long long ldk, long long row0, long long rows);
/*                                                  _core.pyx:117-132        */
DCG_API int dcg_k_rbf_cross(dcg_context* ctx, void* stream, const double* d_xa, long long na,
                    const double* d_xb, long long nb, long long dim, double signal_var,
                    double inv_two_ell2, double* d_k);
/* one cyclic Jacobi sweep in place                  _core.pyx:135-177       */
DCG_API int dcg_k_jacobi_sweep(dcg_context* ctx, void* stream, double* d_a, double* d_v,
                       long long n, long long* rotations);

/* ---- L1: dense linear algebra (linalg.py) -------------------------------- */
/* max|A - A'| <= rtol * max|A|  -> *symmetric = 1     linalg.py:49-55       */
DCG_API int dcg_check_symmetric(dcg_context* ctx, void* stream, const double* d_a, long long n,
                        long long lda, double rtol, int* symmetric);
/* cyclic-Jacobi eigen-decomposition, ascending      linalg.py:139-165        */
DCG_API int dcg_sym_eigen(dcg_context* ctx, void* stream, const double* d_a, long long n,
                  long long max_sweeps, double rtol, double* d_values, double* d_vectors,
                  long long* info);
/* G u = theta F u via F = L L'                       linalg.py:168-191        */
DCG_API int dcg_gen_sym_eigen(dcg_context* ctx, void* stream, const double* d_g, const double* d_f,
                      long long n, long long max_sweeps, double* d_values,
                      double* d_vectors, long long* info);

/* Packed copy of an exactly symmetric K for DCG_OP_DENSE_SYM operators: the
 * lower-triangle 64 x 64 tiles in tile-row order, each one contiguous 32 KB
 * block (zero beyond n, XOR-swizzled as the GEMV's shared-memory ring holds
 * it), so every tile is ONE bulk copy and DRAM pages are read sequentially.
 * The products and solves read d_kp instead of d_k when it is set; values
 * are those of the row-major path.  Not in the reference: its matvec reads
 * the dense ndarray (_core.pyx:16-28, linalg.py:58-63).                      */
DCG_API long long dcg_packed_sym_doubles(long long n);
/* 1 when a block product of k columns over a DENSE_SYM operator with d_kp runs
 * on the packed tiles (then d_k may be NULL), 0 when it needs d_k.          */
DCG_API int dcg_block_uses_packed(int k);
DCG_API int dcg_pack_sym(dcg_context* ctx, void* stream, const double* d_k, long long ldk, long long n,
                 double* d_kp);

/* ---- L2: operator and Krylov solvers (solvers.py) ------------------------ */
/* y = A x (rows of this rank only: y has op->rows entries)                    */
DCG_API int dcg_op_apply(dcg_context* ctx, void* stream, const dcg_operator* op,
                 const double* d_x, double* d_y);
/* Y = A X for a row-major n x k block (multi-vector, FP64 MMA)  recycle.py:90 */
DCG_API int dcg_op_apply_block(dcg_context* ctx, void* stream, const dcg_operator* op,
                       const double* d_x, long long k, double* d_y);
/* Gram = sym(W'AW); Cholesky with pivot 1e-14*max diag.  prune != 0 deletes the
 * failing-pivot column of W and AW in place and retries (recycle.py:66-77);
 * prune == 0 fails with DCG_E_GRAM_NOT_SPD (solvers.py:107-115).  d_chol gets
 * the k_out x k_out factor.                                                  */
DCG_API int dcg_gram_factor(dcg_context* ctx, void* stream, double* d_w, double* d_aw,
                    long long n, long long k, int prune, double* d_chol,
                    long long* k_out, long long* info);
/* refresh_basis (recycle.py:80-92): AW = A W for the new operator (FP64 MMA,
 * one pass over K), Gram factorisation with failing-pivot pruning; the
 * surviving columns are written compacted to d_w_out / d_aw_out (n x k_out). */
DCG_API int dcg_refresh_basis(dcg_context* ctx, void* stream, const dcg_operator* op,
                      const double* d_w, long long k, double* d_w_out, double* d_aw_out,
                      double* d_chol, long long* k_out, long long* info);
/* CG (basis == NULL or basis->k == 0, solvers.py:207-219) or deflated CG with
 * the x_prev warm-start correction (solvers.py:222-239); the whole
 * _run_loop (solvers.py:131-204) runs as one persistent cooperative kernel.
 * d_history needs max_iters + 1 entries.                                      */
DCG_API int dcg_solve(dcg_context* ctx, void* stream, const dcg_operator* op, const double* d_b,
              const double* d_x0, const dcg_basis* basis, const dcg_solver_config* cfg,
              double* d_x, dcg_krylov_log* log, double* d_history,
              dcg_solve_info* out, long long* info);
/* Enqueue-only dcg_solve: no host synchronisation.  d_kuse (optional device
 * int64): basis columns in use (<= basis->k, 0 = plain CG), as written by
 * dcg_refresh_basis_async.  d_status (64 bytes on the device) receives
 * {int32 status, int32 columns used, int64 info, int64 iterations, int64
 * stored log entries, f64 rel residual, f64 norm_b} in stream order.  The
 * log's mu rows keep the stride basis->k.  d_ax0 (optional): A x0 already
 * computed (the warm-start correction's first product, solvers.py:237).     */
DCG_API int dcg_solve_async(dcg_context* ctx, void* stream, const dcg_operator* op,
                            const double* d_b, const double* d_x0, const dcg_basis* basis,
                            const dcg_solver_config* cfg, double* d_x, dcg_krylov_log* log,
                            double* d_history, const long long* d_kuse, void* d_status,
                            const double* d_ax0);
/* Enqueue-only refresh_basis: surviving column count to *d_kout (device
 * int64; 0 when nothing survives -- BasisDeficient -- or when d_valid, the
 * result block of the extraction that produced d_w, reports a failure).
 * Outputs compacted to d_kout columns; d_w_out / d_aw_out hold n x k.       */
DCG_API int dcg_refresh_basis_async(dcg_context* ctx, void* stream, const dcg_operator* op,
                                    const double* d_w, long long k, const long long* d_valid,
                                    double* d_w_out, double* d_aw_out, double* d_chol,
                                    long long* d_kout);
/* v - AW (W'AW)^-1 W' v                              solvers.py:242-256       */
DCG_API int dcg_deflation_project(dcg_context* ctx, void* stream, long long n,
                          const dcg_basis* basis, const double* d_v, double* d_out);

/* ---- L3: recycling (recycle.py) ------------------------------------------ */
enum dcg_selection { DCG_SELECT_SMALLEST = 0, DCG_SELECT_LARGEST = 1 };
/* harmonic Ritz extraction (recycle.py:95-159).  prev may be NULL.  Outputs:
 * theta (k), u (T x k row-major, T = columns kept), z (n x T), w_next, aw_next
 * (n x k).  z/u may be NULL.  *t_out = T after zero-column dropping/pruning.
 * DCG_E_BASIS_DEFICIENT carries the reference's `remaining` in *info.        */
DCG_API int dcg_ritz_extract(dcg_context* ctx, void* stream, long long n, const dcg_krylov_log* log,
                     long long m, const dcg_basis* prev, long long k, int selection,
                     double* d_theta, double* d_u, double* d_z, double* d_w_next,
                     double* d_aw_next, long long* t_out, long long* info);

/* Asynchronous form: enqueue the whole extraction on `stream` without any host
 * synchronisation (the zero-column scan and the pruning decide the pencil
 * order on the device).  When the stream reaches the end, d_result[0..2]
 * (device int64) hold status, info payload and the kept column count T.     */
DCG_API int dcg_ritz_extract_async(dcg_context* ctx, void* stream, long long n,
                                   const dcg_krylov_log* log, long long m, const dcg_basis* prev,
                                   long long k, int selection, double* d_theta, double* d_u,
                                   double* d_z, double* d_w_next, double* d_aw_next,
                                   long long* d_result);

/* Device-driven form, enqueued behind dcg_solve_async without waiting for it:
 * the stored log length and the basis columns that solve used are read from
 * its status block (d_solve_status); prev->k is the basis' column capacity
 * (columns compacted, stride = columns used), log->ell the log capacity.
 * d_result as for dcg_ritz_extract_async (BasisDeficient when k > T).
 * stage 0 enqueues everything; stage 1 only the device-wide column work
 * (Z / AZ gather, normalisation, F and G), stage 2 the single-CTA pencil and
 * the W_next tail -- the two halves may go to different streams (the caller
 * orders stage 2 after stage 1) and must get identical arguments.  Stage 2
 * splits further into 3 (the pencil) and 4 (the SM-wide W_next tail), so
 * the tail can follow the pencil on another stream (ordered after it).
 * d_aw_next may be NULL when the caller refreshes the basis against its next
 * matrix before any use (AW_next = A W_next is then never formed).         */
DCG_API int dcg_ritz_extract_dev(dcg_context* ctx, void* stream, long long n,
                                 const dcg_krylov_log* log, const void* d_solve_status,
                                 const dcg_basis* prev, long long k, int selection,
                                 double* d_theta, double* d_w_next, double* d_aw_next,
                                 long long* d_result, int stage);

/* ---- L4: GPC Laplace-Newton glue (gpc.py) -------------------------------- */
/* loglik, grad, h of the logistic likelihood          gpc.py:126-157          */
DCG_API int dcg_gpc_derivs(dcg_context* ctx, void* stream, long long n, const double* d_f,
                   const double* d_y, double* d_grad, double* d_h, double* loglik);
/* start state f = a = 0 with its derivatives and loglik, and the number of
 * labels not in {-1, +1} (InvalidLabel)             gpc.py:135-172          */
DCG_API int dcg_gpc_init(dcg_context* ctx, void* stream, long long n, const double* d_y, double* d_f,
                 double* d_a, double* d_grad, double* d_h, double* loglik, long long* bad_labels);
/* s = sqrt(h); inner = h f + grad; b = s * (K inner)   gpc.py:175-183          */
/* dcg_gpc_init without the host read (the start state of gpc.py:160-172 and
 * the label check of gpc.py:135-139 for a pipelined caller): the 64-byte
 * status block -- int32 status at byte 0, int64 count of labels outside
 * {-1, +1} at byte 8, f64 loglik at byte 32 -- is left in d_status (device).  */
DCG_API int dcg_gpc_init_async(dcg_context* ctx, void* stream, long long n, const double* d_y,
                               double* d_f, double* d_a, double* d_grad, double* d_h, void* d_status);
DCG_API int dcg_gpc_newton_system(dcg_context* ctx, void* stream, const dcg_operator* kop,
                          const double* d_f, const double* d_grad, const double* d_h,
                          double* d_s, double* d_inner, double* d_b);
/* newton_system plus ax0 = (I + S K S) x_prev, the next solve's first product
 * (pass it to dcg_solve_async as d_ax0): one pass over a symmetric-stored K
 * serves both products, bitwise equal to computing them separately.
 * Replaces the pair build_newton_system (gpc.py:175-183) + the first A x0 of
 * the deflated solve, r_prev = b - A x_prev (solvers.py:237).              */
DCG_API int dcg_gpc_newton_system_ax0(dcg_context* ctx, void* stream, const dcg_operator* kop,
                          const double* d_f, const double* d_grad, const double* d_h,
                          const double* d_x_prev, double* d_s, double* d_inner, double* d_b,
                          double* d_ax0);
/* a = inner - s x; f = K a; (loglik, grad, h)(f); psi = loglik - f'a / 2
 *                                                     gpc.py:186-209
 * For a row-slab kop (sharded): a for all n entries, f for the slab's rows
 * only; loglik / psi untouched (gather f, then dcg_gpc_objective).          */
DCG_API int dcg_gpc_newton_update(dcg_context* ctx, void* stream, const dcg_operator* kop,
                          const double* d_inner, const double* d_s, const double* d_x,
                          const double* d_y, double* d_a, double* d_f, double* d_grad,
                          double* d_h, double* loglik, double* psi);

/* Enqueue-only newton_update for a full operator: (loglik, psi) are written
 * to d_llpsi (2 doubles on the device) in stream order.                     */
DCG_API int dcg_gpc_newton_update_async(dcg_context* ctx, void* stream, const dcg_operator* kop,
                                        const double* d_inner, const double* d_s, const double* d_x,
                                        const double* d_y, double* d_a, double* d_f, double* d_grad,
                                        double* d_h, double* d_llpsi);
/* (loglik, grad, h)(f) and psi = loglik - f'a / 2 for full f, a (gpc.py:204-209) */
DCG_API int dcg_gpc_objective(dcg_context* ctx, void* stream, long long n, const double* d_f,
                              const double* d_y, const double* d_a, double* d_grad, double* d_h,
                              double* loglik, double* psi);

/* ---- L5: row-sharded def-CG ------------------------------ *
 * K is row-partitioned over R ranks (one process per GPU); a rank owns the
 * slab rows [row0, row0 + rows) of K (op->kind = DCG_OP_DENSE, op->d_k = its
 * first row) and the same rows of x, r, p, Ap, W, AW.  The iteration of
 * solvers.py:131-204 becomes, per rank (collectives by the caller, e.g. NCCL):
 *     all-gather p -> dcg_shard_apply_dot -> all-reduce(1)
 *     -> dcg_shard_update -> all-reduce(1 + k) -> dcg_shard_direction
 * Scalars never leave the device: every kernel reads a dcg_shard_state at
 * entry and only the last CTA to finish writes it, so a kernel enqueued after
 * convergence (done != 0) is a no-op and every rank enqueues the same
 * collectives.  Reductions are fixed-order; with the all-reduced inputs being
 * bit-identical on all ranks, every rank takes the same decisions.          */
typedef struct dcg_shard_state {
    double rr;            /* r'r of the current residual (global)              */
    double norm_b;        /* ||b||                                             */
    double rel;           /* sqrt(rr) / norm_b                                 */
    double alpha, beta, d;
    double tol;
    long long it;         /* completed iterations                              */
    long long max_iters;
    long long done;       /* 1: converged / max_iters / breakdown / zero rhs   */
    long long status;     /* DCG_OK or DCG_E_BREAKDOWN                         */
    long long info;       /* breakdown iteration                               */
    long long ell;        /* KrylovLog capacity                                */
    long long pad[3];
} dcg_shard_state;

/* out = A_rows v (v: all n entries) for this rank's rows; part[0] = sum over
 * the rank's rows of v_i out_i (p'Ap partial) when part != NULL.  No-op if
 * state != NULL and state->done.                                              */
DCG_API int dcg_shard_apply_dot(dcg_context* ctx, void* stream, const dcg_operator* op,
                                const double* d_v, double* d_out, double* d_part,
                                const dcg_shard_state* d_state);
/* r = b - A_rows v (v full): r_prev (warm start), r_0, and the true-residual
 * refresh (solvers.py:175-177; no-op if state != NULL and state->done).      */
DCG_API int dcg_shard_residual(dcg_context* ctx, void* stream, const dcg_operator* op,
                               const double* d_v, const double* d_b, double* d_r,
                               const dcg_shard_state* d_state);
/* part = [u'u, M' w] over the rank's rows (M: rows x k row-major; k may be 0). */
DCG_API int dcg_shard_partials(dcg_context* ctx, void* stream, long long rows, int k,
                               const double* d_u, const double* d_w, const double* d_m,
                               double* d_part);
/* Warm start (deflated_cg_solve, solvers.py:236-238) from the reduced
 * [b'b, W' r_prev]: x0 = x_prev + W chol_solve(L, W'r_prev); initialises the
 * state (norm_b, tol, max_iters, ell, it = 0).  k = 0: x0 = x_prev.           */
DCG_API int dcg_shard_start(dcg_context* ctx, void* stream, long long rows, int k,
                            const double* d_red, const double* d_chol, const double* d_w,
                            const double* d_xprev, double* d_x0, dcg_shard_state* d_state,
                            double tol, long long max_iters, long long ell);
/* From the reduced [r0'r0, AW' r0]: mu_0, p_0 = r_0 - W mu_0 (or r_0), rel_0,
 * history[0], log r_0 / p_0 / mu_0, done; zero rhs -> x = 0 (solvers.py:142-147). */
/* dcg_shard_start and r0 = r_prev - (AW) c in d_r (holding r_prev = b - A x_prev on
 * entry): the deflated warm start without a second product (solvers.py:236-238). */
DCG_API int dcg_shard_start_r(dcg_context* ctx, void* stream, long long rows, int k,
                              const double* d_red, const double* d_chol, const double* d_w,
                              const double* d_aw, const double* d_xprev, double* d_x0, double* d_r,
                              dcg_shard_state* d_state, double tol, long long max_iters, long long ell);
DCG_API int dcg_shard_begin(dcg_context* ctx, void* stream, long long rows, int k,
                            const double* d_red, const double* d_chol, const double* d_w,
                            const double* d_r, double* d_p, double* d_x, dcg_shard_state* d_state,
                            double* d_history, double* d_log_r, double* d_log_p, double* d_log_mu);
/* mode 0: alpha = rr / d (d = reduced p'Ap; d <= 0 -> breakdown); x += alpha p;
 *         r -= alpha Ap; part = [r'r, AW' r]; logs d, alpha, r_it.
 * mode 1 (true-residual iteration): only the alpha / x / it / d, alpha part;
 * mode 2 (after dcg_shard_residual): only part = [r'r, AW' r] and the r_it log. */
DCG_API int dcg_shard_update(dcg_context* ctx, void* stream, int mode, long long rows, int k,
                             const double* d_red_d, double* d_x, double* d_r, const double* d_p,
                             const double* d_ap, const double* d_aw, double* d_part,
                             dcg_shard_state* d_state, double* d_log_r, double* d_log_d,
                             double* d_log_alpha, double* d_log_beta);
/* beta = rr'/rr, mu = chol_solve(L, AW'r), p = beta p + r - W mu (k > 0) or
 * r + beta p; rel, history[it], logs p_it / mu_it; done.                       */
DCG_API int dcg_shard_direction(dcg_context* ctx, void* stream, long long rows, int k,
                                const double* d_red, const double* d_chol, const double* d_w,
                                const double* d_r, double* d_p, dcg_shard_state* d_state,
                                double* d_history, double* d_log_p, double* d_log_mu,
                                double* d_log_beta);
/* The vector phases of one iteration of _run_loop (solvers.py:169-191) on
 * replicated vectors (the tile-share path: rows = n on every rank) in ONE
 * cooperative launch: Ap = shift p + s (.) t with d_t the all-reduced
 * K (s (.) p), d = p'Ap, alpha, x, r, [r'r, AW'r], beta, mu, p, history and
 * logs -- dcg_shard_epilogue(0) + dcg_shard_update(0) + dcg_shard_direction
 * with two grid barriers instead of three launches.  No-op if state->done.   */
DCG_API int dcg_shard_step(dcg_context* ctx, void* stream, long long rows, int k, const double* d_t,
                           const double* d_s, double shift, double* d_x, double* d_r, double* d_p,
                           double* d_ap, const double* d_w, const double* d_aw, const double* d_chol,
                           dcg_shard_state* d_state, double* d_history, double* d_log_r,
                           double* d_log_p, double* d_log_d, double* d_log_alpha, double* d_log_beta,
                           double* d_log_mu);

/* ---- L5b: sharded matrix-free products in the symmetric form (config 5) -- *
 * Rank `rank` of `world` evaluates an equal-cost share of the lower-triangle
 * 64 x 64 tiles of K (each pair once) for the full vector d_v (n, gathered)
 * and writes its partial t = (K (s (.) v)) share to d_t (all n rows, zero
 * where it has no tiles); the caller all-reduces d_t over the ranks and runs
 * dcg_shard_epilogue.  op: the rank's RBF slab (d_s, shift, row0/rows used by
 * the epilogue only).  Work per rank: n^2 / (2 world) pairs, against n^2 /
 * world for the row-slab dcg_shard_apply_dot.                              */
DCG_API int dcg_shard_rbf_sym_partial(dcg_context* ctx, void* stream, const dcg_operator* op,
                                      int rank, int world, const double* d_v, double* d_t,
                                      const dcg_shard_state* d_state);
/* mode 0: d_out = (A v) on the slab rows and d_part = its p'Ap partial;
 * mode 1: d_out = b - (A v) -- from the all-reduced t = K (s (.) v) (full).  */
/* Stored Gram over a TILE SHARE (replicated vectors, one all-reduce of n
 * doubles per product): rank r of R holds the packed lower-triangle tiles
 * [t_lo, t_hi) of dcg_shard_tile_range (an equal-cost split of the tile
 * sequence), built from the replicated points by dcg_k_rbf_gram_packed
 * (entries bitwise those of dcg_k_rbf_gram).  dcg_shard_tiles_partial writes
 * the rank's partial t = K_share (s (.) v) for all n rows (op: DENSE_SYM,
 * d_kp = the share, d_s the full scale vector); the sum over ranks is
 * K (s (.) v).  Replaces the slab GEMV + all-gather of p of
 * solvers.py:169 (matvec) in the sharded loop; no reference counterpart.   */
DCG_API int dcg_shard_tile_range(long long n, int rank, int world, long long* t_lo, long long* t_hi);
DCG_API int dcg_k_rbf_gram_packed(dcg_context* ctx, void* stream, const double* d_x, long long n,
                          long long dim, double signal_var, double inv_two_ell2, double jitter,
                          long long t_lo, long long t_hi, double* d_kp);
DCG_API int dcg_shard_tiles_partial(dcg_context* ctx, void* stream, const dcg_operator* op, int rank,
                            int world, const double* d_v, double* d_t,
                            const dcg_shard_state* d_state);
/* Two unscaled products K v1, K v2 over one pass of the tile share (partials
 * for all n rows; the caller all-reduces both): the Newton system's K inner
 * and the next solve's first product (gpc.py:175-183, solvers.py:237).     */
DCG_API int dcg_shard_tiles_partial2(dcg_context* ctx, void* stream, const dcg_operator* op, int rank,
                             int world, const double* d_v1, const double* d_v2, double* d_t1,
                             double* d_t2);
DCG_API int dcg_shard_epilogue(dcg_context* ctx, void* stream, int mode, const dcg_operator* op,
                               const double* d_v, const double* d_b, const double* d_t,
                               double* d_out, double* d_part, const dcg_shard_state* d_state);

#ifdef __cplusplus
}
#endif
#endif /* DEFCG_B200_H */
