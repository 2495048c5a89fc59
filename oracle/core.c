/*
 * oracle/core.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product path).  Plain-C restatement of the reference's compiled kernel core
 * /root/reference/pkg/src/defcg/_kernels/_core.pyx (Cython, built there with
 * -O3 and no -ffast-math, setup.py:31-44).  Every loop keeps the reference's
 * strictly left-to-right accumulation order, and this file is compiled with
 * -ffp-contract=off, so the results are bit-identical to `_core` on the same
 * inputs (pinned by tests/test_oracle.py against tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
 * the shared object built from this file.
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

typedef long long i64;

/* y = A x, each row one serial chain            _core.pyx:16-28 */
void or_matvec(const double* a, i64 m, i64 n, const double* x, double* y) {
    for (i64 i = 0; i < m; ++i) {
        const double* row = a + i * n;
        double acc = 0.0;
        for (i64 j = 0; j < n; ++j) acc = acc + row[j] * x[j];
        y[i] = acc;
    }
}

/* C = A B in i-k-j order, C starts at zero       _core.pyx:31-44 */
void or_gemm(const double* a, const double* b, double* c, i64 m, i64 kk, i64 n) {
    memset(c, 0, sizeof(double) * (size_t)(m * n));
    for (i64 i = 0; i < m; ++i)
        for (i64 t = 0; t < kk; ++t) {
            const double ait = a[i * kk + t];
            double* crow = c + i * n;
            const double* brow = b + t * n;
            for (i64 j = 0; j < n; ++j) crow[j] = crow[j] + ait * brow[j];
        }
}

/* lower Cholesky; returns failing pivot or -1    _core.pyx:47-66 */
i64 or_cholesky(const double* a, i64 n, double pivot_tol, double* l) {
    memset(l, 0, sizeof(double) * (size_t)(n * n));
    for (i64 j = 0; j < n; ++j) {
        double acc = a[j * n + j];
        for (i64 t = 0; t < j; ++t) acc = acc - l[j * n + t] * l[j * n + t];
        if (acc <= pivot_tol) return j;
        const double ljj = sqrt(acc);
        l[j * n + j] = ljj;
        for (i64 i = j + 1; i < n; ++i) {
            acc = a[i * n + j];
            for (i64 t = 0; t < j; ++t) acc = acc - l[i * n + t] * l[j * n + t];
            l[i * n + j] = acc / ljj;
        }
    }
    return -1;
}

/*                                                 _core.pyx:69-80 */
void or_solve_lower(const double* l, i64 n, const double* b, double* y) {
    for (i64 i = 0; i < n; ++i) {
        double acc = b[i];
        for (i64 j = 0; j < i; ++j) acc = acc - l[i * n + j] * y[j];
        y[i] = acc / l[i * n + i];
    }
}

/*                                                 _core.pyx:83-94 */
void or_solve_lower_trans(const double* l, i64 n, const double* b, double* x) {
    for (i64 i = n - 1; i >= 0; --i) {
        double acc = b[i];
        for (i64 j = i + 1; j < n; ++j) acc = acc - l[j * n + i] * x[j];
        x[i] = acc / l[i * n + i];
    }
}

/* lower triangle by difference-squared, mirrored; exact diagonal
 *                                                 _core.pyx:97-114 */
void or_rbf_gram(const double* x, i64 n, i64 d, double var, double inv_two_ell2, double jitter, double* k) {
    for (i64 i = 0; i < n; ++i) {
        k[i * n + i] = var + jitter;
        for (i64 j = 0; j < i; ++j) {
            double acc = 0.0;
            for (i64 t = 0; t < d; ++t) {
                const double diff = x[i * d + t] - x[j * d + t];
                acc = acc + diff * diff;
            }
            const double val = var * exp(-acc * inv_two_ell2);
            k[i * n + j] = val;
            k[j * n + i] = val;
        }
    }
}

/*                                                 _core.pyx:117-132 */
void or_rbf_cross(const double* xa, i64 na, const double* xb, i64 nb, i64 d, double var, double inv_two_ell2,
                  double* k) {
    for (i64 i = 0; i < na; ++i)
        for (i64 j = 0; j < nb; ++j) {
            double acc = 0.0;
            for (i64 t = 0; t < d; ++t) {
                const double diff = xa[i * d + t] - xb[j * d + t];
                acc = acc + diff * diff;
            }
            k[i * nb + j] = var * exp(-acc * inv_two_ell2);
        }
}

/* one cyclic Jacobi sweep in place; returns rotation count
 *                                                 _core.pyx:135-177 */
i64 or_jacobi_sweep(double* a, double* v, i64 n) {
    i64 rotations = 0;
    for (i64 p = 0; p < n - 1; ++p) {
        for (i64 q = p + 1; q < n; ++q) {
            const double apq = a[p * n + q];
            const double g = 100.0 * fabs(apq);
            if (fabs(a[p * n + p]) + g == fabs(a[p * n + p]) && fabs(a[q * n + q]) + g == fabs(a[q * n + q])) {
                a[p * n + q] = 0.0;
                a[q * n + p] = 0.0;
                continue;
            }
            if (apq == 0.0) continue;
            const double tau = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
            double t;
            if (tau >= 0.0) t = 1.0 / (tau + sqrt(1.0 + tau * tau));
            else t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = t * c;
            for (i64 i = 0; i < n; ++i) {
                const double aip = a[i * n + p], aiq = a[i * n + q];
                a[i * n + p] = c * aip - s * aiq;
                a[i * n + q] = s * aip + c * aiq;
            }
            for (i64 i = 0; i < n; ++i) {
                const double aip = a[p * n + i], aiq = a[q * n + i];
                a[p * n + i] = c * aip - s * aiq;
                a[q * n + i] = s * aip + c * aiq;
            }
            a[p * n + q] = 0.0;
            a[q * n + p] = 0.0;
            for (i64 i = 0; i < n; ++i) {
                const double vp = v[i * n + p], vq = v[i * n + q];
                v[i * n + p] = c * vp - s * vq;
                v[i * n + q] = s * vp + c * vq;
            }
            rotations += 1;
        }
    }
    return rotations;
}
