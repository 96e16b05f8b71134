/*
 * mrs_oracle.c -- CPU restatement of the reference's hot kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the *checker*: tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline leg may load
 * it; the product (paper_2103_07329_b200/) never does.
 *
 * Each function restates one kernel of the reference plugin
 * (/root/reference/pkg/src/mrsolve/kernels/_ckernels.pyx) with the exact
 * arithmetic order documented there and in kernels/python_ref.py:1-15:
 *   - vectors are (n, m) row-major float64; matrix values float32/float64
 *     widened to double before the multiply;
 *   - every multiply-add is a separately rounded multiply then add
 *     (compiled with -ffp-contract=off; the reference is built without FMA);
 *   - per-(row, column) accumulation runs in CSR entry order.
 * Built by oracle/Makefile with gcc -O2 -ffp-contract=off.
 */
#include <stdint.h>
#include <stddef.h>

enum { ORC_ASSIGN = 0, ORC_ADD = 1, ORC_SUB = 2, ORC_RSUB = 3 };

static inline int64_t col_at(const void* ci, int idx_bytes, int64_t k) {
    switch (idx_bytes) {
    case 1: return ((const uint8_t*)ci)[k];
    case 2: return ((const uint16_t*)ci)[k];
    case 4: return ((const uint32_t*)ci)[k];
    default: return ((const int64_t*)ci)[k];
    }
}

static inline double val_at(const void* v, int val_bytes, int64_t k) {
    return val_bytes == 4 ? (double)((const float*)v)[k] : ((const double*)v)[k];
}

/* _ckernels.pyx:30-57 (csr_spmv): y op= A x, op by mode. */
int orc_csr_spmv(int64_t nrows, const int64_t* row_ptr, const void* col_idx,
                 int idx_bytes, const void* values, int val_bytes,
                 const double* x, int64_t m, double* y, int mode,
                 const double* b) {
    if (mode < 0 || mode > 3) return -1;
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
        double* yi = y + i * m;
        if (mode == ORC_ASSIGN)
            for (int64_t j = 0; j < m; ++j) yi[j] = 0.0;
        else if (mode == ORC_RSUB)
            for (int64_t j = 0; j < m; ++j) yi[j] = b[i * m + j];
        int add = (mode == ORC_ASSIGN || mode == ORC_ADD);
        for (int64_t k = lo; k < hi; ++k) {
            double v = val_at(values, val_bytes, k);
            const double* xc = x + col_at(col_idx, idx_bytes, k) * m;
            if (add)
                for (int64_t j = 0; j < m; ++j) yi[j] += v * xc[j];
            else
                for (int64_t j = 0; j < m; ++j) yi[j] -= v * xc[j];
        }
    }
    return 0;
}

/* _ckernels.pyx:82-89 (axpby): y = b*y + a*x per column. */
void orc_axpby(int64_t n, int64_t m, const double* a, const double* x,
               const double* b, double* y) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j)
            y[i * m + j] = b[j] * y[i * m + j] + a[j] * x[i * m + j];
}

/* _ckernels.pyx:92-99 (add2_scaled): y = (y + a*u) + b*v. */
void orc_add2_scaled(int64_t n, int64_t m, double* y, const double* a,
                     const double* u, const double* b, const double* v) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j)
            y[i * m + j] = y[i * m + j] + a[j] * u[i * m + j] + b[j] * v[i * m + j];
}

/* _ckernels.pyx:102-111 (dot_partial): sequential row-order fold from 0. */
void orc_dot_partial(int64_t n, int64_t m, const double* x, const double* y,
                     double* out) {
    for (int64_t j = 0; j < m; ++j) out[j] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) out[j] += x[i * m + j] * y[i * m + j];
}

/* _ckernels.pyx:114-127 (fused_update_dot). */
void orc_fused_update_dot(int64_t n, int64_t m, const double* a,
                          const double* x, const double* b, double* y,
                          double* out) {
    for (int64_t j = 0; j < m; ++j) out[j] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) {
            double t = b[j] * y[i * m + j] + a[j] * x[i * m + j];
            y[i * m + j] = t;
            out[j] += t * t;
        }
}

/* _ckernels.pyx:130-142 (fused_paired_update). */
void orc_fused_paired_update(int64_t n, int64_t m, double* y1, const double* a,
                             const double* u, const double* b, const double* s,
                             double* y2, const double* c, const double* w) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) {
            double sv = s[i * m + j];
            y1[i * m + j] = y1[i * m + j] + a[j] * u[i * m + j] + b[j] * sv;
            y2[i * m + j] = sv - c[j] * w[i * m + j];
        }
}

/* _ckernels.pyx:145-162 (fused_update_dot2). */
void orc_fused_update_dot2(int64_t n, int64_t m, double* y, const double* u,
                           const double* c, const double* w, const double* z,
                           double* d1, double* d2) {
    for (int64_t j = 0; j < m; ++j) { d1[j] = 0.0; d2[j] = 0.0; }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) {
            double t = u[i * m + j] - c[j] * w[i * m + j];
            y[i * m + j] = t;
            d1[j] += z[i * m + j] * t;
            d2[j] += t * t;
        }
}

/* _ckernels.pyx:60-79 (gs_sweep), kept so the oracle covers every plugin
 * entry point even though the hybrid-GS smoother is not on the device path. */
void orc_gs_sweep(int64_t nrows, const int64_t* row_ptr, const void* col_idx,
                  int idx_bytes, const void* values, int val_bytes,
                  const int64_t* diag_pos, const double* b, const double* c,
                  double* x, int64_t m, int forward) {
    for (int64_t ii = 0; ii < nrows; ++ii) {
        int64_t i = forward ? ii : nrows - 1 - ii;
        int64_t lo = row_ptr[i], hi = row_ptr[i + 1], dp = diag_pos[i];
        double d = val_at(values, val_bytes, dp);
        for (int64_t j = 0; j < m; ++j) {
            double v = b[i * m + j] - c[i * m + j];
            for (int64_t k = lo; k < hi; ++k)
                if (k != dp)
                    v -= val_at(values, val_bytes, k) * x[col_at(col_idx, idx_bytes, k) * m + j];
            x[i * m + j] = v / d;
        }
    }
}
