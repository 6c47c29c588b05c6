/*
 * CPU oracle kernels for the ocmg hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library, and only as the checker or the
 * timed CPU baseline.  The product path never links it.
 *
 * Plain sequential C restatement of the reference's numba kernels and of the
 * scipy CSR matvec the reference reaches through SparseMatrix.matvec.
 * Compiled with -ffp-contract=off so that, like the numba build of the
 * reference (no vfmadd in its asm, SURVEY.md §8(a) parity fact (i)), every
 * multiply and add rounds separately.
 *
 *   orc_csr_matvec   <- sparse.py:152-158 (scipy sparsetools csr_matvec:
 *                       y_i = sum over the row, from 0.0, in column order)
 *   orc_normal_sweep <- kernels.py:17-39 (two-phase NE-Jacobi sweep)
 *   orc_lsgs_sweep   <- kernels.py:43-66 (sequential NE-GS sweep)
 *   orc_collective_sweep <- kernels.py:70-96 (CGS over vertex pairs)
 *
 * All indices int64, values fp64, arrays in the reference's CSR / CSC
 * layout.  Each sweep returns the number of touched matrix entries, as the
 * reference kernels do (kernels.py:25-39, 52-66).
 */
#include <stdint.h>

void orc_csr_matvec(int64_t nrows, const int64_t *off, const int64_t *col,
                    const double *val, const double *x, double *y)
{
    for (int64_t i = 0; i < nrows; ++i) {
        double s = 0.0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t)
            s += val[t] * x[col[t]];
        y[i] = s;
    }
}

/* r <- rhs - A x  in the reference's rounding order: -(A x) + rhs
 * (assembly.py:259-263). rhs may be NULL (then r = -(A x)). */
void orc_residual(int64_t n, const int64_t *off, const int64_t *col,
                  const double *val, const double *x, const double *rhs,
                  double *r)
{
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t)
            s += val[t] * x[col[t]];
        double v = -s;
        if (rhs) v += rhs[i];
        r[i] = v;
    }
}

int64_t orc_normal_sweep(int64_t n,
                         const int64_t *row_off, const int64_t *row_col,
                         const double *row_scaled,
                         const int64_t *col_off, const int64_t *col_row,
                         const double *col_val,
                         const double *weight, double tau,
                         double *x, double *r, double *update)
{
    int64_t ops = 0;
    /* phase one: every correction from the entering residual */
    for (int64_t i = 0; i < n; ++i) {
        double q = 0.0;
        for (int64_t t = row_off[i]; t < row_off[i + 1]; ++t)
            q += row_scaled[t] * r[row_col[t]];
        update[i] = tau * q / weight[i];
        ops += row_off[i + 1] - row_off[i];
    }
    /* phase two: apply, downdate the residual column by column */
    for (int64_t i = 0; i < n; ++i) {
        const double p = update[i];
        x[i] += p;
        for (int64_t t = col_off[i]; t < col_off[i + 1]; ++t)
            r[col_row[t]] -= col_val[t] * p;
        ops += col_off[i + 1] - col_off[i];
    }
    return ops;
}

int64_t orc_lsgs_sweep(int64_t n,
                       const int64_t *row_off, const int64_t *row_col,
                       const double *row_scaled,
                       const int64_t *col_off, const int64_t *col_row,
                       const double *col_val,
                       const double *n_diag, double *x, double *r,
                       int forward)
{
    int64_t ops = 0;
    for (int64_t s = 0; s < n; ++s) {
        const int64_t i = forward ? s : n - 1 - s;
        double q = 0.0;
        for (int64_t t = row_off[i]; t < row_off[i + 1]; ++t)
            q += row_scaled[t] * r[row_col[t]];
        const double p = q / n_diag[i];
        x[i] += p;
        for (int64_t t = col_off[i]; t < col_off[i + 1]; ++t)
            r[col_row[t]] -= col_val[t] * p;
        ops += (row_off[i + 1] - row_off[i]) + (col_off[i + 1] - col_off[i]);
    }
    return ops;
}

/* Collective Gauss-Seidel over state/adjoint vertex pairs (kernels.py:70-96,
 * smoothers.py:288-295): vertex i owns unknowns (i, i + n_nodes); the local
 * 2x2 system [[m, k], [k, -m/alpha]] is solved in closed form with the
 * reference's operation order (no contraction), then both columns are
 * scattered into r in CSC order. */
int64_t orc_collective_sweep(int64_t n_nodes,
                             const int64_t *col_off, const int64_t *col_row,
                             const double *col_val,
                             const double *mass_diag, const double *stiff_diag,
                             double alpha, double *x, double *r)
{
    int64_t ops = 0;
    for (int64_t i = 0; i < n_nodes; ++i) {
        const int64_t j = i + n_nodes;
        const double m = mass_diag[i];
        const double k = stiff_diag[i];
        const double det = -m * m / alpha - k * k;
        const double ra = r[i];
        const double rb = r[j];
        const double s = (-m / alpha * ra - k * rb) / det;
        const double t = (-k * ra + m * rb) / det;
        x[i] += s;
        x[j] += t;
        for (int64_t tt = col_off[i]; tt < col_off[i + 1]; ++tt)
            r[col_row[tt]] -= col_val[tt] * s;
        for (int64_t tt = col_off[j]; tt < col_off[j + 1]; ++tt)
            r[col_row[tt]] -= col_val[tt] * t;
        ops += (col_off[i + 1] - col_off[i]) + (col_off[j + 1] - col_off[j]);
    }
    return ops;
}
