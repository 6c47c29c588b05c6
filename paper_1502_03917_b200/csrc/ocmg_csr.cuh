// Generic CSR kernels (any block operator: Stokes Taylor-Hood, Poisson on
// levels too small for the stencil path).  Every kernel reproduces the
// reference's per-unknown arithmetic exactly: sums start at 0.0 and run in
// CSR column order, multiplies and adds round separately (the library is
// built with --fmad=false; see Makefile), division is IEEE.
//
//   k_csr_residual      <- BlockSystem.residual   assembly.py:259-263
//   k_csr_ne_p          <- normal_sweep phase 1   kernels.py:27-32
//   k_csr_ne_apply      <- normal_sweep phase 2   kernels.py:33-38 (row gather:
//                          r_j receives A_ji p_i in increasing i, exactly the
//                          order of the reference's column scatter)
//   k_csr_gs_rows       <- lsgs_sweep body        kernels.py:57-64, run over the
//                          rows of one dependency level (or one colour)
//   k_csr_spmv(_add)    <- SparseMatrix.matvec    sparse.py:152-158
#pragma once

#include "ocmg_common.cuh"

namespace ocmg {

struct CsrDev {
    int64_t n = 0, ncols = 0, nnz = 0;
    DevBuf<int64_t> off;
    DevBuf<int32_t> col;
    DevBuf<double> val;
};

__global__ void k_csr_residual(int64_t n, const int64_t *__restrict__ off,
                               const int32_t *__restrict__ col,
                               const double *__restrict__ val,
                               const double *__restrict__ x,
                               const double *__restrict__ f,
                               double *__restrict__ r) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        s = __dadd_rn(s, __dmul_rn(val[t], x[col[t]]));
    double v = -s;
    if (f) v = __dadd_rn(v, f[i]);
    r[i] = v;
}

// y = A x (y_i from 0.0 in column order)
__global__ void k_csr_spmv(int64_t n, const int64_t *__restrict__ off,
                           const int32_t *__restrict__ col,
                           const double *__restrict__ val,
                           const double *__restrict__ x,
                           double *__restrict__ y) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        s = __dadd_rn(s, __dmul_rn(val[t], x[col[t]]));
    y[i] = s;
}

// y += A x, the product summed first (x += P.matvec(c), multigrid.py:153)
__global__ void k_csr_spmv_add(int64_t n, const int64_t *__restrict__ off,
                               const int32_t *__restrict__ col,
                               const double *__restrict__ val,
                               const double *__restrict__ x,
                               double *__restrict__ y) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        s = __dadd_rn(s, __dmul_rn(val[t], x[col[t]]));
    y[i] = __dadd_rn(y[i], s);
}

// p_i = (tau * sum_j W_ij r_j) / L_i   (W = row_scaled)
__global__ void k_csr_ne_p(int64_t n, const int64_t *__restrict__ off,
                           const int32_t *__restrict__ col,
                           const double *__restrict__ w,
                           const double *__restrict__ L, double tau,
                           const double *__restrict__ r,
                           double *__restrict__ p) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double q = 0.0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        q = __dadd_rn(q, __dmul_rn(w[t], r[col[t]]));
    p[i] = __ddiv_rn(__dmul_rn(tau, q), L[i]);
}

// x_i += p_i; r_i -= A_ij p_j for j in increasing column order
__global__ void k_csr_ne_apply(int64_t n, const int64_t *__restrict__ off,
                               const int32_t *__restrict__ col,
                               const double *__restrict__ val,
                               const double *__restrict__ p,
                               double *__restrict__ x,
                               double *__restrict__ r) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = __dadd_rn(x[i], p[i]);
    double ri = r[i];
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        ri = __dsub_rn(ri, __dmul_rn(val[t], p[col[t]]));
    r[i] = ri;
}

// ---------------------------------------------------------------------------
// SELL-32 (sliced ELLPACK, slice height 32 = a warp): the rows of a slice
// are padded to the slice's longest row and stored entry-major, so the k-th
// entries of a warp's 32 rows are 32 consecutive words -- coalesced loads
// where the thread-per-row CSR kernels read 32 scattered rows.  Each thread
// still sums its own row in column order and stops at the row's length, so
// the three kernels below are the CSR kernels' arithmetic bit for bit.
// ---------------------------------------------------------------------------
struct SellDev {
    int64_t nslices = 0;
    DevBuf<int64_t> base;   // [nslices + 1] first entry of each slice
    DevBuf<int32_t> len;    // [n] row lengths
    DevBuf<int32_t> col;    // [entries]
    DevBuf<double> val, w;  // A and row_scaled, same layout
};

// slice widths -> bases on the host (tiny), entries scattered on the device
__global__ void k_sell_fill(int64_t n, const int64_t *__restrict__ off,
                            const int32_t *__restrict__ col,
                            const double *__restrict__ val,
                            const double *__restrict__ w,
                            const int64_t *__restrict__ base,
                            int32_t *__restrict__ len, int32_t *__restrict__ scol,
                            double *__restrict__ sval, double *__restrict__ sw) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = off[i], m = off[i + 1] - b;
    len[i] = (int32_t)m;
    const int64_t dst = base[i >> 5] + (i & 31);
    for (int64_t k = 0; k < m; ++k) {
        scol[dst + 32 * k] = col[b + k];
        sval[dst + 32 * k] = val[b + k];
        sw[dst + 32 * k] = w[b + k];
    }
}

#define OCMG_SELL_ROW(i, t, k, m)                                             \
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;       \
    if (i >= n) return;                                                      \
    const int64_t t##0 = base[i >> 5] + (i & 31);                            \
    const int m = len[i];

__global__ void k_sell_residual(int64_t n, const int64_t *__restrict__ base,
                                const int32_t *__restrict__ len,
                                const int32_t *__restrict__ col,
                                const double *__restrict__ val,
                                const double *__restrict__ x,
                                const double *__restrict__ f,
                                double *__restrict__ r) {
    OCMG_SELL_ROW(i, t, k, m)
    double s = 0.0;
    for (int k = 0; k < m; ++k) {
        const int64_t t = t0 + 32 * k;
        s = __dadd_rn(s, __dmul_rn(val[t], x[col[t]]));
    }
    double v = -s;
    if (f) v = __dadd_rn(v, f[i]);
    r[i] = v;
}

__global__ void k_sell_ne_p(int64_t n, const int64_t *__restrict__ base,
                            const int32_t *__restrict__ len,
                            const int32_t *__restrict__ col,
                            const double *__restrict__ w,
                            const double *__restrict__ L, double tau,
                            const double *__restrict__ r,
                            double *__restrict__ p) {
    OCMG_SELL_ROW(i, t, k, m)
    double q = 0.0;
    for (int k = 0; k < m; ++k) {
        const int64_t t = t0 + 32 * k;
        q = __dadd_rn(q, __dmul_rn(w[t], r[col[t]]));
    }
    p[i] = __ddiv_rn(__dmul_rn(tau, q), L[i]);
}

__global__ void k_sell_ne_apply(int64_t n, const int64_t *__restrict__ base,
                                const int32_t *__restrict__ len,
                                const int32_t *__restrict__ col,
                                const double *__restrict__ val,
                                const double *__restrict__ p,
                                double *__restrict__ x,
                                double *__restrict__ r) {
    OCMG_SELL_ROW(i, t, k, m)
    x[i] = __dadd_rn(x[i], p[i]);
    double ri = r[i];
    for (int k = 0; k < m; ++k) {
        const int64_t t = t0 + 32 * k;
        ri = __dsub_rn(ri, __dmul_rn(val[t], p[col[t]]));
    }
    r[i] = ri;
}
#undef OCMG_SELL_ROW

// One dependency level (or colour) of the sequential NE-GS sweep: the rows
// in `rows` are pairwise at graph distance >= 3, so their updates commute
// and every r_j still receives its updates in index order.  A is symmetric
// (checked at level creation), so column i of A is row i.
__device__ __forceinline__ void csr_gs_row(int32_t i, const int64_t *__restrict__ off,
                                           const int32_t *__restrict__ col,
                                           const double *__restrict__ val,
                                           const double *__restrict__ w,
                                           const double *__restrict__ ndiag,
                                           double *__restrict__ x,
                                           double *__restrict__ r) {
    const int64_t b = off[i], e = off[i + 1];
    double q = 0.0;
    for (int64_t t = b; t < e; ++t)
        q = __dadd_rn(q, __dmul_rn(w[t], r[col[t]]));
    const double p = __ddiv_rn(q, ndiag[i]);
    x[i] = __dadd_rn(x[i], p);
    // the columns of a row are distinct, so a batch of loads may precede its
    // stores (one-at-a-time read-modify-writes serialize on L2 latency)
    constexpr int kB = 8;
    for (int64_t t0 = b; t0 < e; t0 += kB) {
        double rv[kB];
        int32_t jv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (t0 + u < e) {
                jv[u] = col[t0 + u];
                rv[u] = r[jv[u]];
            }
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (t0 + u < e) r[jv[u]] = __dsub_rn(rv[u], __dmul_rn(val[t0 + u], p));
    }
}

__global__ void k_csr_gs_rows(int cnt, const int32_t *__restrict__ rows,
                              const int64_t *__restrict__ off,
                              const int32_t *__restrict__ col,
                              const double *__restrict__ val,
                              const double *__restrict__ w,
                              const double *__restrict__ ndiag,
                              double *__restrict__ x,
                              double *__restrict__ r) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    csr_gs_row(rows[k], off, col, val, w, ndiag, x, r);
}

// The same row update with one warp per row (the "wavefront" mode on
// generic levels: reference order, FMA arithmetic and a tree-summed dot
// product, held to 1e-12 like the structured wavefront sweep): lanes gather
// the row in parallel, a butterfly sums it, lanes scatter in parallel.  The
// thread-per-row form serializes a ~38-term chain and the scatter's
// read-modify-writes (Stokes rows).
__global__ void k_csr_gs_rows_warp(int cnt, const int32_t *__restrict__ rows,
                                   const int64_t *__restrict__ off,
                                   const int32_t *__restrict__ col,
                                   const double *__restrict__ val,
                                   const double *__restrict__ w,
                                   const double *__restrict__ ndiag,
                                   double *__restrict__ x, double *__restrict__ r) {
    const int wid = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    pdl_trigger();  // the next level may start launching now
    if (wid >= cnt) return;
    // the row's structure does not depend on the previous level; r and x do
    const int32_t i = rows[wid];
    const int64_t b = off[i], e = off[i + 1];
    pdl_wait();
    double q = 0.0;
    for (int64_t t = b + lane; t < e; t += 32) q = fma(w[t], r[col[t]], q);
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const double p = q / ndiag[i];
    if (lane == 0) x[i] += p;
    for (int64_t t = b + lane; t < e; t += 32) {
        const int32_t j = col[t];
        r[j] = fma(-val[t], p, r[j]);
    }
}

// grouped SELL-32 (a schedule's groups in slices of 32 rows, see
// build_group_sell): fill, and one group of the NE-GS sweep with csr_gs_row's
// arithmetic (bit-identical), matrix loads coalesced over a slice
__global__ void k_gsell_fill(int64_t nslots, const int32_t *__restrict__ srow,
                             const int64_t *__restrict__ base,
                             const int64_t *__restrict__ off,
                             const int32_t *__restrict__ col,
                             const double *__restrict__ val,
                             const double *__restrict__ w, int32_t *__restrict__ slen,
                             int32_t *__restrict__ scol, double *__restrict__ sval,
                             double *__restrict__ sw) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nslots) return;
    const int32_t i = srow[k];
    if (i < 0) {
        slen[k] = 0;
        return;
    }
    const int64_t b = off[i], m = off[i + 1] - b;
    slen[k] = (int32_t)m;
    const int64_t dst = base[k >> 5] + (k & 31);
    for (int64_t t = 0; t < m; ++t) {
        scol[dst + 32 * t] = col[b + t];
        sval[dst + 32 * t] = val[b + t];
        sw[dst + 32 * t] = w[b + t];
    }
}

__global__ void k_gsell_gs_rows(int64_t nslots, int64_t slice0,
                                const int32_t *__restrict__ srow,
                                const int64_t *__restrict__ base,
                                const int32_t *__restrict__ slen,
                                const int32_t *__restrict__ col,
                                const double *__restrict__ val,
                                const double *__restrict__ w,
                                const double *__restrict__ ndiag,
                                double *__restrict__ x, double *__restrict__ r) {
    const int64_t k = slice0 * 32 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= slice0 * 32 + nslots) return;
    const int32_t i = srow[k];
    if (i < 0) return;
    const int m = slen[k];
    const int64_t t0 = base[k >> 5] + (k & 31);
    double q = 0.0;
    for (int t = 0; t < m; ++t) {
        const int64_t e = t0 + 32 * t;
        q = __dadd_rn(q, __dmul_rn(w[e], r[col[e]]));
    }
    const double p = __ddiv_rn(q, ndiag[i]);
    x[i] = __dadd_rn(x[i], p);
    constexpr int kB = 8;
    for (int tb = 0; tb < m; tb += kB) {
        double rv[kB];
        int32_t jv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (tb + u < m) {
                jv[u] = col[t0 + 32 * (tb + u)];
                rv[u] = r[jv[u]];
            }
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (tb + u < m) r[jv[u]] = __dsub_rn(rv[u], __dmul_rn(val[t0 + 32 * (tb + u)], p));
    }
}

// Whole sweep of a small level in one CTA: the groups (dependency levels or
// colours) in order, __syncthreads between them (one launch instead of one
// per group -- the coarse levels of a W-cycle are visited thousands of times)
constexpr int64_t kCsrSmallN = 8192;

// The same one-CTA sweep with the level staged in shared memory (rows,
// columns, values, row_scaled, n_diag, x and r): the row updates of a group
// are chains of dependent loads, and from global memory every link was an
// L2 round trip (the W-cycle visits these bottom levels thousands of times
// per cycle).  Identical arithmetic, so bit-identical to the global form.
inline size_t csr_small_smem(int64_t n, int64_t nnz, int64_t ng) {
    return (size_t)(nnz * (8 + 8 + 4) + n * (8 + 8 + 8 + 4) + (ng + 1) * 4 + (n + 1) * 4 + 64);
}
constexpr size_t kCsrSmallSmemMax = 200 * 1024;

// Exact order (wavefront mode) on a tiny generic level (Poisson L2: 50
// unknowns whose dependency DAG is nearly a chain): ONE warp, the level in
// shared memory, the rows of the schedule one after another with
// k_csr_gs_rows_warp's arithmetic (lanes over a row's entries, butterfly sum,
// FMA; the 1e-12 mode).  A CTA barrier per dependency level cost more than
// the row.
constexpr int64_t kCsrWarpN = 256;

// Tiny generic levels as dense maps.  A sweep in a fixed order is linear in
// the entering (x, r): x += S r, r <- T r.  For levels of at most kDenseN
// unknowns (Poisson L2: 50, Stokes L2: 246) S and T are built once at level
// creation by running the sequential sweep (k_csr_gs_sched_smem, the
// reference's arithmetic) on the n unit residuals in one batched launch, and
// a sweep becomes two dense products (rounding differs from the sequential
// sweep by ~1e-16 per entry: the exact mode's 1e-12 bar, and the multicolour
// mode's own smoother).  The L2 sweeps were ~110 ms of an exact L12 W-cycle
// at coarsest L1 (4096 sweeps of a 50-row DAG that is nearly a chain).
// Stored transposed: ST[j * n + i] = S[i][j], so thread i reads coalesced.
constexpr int64_t kDenseN = 256;
__global__ void __launch_bounds__(256)
    k_dense_sweep(int n, const double *__restrict__ ST, const double *__restrict__ TT,
                  double *__restrict__ x, double *__restrict__ r) {
    __shared__ double rs[kDenseN];
    for (int j = threadIdx.x; j < n; j += blockDim.x) rs[j] = r[j];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double ds = 0.0, rt = 0.0;
        for (int j = 0; j < n; ++j) {
            const double rj = rs[j];
            ds = fma(__ldg(ST + (int64_t)j * n + i), rj, ds);
            rt = fma(__ldg(TT + (int64_t)j * n + i), rj, rt);
        }
        x[i] += ds;
        r[i] = rt;
    }
}
// unit residuals for the batched build: R[b * n + i] = (i == b), X = 0
__global__ void k_dense_unit(int n, double *X, double *R) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n * n) {
        X[t] = 0.0;
        R[t] = (t / n == t % n) ? 1.0 : 0.0;
    }
}
__global__ void __launch_bounds__(32)
    k_csr_gs_warp_small(int ngroups, const int64_t *__restrict__ goff_g,
                        const int32_t *__restrict__ rows_g, int reverse, int n,
                        const int64_t *__restrict__ off_g, const int32_t *__restrict__ col_g,
                        const double *__restrict__ val_g, const double *__restrict__ w_g,
                        const double *__restrict__ nd_g, double *__restrict__ x_g,
                        double *__restrict__ r_g) {
    extern __shared__ __align__(16) double smc[];
    const int lane = threadIdx.x;
    const int nnz = (int)off_g[n];
    double *val = smc, *w = val + nnz, *nd = w + nnz, *x = nd + n, *r = x + n;
    int *col = reinterpret_cast<int *>(r + n), *off = col + nnz, *rows = off + n + 1,
        *goff = rows + n;
    // staging: every load of a pass in flight at once (a dependent load per
    // group of the schedule cost ~20 us at L2)
#pragma unroll 4
    for (int t = lane; t < nnz; t += 32) {
        val[t] = val_g[t];
        w[t] = w_g[t];
        col[t] = col_g[t];
    }
#pragma unroll 4
    for (int i = lane; i < n; i += 32) {
        nd[i] = nd_g[i];
        x[i] = x_g[i];
        r[i] = r_g[i];
        rows[i] = rows_g[i];
    }
    for (int i = lane; i <= n; i += 32) off[i] = (int)off_g[i];
    for (int g = lane; g <= ngroups; g += 32) goff[g] = (int)goff_g[g];
    __syncwarp();
    // rows in schedule order: groups forward (or reversed for a reverse sweep)
    const int m = goff[ngroups];
    for (int k0 = 0; k0 < m; ++k0) {
        int k = k0;
        if (reverse) {  // k0-th row of the reversed group order
            int g = 0, acc = 0;
            for (g = ngroups - 1; g >= 0; --g) {
                const int len = goff[g + 1] - goff[g];
                if (k0 < acc + len) break;
                acc += len;
            }
            k = goff[g] + (k0 - acc);
        }
        const int i = rows[k], b = off[i], e = off[i + 1];
        double q = 0.0;
        for (int t = b + lane; t < e; t += 32) q = fma(w[t], r[col[t]], q);
#pragma unroll
        for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        const double p = q / nd[i];
        if (lane == 0) x[i] += p;
        for (int t = b + lane; t < e; t += 32) {
            const int j = col[t];
            r[j] = fma(-val[t], p, r[j]);
        }
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) {
        x_g[i] = x[i];
        r_g[i] = r[i];
    }
}

__global__ void __launch_bounds__(1024)
    k_csr_gs_sched_smem(int ngroups, const int64_t *__restrict__ goff_g,
                        const int32_t *__restrict__ rows_g, int reverse, int n,
                        const int64_t *__restrict__ off_g, const int32_t *__restrict__ col_g,
                        const double *__restrict__ val_g, const double *__restrict__ w_g,
                        const double *__restrict__ nd_g, double *__restrict__ x_g,
                        double *__restrict__ r_g, int64_t batch = 0) {
    extern __shared__ __align__(16) double smc[];
    const int nnz = (int)off_g[n];
    double *val = smc, *w = val + nnz, *nd = w + nnz, *x = nd + n, *r = x + n;
    x_g += blockIdx.x * batch;  // batched: one independent (x, r) per block
    r_g += blockIdx.x * batch;
    int *col = reinterpret_cast<int *>(r + n), *off = col + nnz, *rows = off + n + 1,
        *goff = rows + n;
#pragma unroll 4
    for (int t = threadIdx.x; t < nnz; t += blockDim.x) {
        val[t] = val_g[t];
        w[t] = w_g[t];
        col[t] = col_g[t];
    }
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        nd[i] = nd_g[i];
        x[i] = x_g[i];
        r[i] = r_g[i];
        rows[i] = rows_g[i];
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x) off[i] = (int)off_g[i];
    for (int g = threadIdx.x; g <= ngroups; g += blockDim.x) goff[g] = (int)goff_g[g];
    __syncthreads();
    for (int g = 0; g < ngroups; ++g) {
        const int l = reverse ? ngroups - 1 - g : g;
        for (int k = goff[l] + threadIdx.x; k < goff[l + 1]; k += blockDim.x) {
            const int i = rows[k];
            const int b = off[i], e = off[i + 1];
            double q = 0.0;
            for (int t = b; t < e; ++t) q = __dadd_rn(q, __dmul_rn(w[t], r[col[t]]));
            const double p = __ddiv_rn(q, nd[i]);
            x[i] = __dadd_rn(x[i], p);
            // a row's columns are distinct: batches of loads before their
            // stores (one read-modify-write at a time serialised on the
            // shared-memory latency, 1.5 us per dependency level at L2)
            constexpr int kB = 8;
            for (int t0 = b; t0 < e; t0 += kB) {
                double rv[kB];
                int jv[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (t0 + u < e) {
                        jv[u] = col[t0 + u];
                        rv[u] = r[jv[u]];
                    }
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (t0 + u < e) r[jv[u]] = __dsub_rn(rv[u], __dmul_rn(val[t0 + u], p));
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        x_g[i] = x[i];
        r_g[i] = r[i];
    }
}

__global__ void __launch_bounds__(1024)
    k_csr_gs_sched_small(int ngroups, const int64_t *__restrict__ goff,
                         const int32_t *__restrict__ rows, int reverse,
                         const int64_t *__restrict__ off,
                         const int32_t *__restrict__ col,
                         const double *__restrict__ val,
                         const double *__restrict__ w,
                         const double *__restrict__ ndiag,
                         double *__restrict__ x, double *__restrict__ r) {
    for (int g = 0; g < ngroups; ++g) {
        const int l = reverse ? ngroups - 1 - g : g;
        const int lo = (int)goff[l], hi = (int)goff[l + 1];
        for (int k = lo + threadIdx.x; k < hi; k += blockDim.x)
            csr_gs_row(rows[k], off, col, val, w, ndiag, x, r);
        __syncthreads();
    }
}

// setup helpers -------------------------------------------------------------

// W_t = A_t / L_col(t)
__global__ void k_csr_row_scaled(int64_t nnz, const int32_t *__restrict__ col,
                                 const double *__restrict__ val,
                                 const double *__restrict__ L,
                                 double *__restrict__ w) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nnz) w[t] = __ddiv_rn(val[t], L[col[t]]);
}

// n_diag_i = sum_t A_t * W_t, sequential in row order from 0.0
// (np.add.at over the CSR entries, smoothers.py:208-212)
__global__ void k_csr_ndiag(int64_t n, const int64_t *__restrict__ off,
                            const double *__restrict__ val,
                            const double *__restrict__ w,
                            double *__restrict__ nd) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
        s = __dadd_rn(s, __dmul_rn(val[t], w[t]));
    nd[i] = s;
}

}  // namespace ocmg
