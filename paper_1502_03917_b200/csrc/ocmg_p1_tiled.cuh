// Tiled structured-P1 kernels for the HBM-bound level operations
// (residual, NE-Jacobi, restriction, prolongation).
//
// Layout: a block is 32 x 8 threads; lane = one column, each thread walks
// kRPT consecutive rows keeping a 3-row x 3-column register window per field,
// so every value is loaded from HBM once (halo rows and columns come from L1).
// Interior kernels cover the class-(3,3) region (3 <= ix, iy <= n1-4) where
// every coefficient is the same: the 14+14 coefficients are passed as kernel
// parameters (constant bank operands, no registers, no table lookups).  The
// width-3 ring of boundary classes is a separate small launch that reuses the
// per-node code of ocmg_p1.cuh.  The arithmetic (sequential sums from 0.0 in
// CSR column order, no FMA) is the same as ocmg_p1.cuh, so results are
// bit-identical to the per-node kernels and to the oracle.
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {

constexpr int kTX = 32, kTY = 8, kRPT = 8;  // block tile: 32 cols x 64 rows
constexpr int kPRPT = 4;  // prolongation: coarse rows per thread (8 fine rows)
constexpr int kRing = 3;                     // boundary classes 0..2, n1-3..n1-1

struct P1Coef28 {
    double c[28];  // A (or W) of class (3,3): [block-row][state 0..6, adj 7..13]
};
struct P1JacCoef {
    double w[28];
    double l[2];
    double tau;
};

// vertex of the ring of width w (rows < w or >= n1-w, else columns < w or
// >= n1-w), enumerated by k in [0, n1^2 - (n1-2w)^2)
__device__ __forceinline__ bool p1_ring_node(int64_t k, int n1, int w, int &ix,
                                             int &iy) {
    const int64_t band = (int64_t)w * n1;
    if (k < 2 * band) {
        const int row = (int)(k / n1);
        ix = (int)(k - (int64_t)row * n1);
        iy = row < w ? row : n1 - 2 * w + row;
        return true;
    }
    k -= 2 * band;
    const int mid = n1 - 2 * w;
    if (k >= (int64_t)mid * 2 * w) return false;
    const int rr = (int)(k / (2 * w)), j = (int)(k - (int64_t)rr * 2 * w);
    iy = w + rr;
    ix = j < w ? j : n1 - 2 * w + j;
    return true;
}

__host__ __device__ __forceinline__ int64_t p1_ring_count(int n1, int w) {
    return (int64_t)n1 * n1 - (int64_t)(n1 - 2 * w) * (n1 - 2 * w);
}

// window value for stencil offset d (CSR order) from rows {below, cur, above}
// x cols {left, own, right}
#define OCMG_W7(w, f)                                                      \
    { w[f][0][0], w[f][0][1], w[f][1][0], w[f][1][1], w[f][1][2], w[f][2][1], \
      w[f][2][2] }

__device__ __forceinline__ double p1_dot14(const double *c, const double (&s)[7],
                                           const double (&a)[7]) {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) acc = __dadd_rn(acc, __dmul_rn(c[d], s[d]));
#pragma unroll
    for (int d = 0; d < 7; ++d) acc = __dadd_rn(acc, __dmul_rn(c[7 + d], a[d]));
    return acc;
}

__device__ __forceinline__ void p1_load_row(const double *__restrict__ p,
                                            double (&o)[3]) {
    o[0] = __ldg(p - 1);
    o[1] = __ldg(p);
    o[2] = __ldg(p + 1);
}

// ---------------------------------------------------------------------------
// residual r = -(A x) + f
// ---------------------------------------------------------------------------
template <int NR>
__device__ __forceinline__ void p1_residual_rows(const P1Coef28 &A, int64_t N,
                                                 int n1, int64_t v0,
                                                 const double *__restrict__ x,
                                                 const double *__restrict__ f,
                                                 double *__restrict__ r,
                                                 int nrows) {
    double w[2][3][3];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        p1_load_row(x + b * N + v0 - n1, w[b][0]);
        p1_load_row(x + b * N + v0, w[b][1]);
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (NR == kRPT || j < nrows) {
            const int64_t v = v0 + (int64_t)j * n1;
#pragma unroll
            for (int b = 0; b < 2; ++b) p1_load_row(x + b * N + v + n1, w[b][2]);
            const double s[7] = OCMG_W7(w, 0);
            const double a[7] = OCMG_W7(w, 1);
            double s0 = -p1_dot14(A.c, s, a);
            double s1 = -p1_dot14(A.c + 14, s, a);
            if (f) {
                s0 = __dadd_rn(s0, __ldg(f + v));
                s1 = __dadd_rn(s1, __ldg(f + N + v));
            }
            r[v] = s0;
            r[N + v] = s1;
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    w[b][0][c] = w[b][1][c];
                    w[b][1][c] = w[b][2][c];
                }
        }
    }
}

__global__ void __launch_bounds__(kTX *kTY)
    k_p1_residual_int(int n1, const __grid_constant__ P1Coef28 A,
                      const double *__restrict__ x, const double *__restrict__ f,
                      double *__restrict__ r, int ylo, int yhi) {
    // interior columns and rows, restricted to the rows [ylo, yhi)
    const int lo = kRing, hi = n1 - 1 - kRing;
    const int rlo = max(lo, ylo), rhi = min(hi, yhi - 1);
    const int ix = lo + blockIdx.x * kTX + threadIdx.x;
    const int iy0 = rlo + (blockIdx.y * kTY + threadIdx.y) * kRPT;
    if (ix > hi || iy0 > rhi) return;
    const int nrows = min(kRPT, rhi - iy0 + 1);
    const int64_t N = (int64_t)n1 * n1, v0 = (int64_t)iy0 * n1 + ix;
    if (nrows == kRPT)
        p1_residual_rows<kRPT>(A, N, n1, v0, x, f, r, nrows);
    else
        p1_residual_rows<kRPT - 1>(A, N, n1, v0, x, f, r, nrows);
}

__global__ void k_p1_residual_ring(int n1, const double *__restrict__ T,
                                   const double *__restrict__ x,
                                   const double *__restrict__ f,
                                   double *__restrict__ r, int ylo, int yhi) {
    int ix, iy;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!p1_ring_node(k, n1, kRing, ix, iy) || iy < ylo || iy >= yhi) return;
    const int64_t N = (int64_t)n1 * n1;
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
    double s0 = -p1_row_dot(q, A, x, N);
    double s1 = -p1_row_dot(q, A + 14, x, N);
    if (f) {
        s0 = __dadd_rn(s0, f[q.v]);
        s1 = __dadd_rn(s1, f[N + q.v]);
    }
    r[q.v] = s0;
    r[N + q.v] = s1;
}

// the whole level, one thread per vertex (small levels: one launch and no
// per-thread row walk); the ring kernel's arithmetic, which the interior
// kernel reproduces bit for bit
__global__ void k_p1_residual_all(int n1, const double *__restrict__ T,
                                  const double *__restrict__ x,
                                  const double *__restrict__ f,
                                  double *__restrict__ r) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    const int64_t N = (int64_t)n1 * n1;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= N) return;
    const int iy = (int)(k / n1), ix = (int)(k - (int64_t)iy * n1);
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
    double s0 = -p1_row_dot(q, A, x, N);
    double s1 = -p1_row_dot(q, A + 14, x, N);
    if (f) {
        s0 = __dadd_rn(s0, f[q.v]);
        s1 = __dadd_rn(s1, f[N + q.v]);
    }
    r[q.v] = s0;
    r[N + q.v] = s1;
}

// ---------------------------------------------------------------------------
// NE-Jacobi phase 1: p = (tau * W r) / L
// ---------------------------------------------------------------------------
template <int NR>
__device__ __forceinline__ void p1_nep_rows(const P1JacCoef &C, int64_t N, int n1,
                                            int64_t v0,
                                            const double *__restrict__ r,
                                            double *__restrict__ p, int nrows) {
    double w[2][3][3];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        p1_load_row(r + b * N + v0 - n1, w[b][0]);
        p1_load_row(r + b * N + v0, w[b][1]);
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (NR == kRPT || j < nrows) {
            const int64_t v = v0 + (int64_t)j * n1;
#pragma unroll
            for (int b = 0; b < 2; ++b) p1_load_row(r + b * N + v + n1, w[b][2]);
            const double s[7] = OCMG_W7(w, 0);
            const double a[7] = OCMG_W7(w, 1);
            p[v] = __ddiv_rn(__dmul_rn(C.tau, p1_dot14(C.w, s, a)), C.l[0]);
            p[N + v] = __ddiv_rn(__dmul_rn(C.tau, p1_dot14(C.w + 14, s, a)), C.l[1]);
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    w[b][0][c] = w[b][1][c];
                    w[b][1][c] = w[b][2][c];
                }
        }
    }
}

__global__ void __launch_bounds__(kTX *kTY, 4)
    k_p1_ne_p_int(int n1, const __grid_constant__ P1JacCoef C,
                  const double *__restrict__ r, double *__restrict__ p, int ylo, int yhi) {
    // interior columns and rows, restricted to the rows [ylo, yhi)
    const int lo = kRing, hi = n1 - 1 - kRing;
    const int rlo = max(lo, ylo), rhi = min(hi, yhi - 1);
    const int ix = lo + blockIdx.x * kTX + threadIdx.x;
    const int iy0 = rlo + (blockIdx.y * kTY + threadIdx.y) * kRPT;
    if (ix > hi || iy0 > rhi) return;
    const int nrows = min(kRPT, rhi - iy0 + 1);
    const int64_t N = (int64_t)n1 * n1, v0 = (int64_t)iy0 * n1 + ix;
    if (nrows == kRPT)
        p1_nep_rows<kRPT>(C, N, n1, v0, r, p, nrows);
    else
        p1_nep_rows<kRPT - 1>(C, N, n1, v0, r, p, nrows);
}

__global__ void k_p1_ne_p_ring(int n1, const double *__restrict__ T, double tau,
                               const double *__restrict__ r,
                               double *__restrict__ p, int ylo, int yhi) {
    int ix, iy;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!p1_ring_node(k, n1, kRing, ix, iy) || iy < ylo || iy >= yhi) return;
    const int64_t N = (int64_t)n1 * n1;
    const P1Node q = p1_node(ix, iy, n1);
    const double *W = T + kP1OffW + q.c * 28;
    const double *L = T + kP1OffL + q.c * 2;
    p[q.v] = __ddiv_rn(__dmul_rn(tau, p1_row_dot(q, W, r, N)), __ldg(L));
    p[N + q.v] = __ddiv_rn(__dmul_rn(tau, p1_row_dot(q, W + 14, r, N)), __ldg(L + 1));
}

// ---------------------------------------------------------------------------
// NE-Jacobi phase 2: x += p; r_j -= sum_i A_ji p_i (CSR order of row j)
// ---------------------------------------------------------------------------
template <int NR, bool FULL>
__device__ __forceinline__ void p1_neapply_rows(const P1Coef28 &A, int64_t N,
                                                int n1, int64_t v0,
                                                const double *__restrict__ p,
                                                double *__restrict__ x,
                                                double *__restrict__ r,
                                                int nrows) {
    // x and r of all rows first: the compiler cannot prove that row j+1's
    // loads miss row j's stores (same arrays), so interleaving them would
    // expose one HBM round trip per row
    double xo[NR][2], ro[NR][2];
#pragma unroll
    for (int j = 0; j < NR; ++j)
        if (FULL || j < nrows)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int64_t i = b * N + v0 + (int64_t)j * n1;
                xo[j][b] = x[i];
                ro[j][b] = r[i];
            }
    double w[2][3][3];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        p1_load_row(p + b * N + v0 - n1, w[b][0]);
        p1_load_row(p + b * N + v0, w[b][1]);
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (FULL || j < nrows) {
            const int64_t v = v0 + (int64_t)j * n1;
#pragma unroll
            for (int b = 0; b < 2; ++b) p1_load_row(p + b * N + v + n1, w[b][2]);
            const double s[7] = OCMG_W7(w, 0);
            const double a[7] = OCMG_W7(w, 1);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int64_t i = b * N + v;
                x[i] = __dadd_rn(xo[j][b], w[b][1][1]);
                double ri = ro[j][b];
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    ri = __dsub_rn(ri, __dmul_rn(A.c[14 * b + d], s[d]));
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    ri = __dsub_rn(ri, __dmul_rn(A.c[14 * b + 7 + d], a[d]));
                r[i] = ri;
            }
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    w[b][0][c] = w[b][1][c];
                    w[b][1][c] = w[b][2][c];
                }
        }
    }
}

__global__ void __launch_bounds__(kTX *kTY, 3)
    k_p1_ne_apply_int(int n1, const __grid_constant__ P1Coef28 A,
                      const double *__restrict__ p, double *__restrict__ x,
                      double *__restrict__ r, int ylo, int yhi) {
    // 4 rows per thread here: the x/r preload of 8 rows cost occupancy
    constexpr int R = kRPT / 2;
    const int lo = kRing, hi = n1 - 1 - kRing;
    const int rlo = max(lo, ylo), rhi = min(hi, yhi - 1);
    const int ix = lo + blockIdx.x * kTX + threadIdx.x;
    const int iy0 = rlo + (blockIdx.y * kTY + threadIdx.y) * R;
    if (ix > hi || iy0 > rhi) return;
    const int nrows = min(R, rhi - iy0 + 1);
    const int64_t N = (int64_t)n1 * n1, v0 = (int64_t)iy0 * n1 + ix;
    if (nrows == R)
        p1_neapply_rows<R, true>(A, N, n1, v0, p, x, r, nrows);
    else
        p1_neapply_rows<R, false>(A, N, n1, v0, p, x, r, nrows);
}

__global__ void k_p1_ne_apply_ring(int n1, const double *__restrict__ T,
                                   const double *__restrict__ p,
                                   double *__restrict__ x,
                                   double *__restrict__ r, int ylo, int yhi) {
    int ix, iy;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!p1_ring_node(k, n1, kRing, ix, iy) || iy < ylo || iy >= yhi) return;
    const int64_t N = (int64_t)n1 * n1;
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int64_t j = b * N + q.v;
        x[j] = __dadd_rn(x[j], p[j]);
        double rj = r[j];
        const double *a = A + 14 * b;
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d]) rj = __dsub_rn(rj, __dmul_rn(__ldg(a + d), p[q.nb[d]]));
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d]) rj = __dsub_rn(rj, __dmul_rn(__ldg(a + 7 + d), p[N + q.nb[d]]));
        r[j] = rj;
    }
}

// ---------------------------------------------------------------------------
// transfers.  Restriction: thread = coarse column, kRPT coarse rows; coarse
// (cx,cy) sums fine (2cx-1,2cy-1) (2cx,2cy-1) (2cx-1,2cy) (2cx,2cy)
// (2cx+1,2cy) (2cx,2cy+1) (2cx+1,2cy+1) (weights 1/2, centre 1), absent
// vertices skipped.  Fine row 2cy+1 is the next coarse row's 2cy'-1.
// ---------------------------------------------------------------------------
template <int RPT>  // coarse rows per thread (kRPT; 1 on small levels)
__global__ void __launch_bounds__(kTX *kTY)
    k_p1_restrict_tiled(int nc1, int n_fields, const double *__restrict__ rf,
                        double *__restrict__ rc, int cylo, int cyhi) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    // coarse rows [cylo, cyhi)
    const int cx = blockIdx.x * kTX + threadIdx.x;
    const int cy0 = cylo + (blockIdx.y * kTY + threadIdx.y) * RPT;
    if (cx >= nc1 || cy0 >= cyhi) return;
    const int nrows = min(RPT, cyhi - cy0);
    const int nf1 = 2 * nc1 - 1;
    const int64_t Nc = (int64_t)nc1 * nc1, Nf = (int64_t)nf1 * nf1;
    const bool l = cx > 0, rr = cx < nc1 - 1;
    const int fx = 2 * cx;
    for (int b = 0; b < n_fields; ++b) {
        const double *f = rf + b * Nf;
        double dl = 0.0, dc = 0.0;  // fine row 2cy-1: cols 2cx-1, 2cx
        if (cy0 > 0) {
            const double *q = f + (int64_t)(2 * cy0 - 1) * nf1 + fx;
            if (l) dl = __ldg(q - 1);
            dc = __ldg(q);
        }
#pragma unroll 4
        for (int j = 0; j < nrows; ++j) {
            const int cy = cy0 + j;
            const double *q = f + (int64_t)(2 * cy) * nf1 + fx;
            const double ml = l ? __ldg(q - 1) : 0.0, mc = __ldg(q),
                         mr = rr ? __ldg(q + 1) : 0.0;
            const bool up = cy < nc1 - 1;
            double ul = 0.0, uc = 0.0, ur = 0.0;  // fine row 2cy+1
            if (up) {
                if (l) ul = __ldg(q + nf1 - 1);
                uc = __ldg(q + nf1);
                if (rr) ur = __ldg(q + nf1 + 1);
            }
            double s = 0.0;
            if (cy > 0) {
                if (l) s = __dadd_rn(s, __dmul_rn(0.5, dl));
                s = __dadd_rn(s, __dmul_rn(0.5, dc));
            }
            if (l) s = __dadd_rn(s, __dmul_rn(0.5, ml));
            s = __dadd_rn(s, mc);
            if (rr) s = __dadd_rn(s, __dmul_rn(0.5, mr));
            if (up) {
                s = __dadd_rn(s, __dmul_rn(0.5, uc));
                if (rr) s = __dadd_rn(s, __dmul_rn(0.5, ur));
            }
            rc[b * Nc + (int64_t)cy * nc1 + cx] = s;
            dl = ul;
            dc = uc;
        }
    }
}

// Prolongation x_f += P c: thread = fine column, 2*kRPT fine rows; even/even
// vertices copy (1.0*c), edge midpoints average their two ends (lower first)
template <bool ALL, int PR>  // ALL: the whole level (no row-range guards); PR coarse rows per thread
__global__ void __launch_bounds__(kTX *kTY, 3)
    k_p1_prolong_add_tiled(int nc1, int n_fields, const double *__restrict__ c,
                           double *__restrict__ xf, int fylo, int fyhi) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    // fine rows [fylo, fyhi), walked as coarse rows [fylo/2, (fyhi+1)/2)
    const int nf1 = 2 * nc1 - 1;
    const int fx = blockIdx.x * kTX + threadIdx.x;
    const int cylo = fylo >> 1, cyhi = min(nc1, (fyhi + 1) >> 1);
    const int cy0 = cylo + (blockIdx.y * kTY + threadIdx.y) * PR;  // coarse rows
    if (fx >= nf1 || cy0 >= cyhi) return;
    const int64_t Nc = (int64_t)nc1 * nc1, Nf = (int64_t)nf1 * nf1;
    const int ox = fx & 1, hx = fx >> 1;
    const int cend = min(cy0 + PR, cyhi);
    for (int b = 0; b < n_fields; ++b) {
        const double *cc = c + b * Nc;
        double *xb = xf + b * Nf;
        // all loads first (the compiler cannot move row j+1's x load above
        // row j's store to the same array): the coarse values a (column hx)
        // and b (hx+1, odd columns) of rows cy0 .. cend, the fine x pairs
        double a[PR + 1], bb[PR + 1], xe[PR], xo[PR];
#pragma unroll
        for (int j = 0; j <= PR; ++j) {
            const int cy = cy0 + j;
            const bool in = cy < nc1 && j <= cend - cy0;
            const double *q = cc + (int64_t)cy * nc1 + hx;
            a[j] = in ? __ldg(q) : 0.0;
            bb[j] = in && ox ? __ldg(q + 1) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PR; ++j) {
            const int cy = cy0 + j;
            const int64_t fv = (int64_t)(2 * cy) * nf1 + fx;
            const bool e = cy < cend && (ALL || (2 * cy >= fylo && 2 * cy < fyhi));
            const bool o = cy < cend && cy + 1 < nc1 &&
                           (ALL || (2 * cy + 1 >= fylo && 2 * cy + 1 < fyhi));
            xe[j] = e ? xb[fv] : 0.0;
            xo[j] = o ? xb[fv + nf1] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PR; ++j) {
            const int cy = cy0 + j;
            if (cy >= cend) break;
            const int64_t fv = (int64_t)(2 * cy) * nf1 + fx;
            // even fine row 2cy: the coarse-row interpolant at this column
            const double lo = ox ? __dadd_rn(__dmul_rn(0.5, a[j]), __dmul_rn(0.5, bb[j]))
                                 : __dmul_rn(1.0, a[j]);
            if (ALL || (2 * cy >= fylo && 2 * cy < fyhi)) xb[fv] = __dadd_rn(xe[j], lo);
            if (cy + 1 < nc1) {
                // odd fine row 2cy+1: (ox=0) avg of (hx,cy),(hx,cy+1);
                // (ox=1) diagonal edge (hx,cy)-(hx+1,cy+1)
                const double mid = ox ? __dadd_rn(__dmul_rn(0.5, a[j]), __dmul_rn(0.5, bb[j + 1]))
                                      : __dadd_rn(__dmul_rn(0.5, a[j]), __dmul_rn(0.5, a[j + 1]));
                if (ALL || (2 * cy + 1 >= fylo && 2 * cy + 1 < fyhi))
                    xb[fv + nf1] = __dadd_rn(xo[j], mid);
            }
        }
    }
}

}  // namespace ocmg
