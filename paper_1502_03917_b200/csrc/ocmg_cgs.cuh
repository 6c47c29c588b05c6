// Collective Gauss-Seidel (CGS) over state/adjoint vertex pairs
// (kernels.collective_sweep, kernels.py:70-96; smoothers.py:288-295;
// SURVEY.md §8(f) rank 1).  Vertex i owns the unknowns (i, i+N): with
// m = M_ii, k = K_ii the local system [[m, k], [k, -m/alpha]] is solved in
// closed form from the residual at the vertex itself,
//     det = -m m / alpha - k k,  s = (-m/alpha ra - k rb) / det,
//     t = (-k ra + m rb) / det,  x_i += s, x_{i+N} += t,
// and both columns of A are scattered into r.
//
// Dependency: a vertex reads only its own residual, which earlier vertices
// change when they are graph neighbours (distance 1).  On the structured P1
// mesh the earlier neighbours of (ix, iy) sit on anti-diagonal ix+iy-1 or
// ix+iy-2, so processing the anti-diagonals in order is the reference's
// order exactly ("reference" mode, 2 n1 - 1 levels).  "multicolour" mode
// runs the distance-1 3-colouring (ix+iy) mod 3 instead (its own smoother).
// Each level / colour is two launches: the 2x2 solves (own residual only),
// then a row gather r_j -= A_ji s_i + A_{j,i+N} t_i over the selected
// neighbours i in increasing index, which is the reference's scatter order
// for every r_j (CSR column order = increasing vertex index).  Reference
// arithmetic throughout (no contraction): bit-identical to the reference.
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {

// vertex (ix, iy) selected by level (sel_mod == 0: ix+iy == sel) or colour
// (sel_mod == 3: (ix+iy) % 3 == sel)
__device__ __forceinline__ bool cgs_sel(int ix, int iy, int sel_mod, int sel) {
    const int l = ix + iy;
    return sel_mod ? (l % sel_mod) == sel : l == sel;
}

// 2x2 solves of the selected vertices; s, t kept in S (2N) for the gather
__global__ void k_p1_cgs_solve(int n1, const double *__restrict__ T, double alpha,
                               int sel_mod, int sel, double *__restrict__ x,
                               const double *__restrict__ r, double *__restrict__ S) {
    pdl_trigger();  // launched with PDL in the per-level loops
    pdl_wait();
    const int64_t N = (int64_t)n1 * n1;
    int ix, iy;
    if (sel_mod) {  // colour: thread per vertex of the colour in row iy
        const int per_row = (n1 + 2) / 3;
        const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        if (k >= (int64_t)per_row * n1) return;
        iy = (int)(k / per_row);
        const int jj = (int)(k - (int64_t)iy * per_row);
        ix = ((sel - iy) % 3 + 3) % 3 + 3 * jj;
        if (ix >= n1) return;
    } else {  // level: thread per vertex of the anti-diagonal
        const int k = blockIdx.x * blockDim.x + threadIdx.x;
        iy = max(0, sel - (n1 - 1)) + k;
        ix = sel - iy;
        if (iy >= n1 || ix < 0) return;
    }
    const int64_t v = (int64_t)iy * n1 + ix;
    const int c = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
    const double m = __ldg(T + kP1OffA + c * 28 + 3);       // M_ii
    const double kk = __ldg(T + kP1OffA + c * 28 + 7 + 3);  // K_ii
    const double det = __dsub_rn(__ddiv_rn(__dmul_rn(-m, m), alpha), __dmul_rn(kk, kk));
    const double ra = r[v], rb = r[N + v];
    const double s =
        __ddiv_rn(__dsub_rn(__dmul_rn(__ddiv_rn(-m, alpha), ra), __dmul_rn(kk, rb)), det);
    const double t = __ddiv_rn(__dadd_rn(__dmul_rn(-kk, ra), __dmul_rn(m, rb)), det);
    x[v] = __dadd_rn(x[v], s);
    x[N + v] = __dadd_rn(x[N + v], t);
    S[v] = s;
    S[N + v] = t;
}

// r_j -= sum over selected neighbours i (increasing index) of
// A_{j,i} s_i then A_{j,i+N} t_i, for both rows of every touched vertex j
__global__ void k_p1_cgs_apply(int n1, const double *__restrict__ T, int sel_mod,
                               int sel, const double *__restrict__ S,
                               double *__restrict__ r) {
    pdl_trigger();  // launched with PDL in the per-level loops
    pdl_wait();
    const int64_t N = (int64_t)n1 * n1;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int ix, iy;
    if (sel_mod) {  // colour: every vertex may have a neighbour of the colour
        if (k >= N) return;
        iy = (int)(k / n1);
        ix = (int)(k - (int64_t)iy * n1);
    } else {  // level L: the vertices on anti-diagonals L-2 .. L+2
        if (k >= 5 * (int64_t)n1) return;
        const int e = (int)(k / n1), t = (int)(k - (int64_t)e * n1);
        const int lj = sel - 2 + e;
        if (lj < 0 || lj > 2 * (n1 - 1)) return;
        iy = max(0, lj - (n1 - 1)) + t;
        ix = lj - iy;
        if (iy >= n1 || ix < 0) return;
    }
    const P1Node q = p1_node(ix, iy, n1);
    bool any = false;
    bool on[7];
    const int dx[7] = {-1, 0, -1, 0, 1, 0, 1}, dy[7] = {-1, -1, 0, 0, 0, 1, 1};
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        on[d] = q.ex[d] && cgs_sel(ix + dx[d], iy + dy[d], sel_mod, sel);
        any |= on[d];
    }
    if (!any) return;
    const double *A = T + kP1OffA + q.c * 28;
#pragma unroll
    for (int b = 0; b < 2; ++b) {  // state row, adjoint row of vertex j
        double rj = r[b * N + q.v];
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (on[d]) {
                rj = __dsub_rn(rj, __dmul_rn(__ldg(A + 14 * b + d), S[q.nb[d]]));
                rj = __dsub_rn(rj, __dmul_rn(__ldg(A + 14 * b + 7 + d), S[N + q.nb[d]]));
            }
        r[b * N + q.v] = rj;
    }
}

// Generic CSR levels (Poisson k <= 2, a few dozen unknowns): the reference
// loop itself, one thread.  Symmetric A: column i = row i.
__global__ void k_csr_cgs_seq(int64_t n_nodes, const int64_t *__restrict__ off,
                              const int32_t *__restrict__ col,
                              const double *__restrict__ val, double alpha,
                              double *__restrict__ x, double *__restrict__ r) {
    if (threadIdx.x || blockIdx.x) return;
    for (int64_t i = 0; i < n_nodes; ++i) {
        const int64_t j = i + n_nodes;
        double m = 0.0, kk = 0.0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t) {
            if (col[t] == i) m = val[t];
            if (col[t] == j) kk = val[t];
        }
        const double det = __dsub_rn(__ddiv_rn(__dmul_rn(-m, m), alpha), __dmul_rn(kk, kk));
        const double ra = r[i], rb = r[j];
        const double s =
            __ddiv_rn(__dsub_rn(__dmul_rn(__ddiv_rn(-m, alpha), ra), __dmul_rn(kk, rb)), det);
        const double t = __ddiv_rn(__dadd_rn(__dmul_rn(-kk, ra), __dmul_rn(m, rb)), det);
        x[i] = __dadd_rn(x[i], s);
        x[j] = __dadd_rn(x[j], t);
        for (int64_t tt = off[i]; tt < off[i + 1]; ++tt)
            r[col[tt]] = __dsub_rn(r[col[tt]], __dmul_rn(val[tt], s));
        for (int64_t tt = off[j]; tt < off[j + 1]; ++tt)
            r[col[tt]] = __dsub_rn(r[col[tt]], __dmul_rn(val[tt], t));
    }
}

}  // namespace ocmg
