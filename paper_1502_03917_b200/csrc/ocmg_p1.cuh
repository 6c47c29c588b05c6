// Structured P1 (Poisson control) kernels.
//
// Level k holds N = n1*n1 vertices (n1 = 2^k+1), x fastest (mesh.py:146-147);
// the block vector is [state(N), adjoint(N)] (FieldLayout, assembly.py:284).
// A = [[M, K], [K, -M/alpha]] (assembly.py:274-277) is a 7-point stencil per
// block with offsets, in CSR column order,
//     d = 0:(-1,-1) 1:(0,-1) 2:(-1,0) 3:(0,0) 4:(1,0) 5:(0,1) 6:(1,1).
// Coefficients depend only on a node's position class: per axis
//     0,1,2 for i = 0,1,2;  3 for 3 <= i <= n1-4;  4,5,6 for n1-3, n1-2, n1-1,
// 49 classes in all (needs n1 >= 7, i.e. k >= 3).  That resolution is what
// row_scaled (A_ij / L_j) and n_diag need (they see the row class of every
// neighbour).  The tables are built on the host from the reference's own
// assembly rules and are bit-identical to the assembled CSR (see
// paper_1502_03917_b200/assembly.py: p1_class_tables).
//
// Table layout (doubles), class c = 7*cls(iy) + cls(ix):
//   A [49][2][14]  row coefficients of block-row b (0 state, 1 adjoint);
//                  entries 0..6 multiply state-field neighbours d=0..6,
//                  7..13 adjoint-field neighbours; 0 where absent
//   W [49][2][14]  row_scaled = A_ij / L_j     (smoothers.py:204)
//   L [49][2]      norm_diag                   (assembly.py:278-286)
//   ND[49][2]      n_diag                      (smoothers.py:208-212)
#pragma once

#include "ocmg_common.cuh"

namespace ocmg {

constexpr int kP1Classes = 49;
constexpr int kP1OffA = 0;
constexpr int kP1OffW = kP1OffA + kP1Classes * 28;
constexpr int kP1OffL = kP1OffW + kP1Classes * 28;
constexpr int kP1OffND = kP1OffL + kP1Classes * 2;
constexpr int kP1TableDoubles = kP1OffND + kP1Classes * 2;

__device__ __forceinline__ int p1_axis_class(int i, int n1) {
    if (i < 3) return i;
    if (i > n1 - 4) return 6 - (n1 - 1 - i);
    return 3;
}

struct P1Node {
    int ix, iy, c;
    int64_t v;  // vertex index iy*n1+ix
    bool ex[7];
    int64_t nb[7];
};

__device__ __forceinline__ P1Node p1_node(int ix, int iy, int n1) {
    P1Node q;
    q.ix = ix;
    q.iy = iy;
    q.c = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
    q.v = (int64_t)iy * n1 + ix;
    const bool l = ix > 0, rr = ix < n1 - 1, dn = iy > 0, up = iy < n1 - 1;
    q.ex[0] = l && dn;  q.nb[0] = q.v - n1 - 1;
    q.ex[1] = dn;       q.nb[1] = q.v - n1;
    q.ex[2] = l;        q.nb[2] = q.v - 1;
    q.ex[3] = true;     q.nb[3] = q.v;
    q.ex[4] = rr;       q.nb[4] = q.v + 1;
    q.ex[5] = up;       q.nb[5] = q.v + n1;
    q.ex[6] = rr && up; q.nb[6] = q.v + n1 + 1;
    return q;
}

// sum over one block-row: 7 state-field entries then 7 adjoint-field
// entries, sequential from 0.0 (CSR order), absent neighbours skipped
__device__ __forceinline__ double p1_row_dot(const P1Node &q,
                                             const double *__restrict__ coef,
                                             const double *__restrict__ v,
                                             int64_t N) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d)
        if (q.ex[d]) s = __dadd_rn(s, __dmul_rn(__ldg(coef + d), v[q.nb[d]]));
#pragma unroll
    for (int d = 0; d < 7; ++d)
        if (q.ex[d])
            s = __dadd_rn(s, __dmul_rn(__ldg(coef + 7 + d), v[N + q.nb[d]]));
    return s;
}

// r = -(A x) + f    (assembly.py:259-263)
__global__ void k_p1_residual(int n1, const double *__restrict__ T,
                              const double *__restrict__ x,
                              const double *__restrict__ f,
                              double *__restrict__ r) {
    const int64_t N = (int64_t)n1 * n1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int iy = (int)(v / n1), ix = (int)(v - (int64_t)iy * n1);
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
    double s0 = -p1_row_dot(q, A, x, N);
    double s1 = -p1_row_dot(q, A + 14, x, N);
    if (f) {
        s0 = __dadd_rn(s0, f[v]);
        s1 = __dadd_rn(s1, f[N + v]);
    }
    r[v] = s0;
    r[N + v] = s1;
}

// NE-Jacobi phase 1: p = (tau * W r) / L   (kernels.py:27-32)
__global__ void k_p1_ne_p(int n1, const double *__restrict__ T, double tau,
                          const double *__restrict__ r,
                          double *__restrict__ p) {
    const int64_t N = (int64_t)n1 * n1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int iy = (int)(v / n1), ix = (int)(v - (int64_t)iy * n1);
    const P1Node q = p1_node(ix, iy, n1);
    const double *W = T + kP1OffW + q.c * 28;
    const double *L = T + kP1OffL + q.c * 2;
    p[v] = __ddiv_rn(__dmul_rn(tau, p1_row_dot(q, W, r, N)), __ldg(L));
    p[N + v] = __ddiv_rn(__dmul_rn(tau, p1_row_dot(q, W + 14, r, N)),
                         __ldg(L + 1));
}

// NE-Jacobi phase 2 as a row gather (kernels.py:33-38): x += p; r_j -= A_ji
// p_i in increasing i, i.e. CSR order of row j
__global__ void k_p1_ne_apply(int n1, const double *__restrict__ T,
                              const double *__restrict__ p,
                              double *__restrict__ x,
                              double *__restrict__ r) {
    const int64_t N = (int64_t)n1 * n1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int iy = (int)(v / n1), ix = (int)(v - (int64_t)iy * n1);
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int64_t j = b * N + v;
        x[j] = __dadd_rn(x[j], p[j]);
        double rj = r[j];
        const double *a = A + 14 * b;
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d]) rj = __dsub_rn(rj, __dmul_rn(__ldg(a + d), p[q.nb[d]]));
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d])
                rj = __dsub_rn(rj, __dmul_rn(__ldg(a + 7 + d), p[N + q.nb[d]]));
        r[j] = rj;
    }
}

// One unknown of the sequential NE-GS sweep (kernels.py:57-64) in the
// reference's arithmetic.  Column i of A equals row i (A is symmetric
// bitwise: every off-diagonal entry sums the same one or two element
// contributions from both sides).
__device__ __forceinline__ void p1_gs_unknown(int field, int ix, int iy,
                                              int n1,
                                              const double *__restrict__ T,
                                              double *__restrict__ x,
                                              double *__restrict__ r) {
    const int64_t N = (int64_t)n1 * n1;
    const P1Node q = p1_node(ix, iy, n1);
    const double *W = T + kP1OffW + q.c * 28 + 14 * field;
    const double *A = T + kP1OffA + q.c * 28 + 14 * field;
    const double nd = __ldg(T + kP1OffND + q.c * 2 + field);
    const double p = __ddiv_rn(p1_row_dot(q, W, r, N), nd);
    const int64_t i = field * N + q.v;
    x[i] = __dadd_rn(x[i], p);
#pragma unroll
    for (int d = 0; d < 7; ++d)
        if (q.ex[d]) {
            const int64_t j = q.nb[d];
            r[j] = __dsub_rn(r[j], __dmul_rn(__ldg(A + d), p));
            r[N + j] = __dsub_rn(r[N + j], __dmul_rn(__ldg(A + 7 + d), p));
        }
}

// All unknowns of dependency level t.  Forward order: state vertex (ix,iy)
// sits at level ix + 2 iy, adjoint vertex at ix + 2 iy + 7 (depth 3*2^k+8;
// SURVEY.md §8(a)).  Backward order is the point reflection of that with the
// fields swapped.
__global__ void k_p1_gs_level(int n1, const double *__restrict__ T, int t,
                              int forward, double *__restrict__ x,
                              double *__restrict__ r) {
    pdl_trigger();  // launched with PDL in the per-level loops
    pdl_wait();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 2 * n1) return;
    const int field = k >= n1 ? 1 : 0;
    const int row = k - field * n1;
    int ix, iy;
    if (forward) {
        const int lev = field ? t - 7 : t;
        iy = row;
        ix = lev - 2 * iy;
    } else {
        const int lev = field ? t : t - 7;
        const int iyr = row;
        const int ixr = lev - 2 * iyr;
        ix = n1 - 1 - ixr;
        iy = n1 - 1 - iyr;
    }
    if (ix < 0 || ix >= n1 || iy < 0 || iy >= n1) return;
    p1_gs_unknown(field, ix, iy, n1, T, x, r);
}

// The whole reference-order sweep of a small level in one CTA: x, r and the
// class tables are staged in shared memory (cp.async), the 3(n1-1)+8
// dependency levels are separated by __syncthreads instead of kernel
// launches, and the threads are packed onto each level's unknowns (the order
// of k_p1_gs_level).  FAST = false: the arithmetic of p1_gs_unknown, so
// bit-identical to the reference sweep (reference mode).  FAST = true (the
// wavefront mode, checked at 1e-12): two FMA chains and a reciprocal
// multiply, as in p1_mc_vertex, which shortens a level's dependent chain.
// The scatter reuses the gathered residual (no other unknown of the level
// touches it).  A level costs ~0.4 us (one warp's dependent chain and a
// barrier) where a launch per level, or the banded wavefront kernel, costs
// 0.7-1.7 us.
constexpr int kGsSmallMaxN1 = 65;
constexpr int kGsSmallThreads = 128;  // 2 * 32 * ceil(((n1 + 1) / 2) / 32)
inline size_t gs_small_smem(int n1) {
    return (4 * (size_t)n1 * n1 + kP1TableDoubles) * sizeof(double);
}

__device__ __forceinline__ void gs_cp16(double *dst, const double *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

template <bool FAST>
__global__ void __launch_bounds__(kGsSmallThreads, 1)
    k_p1_gs_small(int n1, const double *__restrict__ T, int forward,
                  double *__restrict__ x, double *__restrict__ r, int64_t bstride) {
    extern __shared__ __align__(16) double gs_sm[];
    const int N = n1 * n1;
    // independent problems per CTA (the dense-map build sweeps unit
    // residuals: CTA j works on x + j * bstride, r + j * bstride)
    x += blockIdx.x * bstride;
    r += blockIdx.x * bstride;
    double *sr = gs_sm, *sx = gs_sm + 2 * N, *sT = gs_sm + 4 * N;
    // 2N doubles per array: n1 odd => N odd, 2N even, 16-byte chunks
    for (int i = 2 * threadIdx.x; i < 2 * N; i += 2 * blockDim.x) {
        gs_cp16(sr + i, r + i);
        gs_cp16(sx + i, x + i);
    }
    static_assert(kP1TableDoubles % 2 == 0, "table size");
    for (int i = 2 * threadIdx.x; i < kP1TableDoubles; i += 2 * blockDim.x)
        gs_cp16(sT + i, T + i);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int depth = 3 * (n1 - 1) + 8;
    // threads [0, P) take the leading field's unknowns of a level (diagonal
    // ix + 2 iy = t in the sweep's own frame), [P, 2P) the trailing field's
    // (t - 7), packed in row order so idle warps skip the level
    const int P = blockDim.x / 2, k = threadIdx.x;
    const bool lead = k < P;
    const int idx = lead ? k : k - P;
    const int field = lead == (forward != 0) ? 0 : 1;
    for (int t = 0; t < depth; ++t) {
        const int lev = lead ? t : t - 7;
        const int vy = (lev > n1 - 1 ? (lev - n1 + 2) / 2 : 0) + idx, vx = lev - 2 * vy;
        const int ix = forward ? vx : n1 - 1 - vx, iy = forward ? vy : n1 - 1 - vy;
        if (lev >= 0 && vx >= 0 && vy < n1) {
            const int c = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
            const int v = iy * n1 + ix;
            const bool l = ix > 0, rr = ix < n1 - 1, dn = iy > 0, up = iy < n1 - 1;
            const bool ex[7] = {l && dn, dn, l, true, rr, up, rr && up};
            const int nb[7] = {v - n1 - 1, v - n1, v - 1, v, v + 1, v + n1, v + n1 + 1};
            double g[14];
#pragma unroll
            for (int d = 0; d < 7; ++d) {
                g[d] = ex[d] ? sr[nb[d]] : 0.0;
                g[7 + d] = ex[d] ? sr[N + nb[d]] : 0.0;
            }
            const double *W = sT + kP1OffW + c * 28 + 14 * field;
            const double *A = sT + kP1OffA + c * 28 + 14 * field;
            double s = 0.0;
            if (FAST) {  // two FMA chains (the multicolour formula)
                double s1 = 0.0;
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) {
                        s = __fma_rn(W[d], g[d], s);
                        s1 = __fma_rn(W[7 + d], g[7 + d], s1);
                    }
                s = __dadd_rn(s, s1);
            } else {
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) s = __dadd_rn(s, __dmul_rn(W[d], g[d]));
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) s = __dadd_rn(s, __dmul_rn(W[7 + d], g[7 + d]));
            }
            // every shared load before the first store (sr, sx and sT share
            // one array, so the compiler would not hoist them past a store)
            double a[14];
#pragma unroll
            for (int e = 0; e < 14; ++e) a[e] = A[e];
            const int i = field * N + v;
            const double xi = sx[i];
            const double nd = sT[kP1OffND + c * 2 + field];
            const double p = FAST ? __dmul_rn(s, __drcp_rn(nd)) : __ddiv_rn(s, nd);
            sx[i] = __dadd_rn(xi, p);
#pragma unroll
            for (int d = 0; d < 7; ++d)
                if (ex[d]) {
                    sr[nb[d]] = FAST ? __fma_rn(-a[d], p, g[d]) : __dsub_rn(g[d], __dmul_rn(a[d], p));
                    sr[N + nb[d]] = FAST ? __fma_rn(-a[7 + d], p, g[7 + d])
                                         : __dsub_rn(g[7 + d], __dmul_rn(a[7 + d], p));
                }
        }
        __syncthreads();
    }
    for (int i = 2 * threadIdx.x; i < 2 * N; i += 2 * blockDim.x) {
        *reinterpret_cast<double2 *>(r + i) = *reinterpret_cast<const double2 *>(sr + i);
        *reinterpret_cast<double2 *>(x + i) = *reinterpret_cast<const double2 *>(sx + i);
    }
}

// One vertex of the multicolour sweep (same formula as mcs::node_update in
// ocmg_p1_mc.cuh): both of its unknowns in turn -- state then adjoint on a
// forward sweep, adjoint then state on a backward one -- each
//     p = (sum_d W_d r_S(d) + sum_d W_{7+d} r_A(d)) * (1 / n_diag)
// (two FMA chains from 0), x += p, r(d) = fma(-A_d, p, r(d)); the second
// unknown sees the first one's update.  Absent neighbours are skipped (their
// coefficients are 0).  r goes through L2 only (ld/st.cg): k_p1_mc_grid runs
// colours back to back in one launch.
__device__ __forceinline__ void p1_mc_vertex(int ix, int iy, int n1, bool forward,
                                             const double *__restrict__ T,
                                             double *__restrict__ x,
                                             double *__restrict__ r) {
    const int64_t N = (int64_t)n1 * n1;
    const P1Node q = p1_node(ix, iy, n1);
    double v0[7], v1[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        v0[d] = q.ex[d] ? __ldcg(r + q.nb[d]) : 0.0;
        v1[d] = q.ex[d] ? __ldcg(r + N + q.nb[d]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int field = forward ? u : 1 - u;
        const double *W = T + kP1OffW + q.c * 28 + 14 * field;
        const double *A = T + kP1OffA + q.c * 28 + 14 * field;
        const double rnd = __drcp_rn(__ldg(T + kP1OffND + q.c * 2 + field));
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d]) {
                s0 = __fma_rn(__ldg(W + d), v0[d], s0);
                s1 = __fma_rn(__ldg(W + 7 + d), v1[d], s1);
            }
        const double p = __dmul_rn(__dadd_rn(s0, s1), rnd);
        const int64_t i = field * N + q.v;
        x[i] = __dadd_rn(x[i], p);
#pragma unroll
        for (int d = 0; d < 7; ++d)
            if (q.ex[d]) {
                v0[d] = __fma_rn(-__ldg(A + d), p, v0[d]);
                v1[d] = __fma_rn(-__ldg(A + 7 + d), p, v1[d]);
            }
    }
#pragma unroll
    for (int d = 0; d < 7; ++d)
        if (q.ex[d]) {
            __stcg(r + q.nb[d], v0[d]);
            __stcg(r + N + q.nb[d], v1[d]);
        }
}

// One colour of the distance-2 multicolour order: colour c in 0..6 is the
// vertices with (ix + 2 iy) mod 7 == c (graph distance >= 3 between them: no
// 19-point offset satisfies dx + 2 dy = 0 mod 7), each updating both of its
// unknowns.  A forward sweep runs colours 0..6, a backward one 6..0.
constexpr int kMcColours = 7;
__global__ void k_p1_gs_colour(int n1, const double *__restrict__ T,
                               int colour, int forward, double *__restrict__ x,
                               double *__restrict__ r) {
    const int per_row = (n1 + 6) / 7;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= (int64_t)per_row * n1) return;
    const int iy = (int)(k / per_row);
    const int jj = (int)(k - (int64_t)iy * per_row);
    const int ix = ((colour - 2 * iy) % 7 + 7) % 7 + 7 * jj;
    if (ix >= n1) return;
    p1_mc_vertex(ix, iy, n1, forward != 0, T, x, r);
}

// partial[b] = sum over a grid-strided slice of L_i x_i^2 (both fields)
__global__ void k_p1_wsumsq_partial(int n1, const double *__restrict__ T,
                                    const double *__restrict__ x,
                                    double *__restrict__ partial) {
    __shared__ double sh[32];
    const int64_t N = (int64_t)n1 * n1;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int field = i >= N;
        const int64_t v = i - field * N;
        const int iy = (int)(v / n1), ix = (int)(v - (int64_t)iy * n1);
        const int c = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
        const double xi = x[i];
        acc += __ldg(T + kP1OffL + 2 * c + field) * xi * xi;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// ---------------------------------------------------------------------------
// P1 transfers, both fields (transfer.py:34-55 block-diagonal per field).
// R = P^T: coarse row (cx,cy) gathers, in increasing fine index, the fine
// vertices (2cx-1,2cy-1) (2cx,2cy-1) (2cx-1,2cy) (2cx,2cy) (2cx+1,2cy)
// (2cx,2cy+1) (2cx+1,2cy+1) with weights 1/2 except 1 at the centre.
// ---------------------------------------------------------------------------
__global__ void k_p1_restrict(int nc1, int n_fields,
                              const double *__restrict__ rf,
                              double *__restrict__ rc) {
    const int64_t Nc = (int64_t)nc1 * nc1;
    const int nf1 = 2 * nc1 - 1;
    const int64_t Nf = (int64_t)nf1 * nf1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= Nc) return;
    const int cy = (int)(v / nc1), cx = (int)(v - (int64_t)cy * nc1);
    const int fx = 2 * cx, fy = 2 * cy;
    const int64_t c = (int64_t)fy * nf1 + fx;
    const bool l = cx > 0, rr = cx < nc1 - 1, dn = cy > 0, up = cy < nc1 - 1;
    for (int b = 0; b < n_fields; ++b) {
        const double *f = rf + b * Nf;
        double s = 0.0;
        if (l && dn) s = __dadd_rn(s, __dmul_rn(0.5, f[c - nf1 - 1]));
        if (dn) s = __dadd_rn(s, __dmul_rn(0.5, f[c - nf1]));
        if (l) s = __dadd_rn(s, __dmul_rn(0.5, f[c - 1]));
        s = __dadd_rn(s, f[c]);
        if (rr) s = __dadd_rn(s, __dmul_rn(0.5, f[c + 1]));
        if (up) s = __dadd_rn(s, __dmul_rn(0.5, f[c + nf1]));
        if (rr && up) s = __dadd_rn(s, __dmul_rn(0.5, f[c + nf1 + 1]));
        rc[b * Nc + v] = s;
    }
}

// x_f += P c: coarse vertices copy, midpoints average their edge ends
// (lower end first), the interpolant summed before the add
__global__ void k_p1_prolong_add(int nc1, int n_fields,
                                 const double *__restrict__ c,
                                 double *__restrict__ xf) {
    const int64_t Nc = (int64_t)nc1 * nc1;
    const int nf1 = 2 * nc1 - 1;
    const int64_t Nf = (int64_t)nf1 * nf1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= Nf) return;
    const int fy = (int)(v / nf1), fx = (int)(v - (int64_t)fy * nf1);
    const int ox = fx & 1, oy = fy & 1;
    const int64_t a = (int64_t)(fy >> 1) * nc1 + (fx >> 1);
    const int64_t b2 = (int64_t)((fy >> 1) + oy) * nc1 + (fx >> 1) + ox;
    for (int b = 0; b < n_fields; ++b) {
        const double *cc = c + b * Nc;
        double s;
        if (!(ox | oy))
            s = __dmul_rn(1.0, cc[a]);
        else
            s = __dadd_rn(__dmul_rn(0.5, cc[a]), __dmul_rn(0.5, cc[b2]));
        xf[b * Nf + v] = __dadd_rn(xf[b * Nf + v], s);
    }
}

}  // namespace ocmg
