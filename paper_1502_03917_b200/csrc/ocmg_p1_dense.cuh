// Exact-order NE-GS on the small structured levels (k = 3..5) as a dense
// linear map, wavefront mode only.
//
// A sweep is linear in the residual: x_out = x + S r, r_out = r - A S r
// (kernels.lsgs_sweep, kernels.py:43-66, maps (x, r) to exactly that).  At
// level creation S is built column by column from the reference-order sweep
// of each unit residual (k_p1_gs_small in the reference arithmetic, one CTA
// per column), then stored row-major.  A sweep is then two short, wide
// launches instead of 3 * 2^k + 8 dependent levels in one CTA:
//   k_dense_rows       d = S r, one warp per row (coalesced 16-byte loads of
//                      S, a fixed butterfly sum: deterministic)
//   k_p1_dense_finish  x += d, r -= A d (the P1 stencil, reference order)
// S is n^2 doubles per direction: 0.2 MB (L3), 2.7 MB (L4), 38 MB (L5), so
// the maps of a W-cycle's coarse levels stay in the 126 MB L2 between the
// visits of the fine levels.  L6 (571 MB) would stream from HBM slower than
// its one-CTA sweep, so the map stops at L5.  Rounding differs from the
// sequential sweep (the wavefront mode's 1e-12 contract).
#pragma once

#include "ocmg_common.cuh"
#include "ocmg_p1.cuh"

namespace ocmg {

constexpr int kP1DenseMaxN1 = 33;  // L5
constexpr int kDenseRowsWarps = 8;

// d[i] = sum_j S[i * ld + j] r[j], ld even (rows of S 16-byte aligned); r
// may sit at any double offset: it is read as scalars (from L1)
__global__ void __launch_bounds__(32 * kDenseRowsWarps)
    k_dense_rows(int n, int ld, const double *__restrict__ S, const double *__restrict__ r,
                 double *__restrict__ d) {
    const int row = blockIdx.x * kDenseRowsWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= n) return;
    const double *srow = S + (int64_t)row * ld;
    const double2 *s2 = reinterpret_cast<const double2 *>(srow);
    const int h = n / 2;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    int j = lane;
    // 8 independent 16-byte loads of S per lane in flight
    for (; j + 7 * 32 < h; j += 8 * 32) {
        double2 sv[8], rv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            sv[u] = __ldg(s2 + j + 32 * u);
            rv[u] = make_double2(__ldg(r + 2 * (j + 32 * u)), __ldg(r + 2 * (j + 32 * u) + 1));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a[u & 3] = fma(sv[u].x, rv[u].x, a[u & 3]);
            a[u & 3] = fma(sv[u].y, rv[u].y, a[u & 3]);
        }
    }
    for (; j < h; j += 32) {
        const double2 sv = __ldg(s2 + j), rv = make_double2(__ldg(r + 2 * j), __ldg(r + 2 * j + 1));
        a[0] = fma(sv.x, rv.x, a[0]);
        a[0] = fma(sv.y, rv.y, a[0]);
    }
    if ((n & 1) && lane == 0) a[1] = fma(__ldg(srow + n - 1), __ldg(r + n - 1), a[1]);
    double acc = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) d[row] = acc;
}

// x += d; r -= A d  (both fields of every vertex; A d in the residual's
// reference summation order)
__global__ void k_p1_dense_finish(int n1, const double *__restrict__ T,
                                  const double *__restrict__ d, double *__restrict__ x,
                                  double *__restrict__ r) {
    const int64_t N = (int64_t)n1 * n1;
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int iy = (int)(v / n1), ix = (int)(v - (int64_t)iy * n1);
    const P1Node q = p1_node(ix, iy, n1);
    const double *A = T + kP1OffA + q.c * 28;
    const double s0 = p1_row_dot(q, A, d, N);
    const double s1 = p1_row_dot(q, A + 14, d, N);
    r[v] = __dsub_rn(r[v], s0);
    r[N + v] = __dsub_rn(r[N + v], s1);
    x[v] = __dadd_rn(x[v], d[v]);
    x[N + v] = __dadd_rn(x[N + v], d[N + v]);
}

// unit residuals for the batched build: R[j * n + i] = (i == j), X = 0
__global__ void k_p1_dense_unit(int n, double *__restrict__ X, double *__restrict__ R) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n * n) {
        X[t] = 0.0;
        R[t] = (t / n == t % n) ? 1.0 : 0.0;
    }
}

// S[i * ld + j] = X[j * ld + i]  (32 x 32 tiles through shared memory)
__global__ void k_dense_transpose(int n, int ld, const double *__restrict__ X,
                                  double *__restrict__ S) {
    __shared__ double t[32][33];
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = j0 + k, i = i0 + threadIdx.x;
        if (j < n && i < n) t[k][threadIdx.x] = X[(int64_t)j * ld + i];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + k, j = j0 + threadIdx.x;
        if (i < n && j < n) S[(int64_t)i * ld + j] = t[threadIdx.x][k];
    }
}

// v = e_j (the collapse build's unit right-hand sides)
__global__ void k_unit_vector(int64_t n, int64_t j, double *__restrict__ v) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) v[t] = t == j ? 1.0 : 0.0;
}

// the parallel collapse build: v = e_{*jp}; X column *jp = corr, then *jp += K
__global__ void k_unit_vector_at(int64_t n, const int64_t *__restrict__ jp, double *__restrict__ v) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) v[t] = t == *jp ? 1.0 : 0.0;
}
__global__ void k_store_column(int64_t n, int ld, const int64_t *__restrict__ jp,
                               const double *__restrict__ corr, double *__restrict__ X) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t j = *jp;
    if (t < n && j < n) X[j * ld + t] = corr[t];
}
__global__ void k_index_advance(int64_t *jp, int64_t K) { *jp += K; }

}  // namespace ocmg
