// Exact-order NE-GS sweep of a mid-size structured level (L7, L8) in one CTA
// with an anti-diagonal ring of the residual in shared memory.
//
// The reference order (kernels.py:57-64 over the index order of
// mesh.py:146-147) has dependency levels t: the leading field's unknowns
// sit on the anti-diagonal s = ix + 2 iy = t, the trailing field's on
// s = t - 7 (k_p1_gs_level).  The 7-point stencil moves s by -3..3, so level
// t touches only the diagonals [t-10, t+3] of r.  The kernel keeps a ring of
// R = 32 diagonals (both fields, indexed by row) in shared memory: at level
// t it writes diagonal t-11 back to global memory and prefetches diagonal
// t+R-11 into the same slot with cp.async (the same thread owns an element
// in both, so the slot hand-over needs no barrier).  x of the unknown a
// thread updates two levels ahead is prefetched into registers.  Levels are
// separated by one __syncthreads; threads [0, P) take the leading field's
// unknowns of a level in row order, [P, 2P) the trailing field's.
//
// A backward sweep is the point reflection of a forward one with the fields
// swapped, so the kernel runs in virtual coordinates (vx, vy) = reflected
// (ix, iy) and negates the stencil offsets; the arithmetic follows the real
// CSR order d = 0..6 (p1_gs_unknown), so the result is bit-identical to the
// reference sweep (FAST = false); FAST = true is the wavefront mode's
// arithmetic (two FMA chains, reciprocal multiply; 1e-12).
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {
namespace gsd {
constexpr int kMinN1 = 129, kMaxN1 = 257, kRing = 32;
inline int per_field(int n1) { return 32 * (((n1 + 1) / 2 + 31) / 32); }
inline size_t smem(int n1) {
    return ((size_t)kRing * 2 * n1 + kP1TableDoubles) * sizeof(double);
}
__device__ __forceinline__ void cp8(double *s, const double *g) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void cp16(double *s, const double *g) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace gsd

template <int MAXT, int R, bool BWD, bool FAST>
__global__ void __launch_bounds__(MAXT, 1)
    k_p1_gs_diag(int n1, const double *__restrict__ T, double *__restrict__ x,
                 double *__restrict__ r) {
    extern __shared__ __align__(16) double gd_sm[];
    constexpr int M = R - 1;
    const int N = n1 * n1, NT = blockDim.x, P = NT / 2, j = threadIdx.x;
    const int smax = 3 * (n1 - 1), depth = smax + 8;
    double *ring = gd_sm, *sT = gd_sm + (size_t)R * 2 * n1;
    // global index of virtual vertex (vx, vy)
    auto gv = [&](int vx, int vy) { return BWD ? N - 1 - (vy * n1 + vx) : vy * n1 + vx; };
    // element e in [0, 2 n1) of diagonal s: field e >= n1, row vy
    auto fetch = [&](int s) {
        for (int e = j; e < 2 * n1; e += NT) {
            const int f = e >= n1, vy = e - f * n1, vx = s - 2 * vy;
            if (vx >= 0 && vx < n1)
                gsd::cp8(ring + ((s & M) * 2 + f) * n1 + vy, r + f * N + gv(vx, vy));
        }
    };
    // element idx of field f on diagonal s: row lo(s) + idx
    auto diag_lo = [&](int s) { return s > n1 - 1 ? (s - n1 + 2) / 2 : 0; };
    auto diag_row = [&](int s, int i, int &vx, int &vy) {
        vy = diag_lo(s) + i;
        vx = s - 2 * vy;
        return s >= 0 && s <= smax && vx >= 0 && vy < n1;
    };
    for (int i = 2 * j; i < kP1TableDoubles; i += 2 * NT) gsd::cp16(sT + i, T + i);
    for (int s = 0; s <= min(R - 12, smax); ++s) fetch(s);
    gsd::commit();

    // this thread's unknown at level t: leading field (threads [0, P)) on
    // diagonal t, trailing field on t - 7; rows in increasing vy.  The same
    // threads retire / fetch field (j >= P) of the ring's diagonals.
    const bool lead = j < P;
    const int idx = lead ? j : j - P;
    const int field = lead == !BWD ? 0 : 1;  // real field of the unknown
    const int rf = lead ? 0 : 1;             // ring field this thread moves
    auto xload = [&](int t) {
        int vx, vy;
        return diag_row(lead ? t : t - 7, idx, vx, vy) ? x[field * N + gv(vx, vy)] : 0.0;
    };
    constexpr int DX[7] = {-1, 0, -1, 0, 1, 0, 1}, DY[7] = {-1, -1, 0, 0, 0, 1, 1};
    auto level = [&](int t, double xi) {
        {
            // retire diagonal t-11 (last touched at level t-1); fetch
            // diagonal t+R-12 into the slot retired at level t-1
            int vx, vy;
            const int sw = t - 11, sp = t + R - 12;
            if (diag_row(sw, idx, vx, vy))
                r[rf * N + gv(vx, vy)] = ring[((sw & M) * 2 + rf) * n1 + vy];
            if (t > 0 && diag_row(sp, idx, vx, vy))
                gsd::cp8(ring + ((sp & M) * 2 + rf) * n1 + vy, r + rf * N + gv(vx, vy));
            gsd::commit();
        }
        int vx, vy;
        if (diag_row(lead ? t : t - 7, idx, vx, vy)) {
            const int ix = BWD ? n1 - 1 - vx : vx, iy = BWD ? n1 - 1 - vy : vy;
            const int c = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
            const bool l = ix > 0, rr = ix < n1 - 1, dn = iy > 0, up = iy < n1 - 1;
            const bool ex[7] = {l && dn, dn, l, true, rr, up, rr && up};
            const int s = vx + 2 * vy;
            int o[7];  // ring offset of neighbour d (state field)
#pragma unroll
            for (int d = 0; d < 7; ++d) {
                const int ddx = BWD ? -DX[d] : DX[d], ddy = BWD ? -DY[d] : DY[d];
                o[d] = ((s + ddx + 2 * ddy) & M) * 2 * n1 + vy + ddy;
            }
            double g[14];
#pragma unroll
            for (int d = 0; d < 7; ++d) {
                g[d] = ex[d] ? ring[o[d]] : 0.0;
                g[7 + d] = ex[d] ? ring[o[d] + n1] : 0.0;
            }
            const double *W = sT + kP1OffW + c * 28 + 14 * field;
            const double *A = sT + kP1OffA + c * 28 + 14 * field;
            double sum = 0.0;
            if (FAST) {  // two FMA chains (the multicolour formula)
                double s1 = 0.0;
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) {
                        sum = __fma_rn(W[d], g[d], sum);
                        s1 = __fma_rn(W[7 + d], g[7 + d], s1);
                    }
                sum = __dadd_rn(sum, s1);
            } else {
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) sum = __dadd_rn(sum, __dmul_rn(W[d], g[d]));
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) sum = __dadd_rn(sum, __dmul_rn(W[7 + d], g[7 + d]));
            }
            double a[14];  // before the first shared store (one array)
#pragma unroll
            for (int e = 0; e < 14; ++e) a[e] = A[e];
            const double nd = sT[kP1OffND + c * 2 + field];
            const double p = FAST ? __dmul_rn(sum, __drcp_rn(nd)) : __ddiv_rn(sum, nd);
            x[field * N + iy * n1 + ix] = __dadd_rn(xi, p);
#pragma unroll
            for (int d = 0; d < 7; ++d)
                if (ex[d]) {
                    ring[o[d]] = FAST ? __fma_rn(-a[d], p, g[d]) : __dsub_rn(g[d], __dmul_rn(a[d], p));
                    ring[o[d] + n1] = FAST ? __fma_rn(-a[7 + d], p, g[7 + d])
                                           : __dsub_rn(g[7 + d], __dmul_rn(a[7 + d], p));
                }
        }
        // the diagonal fetched at level t' is first read at level t'+R-15
        gsd::wait_group<R - 16>();
        __syncthreads();
    };
    // x of the unknown two levels ahead is loaded into the register the
    // level just consumed (unrolled by two: no register copy waits on it)
    double xa = xload(0), xb = xload(1);
    gsd::wait_group<0>();
    __syncthreads();
    int t = 0;
    for (; t + 1 < depth; t += 2) {
        level(t, xa);
        xa = xload(t + 2);
        level(t + 1, xb);
        xb = xload(t + 3);
    }
    if (t < depth) level(t, xa);
    gsd::wait_group<0>();
    __syncthreads();
    // diagonals not retired in the loop
    for (int s = max(0, depth - 11); s <= smax; ++s) {
        int vx, vy;
        if (diag_row(s, idx, vx, vy)) r[rf * N + gv(vx, vy)] = ring[((s & M) * 2 + rf) * n1 + vy];
    }
}

}  // namespace ocmg
