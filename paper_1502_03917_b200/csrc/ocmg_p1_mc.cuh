// Distance-2 multicolour NE-GS sweep on a structured P1 level in ONE launch.
//
// Order: colour c in 0..13 is field c/7 and the vertices with
// (ix + 2 iy) mod 7 == c mod 7; all of colour 0, then all of colour 1, ...
// (backward: 13 .. 0).  Same-colour unknowns are at graph distance >= 3, so a
// colour is one parallel step.  Each unknown is the update of kernels.py:57-64
// (p = row_scaled . r / n_diag; x += p; r -= A[:, i] p) in FMA arithmetic
// (node_update below); the sweep is bit-identical to the 14-pass form
// (k_p1_gs_colour, ocmg__debug_mc_passes).  The reference-order modes keep the
// reference's exact arithmetic; this mode is its own smoother.
//
// Pipelining.  Colour q of the sweep at row y reads r on rows y-1..y+1 and
// writes the same rows; colour q+1 at row y' needs colour q finished on rows
// <= y'+2.  So one CTA streams its rows bottom to top, running colour q on
// row s - 3q at step s: the 14 colour-rows of a step touch disjoint rows and
// are independent, one __syncthreads per step.  Warp q owns colour q, lane m
// its m-th vertex in the row (vertices of one colour are 7 columns apart).
// The live rows (s-40 .. s+1) sit in a 44-row shared-memory ring of
// (state, adjoint) pairs, so every neighbour is one 16-byte access; rows are
// prefetched PF steps ahead into registers, row s-41 is final and leaves.
//
// Decomposition.  A CTA owns W columns x seg_h rows.  The valid region of r
// shrinks by 2 columns (rows) per colour, so it loads its tile plus a halo of
// H = 28 on every side, recomputes the halo (only where the result can reach
// the tile: margin 2(13-q)+1 for colour q) and writes only its own tile.
// Halos are read from r_in and the tile is written to r_out (out of place:
// neighbours read what this CTA overwrites); x is updated in place by the
// owning CTA.  One CTA per SM: strips get base or base+1 row segments so the
// grid is exactly the SM count.
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {
namespace mcs {
constexpr int RING = 44;  // rows s-41 .. s+2
constexpr int H = 28;     // 2 columns (rows) per colour x 14 colours
constexpr int NWARP = 14; // one warp per colour of the sweep
constexpr int NT = 32 * NWARP;
constexpr int PF = 4;     // row prefetch depth (steps)
constexpr int W = 160;    // owned columns per CTA
constexpr int STRIDE = W + 2 * H + 2;          // + guard column each side
constexpr int SMEM = RING * STRIDE * 16;
static_assert((W + 2 * H + 6) / 7 <= 32, "one warp per colour-row");
static_assert(2 * STRIDE <= NT, "one row value per thread");
static_assert(2 * W <= NT, "one output value per thread");

// one unknown in the multicolour sweep's arithmetic (mc_unknown in
// ocmg_p1.cuh is the same formula on global arrays):
//   p = (sum_d W_d r_S(d) + sum_d W_{7+d} r_A(d)) * (1 / n_diag),
//   each sum an FMA chain from 0; r(d) = fma(-A_d, p, r(d)).
// Coefficients of absent neighbours are 0 in the tables and the guard cells
// hold 0, so boundary vertices need no branches, only their class row.
// cw/ca/rnd: interior class (shared memory), tc: boundary class (global).
template <bool INTERIOR>
__device__ __forceinline__ double node_update(double2 *const (&adr)[7],
                                              const double *cw, const double *ca,
                                              double rnd,
                                              const double *__restrict__ tc) {
    double2 v[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) v[d] = *adr[d];
    auto W = [&](int d) { return INTERIOR ? cw[d] : __ldg(tc + d); };
    auto A = [&](int d) { return INTERIOR ? ca[d] : __ldg(tc + 14 + d); };
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = __fma_rn(W(d), v[d].x, s0);
        s1 = __fma_rn(W(7 + d), v[d].y, s1);
    }
    const double p = __dmul_rn(__dadd_rn(s0, s1), INTERIOR ? rnd : __ldg(tc + 28));
#pragma unroll
    for (int d = 0; d < 7; ++d)
        *adr[d] = make_double2(__fma_rn(-A(d), p, v[d].x), __fma_rn(-A(7 + d), p, v[d].y));
    return p;
}
}  // namespace mcs

struct McsParams {
    int n1, nstrips, base, rem, forward;
    int y_begin, y_end;        // rows this launch owns (a rank's strip; 0, n1)
    int64_t fs_in, fs_out, fs_x;  // field strides of rin / rout / x
    double ci[2][29];  // interior class (3,3): W row, A row, 1/n_diag per field
    const double *C;   // [49][2][29]: W row, A row, 1/n_diag per (class, field)
    // addressed by global vertex index y*n1+x (+ field * fs_*): rin must hold
    // rows [y_begin-29, y_end+29) of the domain, rout and x rows
    // [y_begin, y_end); a rank passes base pointers shifted by its slab start
    const double *rin;
    double *rout, *x;
};

__global__ void __launch_bounds__(mcs::NT, 1)
    k_p1_mc_sweep(const __grid_constant__ McsParams P) {
    using namespace mcs;
    extern __shared__ double2 ring[];  // [RING][STRIDE] (state, adjoint)
    const int tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
    const int n1 = P.n1;
    const int64_t NI = P.fs_in;
    const int strip = blockIdx.x % P.nstrips, seg = blockIdx.x / P.nstrips;
    const int nseg = P.base + (strip < P.rem ? 1 : 0);
    if (seg >= nseg) return;
    const int rows = P.y_end - P.y_begin;
    const int seg_h = (rows + nseg - 1) / nseg;
    const int X0 = strip * W, X1 = min(n1, X0 + W);
    const int Y0 = P.y_begin + seg * seg_h, Y1 = min(P.y_end, Y0 + seg_h);
    if (Y0 >= Y1) return;
    const int xl = max(0, X0 - H), xr = min(n1, X1 + H);
    const int Ylo = max(0, Y0 - H), Yhi = min(n1, Y1 + H);

    // row loader: thread -> (field, local column incl. guards); rows are
    // fetched while row <= rmax (rows only grow), the rest are zero
    const int lf = tid / STRIDE, lc = tid - lf * STRIDE;
    const int lx = xl - 1 + lc;
    const bool lact = tid < 2 * STRIDE && lx >= xl && lx < xr;
    const int rmax = min(Yhi, n1 - 1);
    double *ldst = reinterpret_cast<double *>(ring) + 2 * lc + lf;
    auto slot0 = [&](int y) { return (y - Ylo + 2 * RING) % RING; };
    if (tid < 2 * STRIDE)
        for (int y = Ylo - 1; y <= Ylo + 1; ++y)
            ldst[2 * STRIDE * slot0(y)] =
                lact && y >= 0 && y <= rmax ? __ldg(P.rin + lf * NI + (int64_t)y * n1 + lx)
                                            : 0.0;
    int lrow = Ylo + 2;  // next row to fetch
    const double *lsrc = P.rin + lf * NI + (int64_t)lrow * n1 + lx;
    double pf[PF];       // rows s+2 .. s+1+PF in flight
#pragma unroll
    for (int i = 0; i < PF; ++i) {
        pf[i] = lact && lrow <= rmax ? __ldg(lsrc) : 0.0;
        ++lrow;
        lsrc += n1;
    }
    int lslot = slot0(Ylo + 2);  // ring slot of row Ylo+s+2

    // compute role: warp q = position q of the sweep
    const int colour = P.forward ? q : 13 - q;
    const int field = colour / 7, cm = colour % 7;
    const int mg = 2 * (13 - q) + 1;  // margin whose result reaches the tile
    const int cxl = max(xl, X0 - mg), cxr = min(xr, X1 + mg);
    const int cyl = max(Ylo, Y0 - mg), cyh = min(Yhi, Y1 + mg);
    // this lane's vertex at step s: row y = Ylo + s - 3q, column
    // x = xl + o + 7 lane with o = (cm - xl - 2y) mod 7, so o(y+1) = o(y) - 2
    int y = Ylo - 3 * q;
    int o = (cm - xl - 2 * y) % 7;
    o += o < 0 ? 7 : 0;
    int sy = slot0(y);
    double *xrow = P.x + field * P.fs_x + (int64_t)y * n1 + xl + 7 * lane;
    const int xbase = xl + 7 * lane;
    auto owned = [&](int yy, int xx) {
        return yy >= Y0 && yy < Y1 && xx >= X0 && xx < X1;
    };
    // x of the vertex two steps ahead (row y+2, o - 4 mod 7)
    auto xpre = [&]() -> double {
        const int o2 = o + 3 >= 7 ? o - 4 : o + 3;
        return owned(y + 2, xbase + o2) ? xrow[2 * (int64_t)n1 + o2] : 0.0;
    };
    double xa, xb;
    {
        const int o1 = o - 2 < 0 ? o + 5 : o - 2;
        xa = owned(y, xbase + o) ? xrow[o] : 0.0;
        xb = owned(y + 1, xbase + o1) ? xrow[n1 + o1] : 0.0;
    }
    __syncthreads();
    // store role: thread -> (field, output column); row Ylo+s-41 leaves at
    // step s, i.e. steps [s_st0, s_st1)
    const int sf = tid / W, sx = X0 + (tid - sf * W);
    const bool sact = tid < 2 * W && sx < X1;
    const double *ssrc = reinterpret_cast<const double *>(ring) + 2 * (sx - xl + 1) + sf;
    double *sdst = P.rout + sf * P.fs_out + (int64_t)Y0 * n1 + sx;
    const int s_st0 = Y0 - Ylo + 41, s_st1 = Y1 - Ylo + 41;

    const int nsteps = (Yhi - Ylo) + 41;
    for (int s = 0; s < nsteps; ++s) {
        const double lnew = lact && lrow <= rmax ? __ldg(lsrc) : 0.0;
        ++lrow;
        lsrc += n1;
        const double xcur = xa;
        xa = xb;
        xb = xpre();
        if (sact && s >= s_st0 && s < s_st1) {
            const int ss = lslot + 1 == RING ? 0 : lslot + 1;  // slot of row Ylo+s-41
            *sdst = ssrc[2 * STRIDE * ss];
            sdst += n1;
        }
        const int x = xbase + o;
        if (y >= cyl && y < cyh && x >= cxl && x < cxr) {
            const int c0 = x - xl + 1;
            const int sb = sy == 0 ? RING - 1 : sy - 1;
            const int su = sy == RING - 1 ? 0 : sy + 1;
            double2 *rb = ring + sb * STRIDE + c0, *rc = ring + sy * STRIDE + c0,
                    *ru = ring + su * STRIDE + c0;
            double2 *const adr[7] = {rb - 1, rb, rc - 1, rc, rc + 1, ru, ru + 1};
            double p;
            if (y >= 3 && y <= n1 - 4 && x >= 3 && x <= n1 - 4) {
                // coefficients straight from the parameter bank (indexed
                // LDC: the constant cache, not the shared-memory pipe)
                p = node_update<true>(adr, P.ci[field], P.ci[field] + 14,
                                      P.ci[field][28], nullptr);
            } else {
                const int cls = 7 * p1_axis_class(y, n1) + p1_axis_class(x, n1);
                p = node_update<false>(adr, nullptr, nullptr, 0.0,
                                       P.C + (cls * 2 + field) * 29);
            }
            if (owned(y, x)) xrow[o] = __dadd_rn(xcur, p);
        }
        if (tid < 2 * STRIDE) ldst[2 * STRIDE * lslot] = pf[0];
#pragma unroll
        for (int i = 0; i + 1 < PF; ++i) pf[i] = pf[i + 1];
        pf[PF - 1] = lnew;
        // advance: row y+1
        lslot = lslot + 1 == RING ? 0 : lslot + 1;
        sy = sy + 1 == RING ? 0 : sy + 1;
        ++y;
        xrow += n1;
        o = o - 2 < 0 ? o + 5 : o - 2;
        __syncthreads();
    }
}

// host-side launch geometry: strips of W columns; base or base+1 row
// segments per strip so that the grid fills the SMs once
struct McsPlan {
    int nstrips = 0, base = 0, rem = 0, grid = 0;
};

inline McsPlan mcs_plan(int n1, int sm_count, int rows = -1) {
    McsPlan p;
    if (rows < 0) rows = n1;
    p.nstrips = (n1 + mcs::W - 1) / mcs::W;
    // segments much shorter than the pipeline fill (2H + 41 rows) waste steps
    const int max_seg = std::max(1, rows / 32);
    const int total = std::max(p.nstrips, std::min(sm_count, p.nstrips * max_seg));
    p.base = total / p.nstrips;
    p.rem = total % p.nstrips;
    p.grid = p.nstrips * (p.base + (p.rem ? 1 : 0));
    return p;
}

}  // namespace ocmg
