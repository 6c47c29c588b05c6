// Distance-2 multicolour NE-GS sweep on a structured P1 level in ONE launch.
//
// Order: colour c in 0..6 is the vertices with (ix + 2 iy) mod 7 == c (graph
// distance >= 3 between them); colours run 0..6 (backward: 6..0) and every
// vertex updates both of its unknowns in turn, state then adjoint (backward:
// adjoint then state).  Each unknown is the update of kernels.py:57-64
// (p = row_scaled . r / n_diag; x += p; r -= A[:, i] p) in FMA arithmetic
// (node_update below, p1_mc_vertex in ocmg_p1.cuh); the sweep is
// bit-identical to its 7-pass form (k_p1_gs_colour, ocmg__debug_mc_passes).
// The reference-order modes keep the reference's exact arithmetic; this mode
// is its own smoother (its own convergence factor).
//
// Pipelining.  Colour q of the sweep at row y reads r on rows y-1..y+1 and
// writes the same rows; colour q+1 at row y' needs colour q finished on rows
// <= y'+2.  So one CTA streams its rows bottom to top, running colour q on
// row s - 3q at step s: the 7 colour-rows of a step touch disjoint rows and
// are independent, one __syncthreads per step.  Warp q owns colour q, lane m
// its m-th vertex in the row (vertices of one colour are 7 columns apart).
// The live rows (s-19 .. s+1) sit in a 24-row shared-memory ring of
// (state, adjoint) pairs, so every neighbour is one 16-byte access and a
// vertex's two unknown updates share one load and one store of its
// neighbourhood; rows are prefetched PF steps ahead into registers, row
// s-20 is final and leaves.
//
// Decomposition.  A CTA owns W columns x seg_h rows.  The valid region of r
// shrinks by 2 columns (rows) per colour, so it loads its tile plus a halo of
// H = 14 on every side, recomputes the halo (only where the result can reach
// the tile: margin 2(6-q)+1 for colour q) and writes only its own tile.
// Halos are read from r_in and the tile is written to r_out (out of place:
// neighbours read what this CTA overwrites); x is updated in place by the
// owning CTA.  Two CTAs per SM (79 KB of shared memory each); strips get base
// or base+1 row segments so the grid fills the SMs once.
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {
namespace mcs {
constexpr int NC = kMcColours;     // 7
constexpr int H = 2 * NC;          // 2 columns (rows) per colour
constexpr int RING = 3 * (NC - 1) + 6;  // rows s-20 .. s+2 (+1 spare)
constexpr int NWARP = NC;          // one warp per colour of the sweep
constexpr int NT = 32 * NWARP;
constexpr int PF = 4;              // row prefetch depth (steps)
constexpr int W = 176;             // owned columns per CTA
constexpr int STRIDE = W + 2 * H + 2;  // + guard column each side
constexpr int SMEM = RING * STRIDE * 16;
constexpr int STORE_LAG = 3 * (NC - 1) + 2;  // row s - STORE_LAG is final at step s
static_assert((W + 2 * H + 6) / 7 <= 31, "one warp per colour-row, lane 31 free");
static_assert(2 * STRIDE <= 2 * NT && 2 * W <= 2 * NT, "two values per thread");

// one unknown (field f of the vertex) in the multicolour sweep's arithmetic:
//   p = (sum_d W_d r_S(d) + sum_d W_{7+d} r_A(d)) * (1 / n_diag),
//   each sum an FMA chain from 0; r(d) = fma(-A_d, p, r(d)).
// v: the neighbourhood (registers), updated in place.  Coefficients of
// absent neighbours are 0 in the tables and the guard cells hold 0, so
// boundary vertices need no branches, only their class row.
// c: W row (14), A row (14), 1/n_diag -- kernel parameters (interior class)
// or the global table (boundary classes).
__device__ __forceinline__ double node_update(double2 (&v)[7], const double *c) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = __fma_rn(c[d], v[d].x, s0);
        s1 = __fma_rn(c[7 + d], v[d].y, s1);
    }
    const double p = __dmul_rn(__dadd_rn(s0, s1), c[28]);
#pragma unroll
    for (int d = 0; d < 7; ++d)
        v[d] = make_double2(__fma_rn(-c[14 + d], p, v[d].x),
                            __fma_rn(-c[21 + d], p, v[d].y));
    return p;
}
// the same update with the coefficients read from shared memory by explicit
// 16-byte ld.shared (asm volatile: one load per use, never hoisted into
// registers -- the 58 interior coefficients would not fit beside the
// neighbourhood at 2 CTAs per SM, and indexed LDC from the parameter bank
// was a fifth of all instructions); cs: shared-memory address of a 30-double
// row (W 14, A 14, 1/n_diag, pad), 16-byte aligned
__device__ __forceinline__ double2 lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double node_update_s(double2 (&v)[7], unsigned cs) {
    double c[30];
#pragma unroll
    for (int i = 0; i < 15; ++i) {
        const double2 t = lds2(cs + 16 * i);
        c[2 * i] = t.x;
        c[2 * i + 1] = t.y;
    }
    return node_update(v, c);
}
}  // namespace mcs

struct McsParams {
    int n1, nstrips, base, rem, forward;
    int y_begin, y_end;        // rows this launch owns (a rank's strip; 0, n1)
    int64_t fs_in, fs_out, fs_x;  // field strides of rin / rout / x
    double ci[2][29];  // interior class (3,3): W row, A row, 1/n_diag per field
    const double *C;   // [49][2][29]: W row, A row, 1/n_diag per (class, field)
    // addressed by global vertex index y*n1+x (+ field * fs_*): rin must hold
    // rows [y_begin-15, y_end+15) of the domain, rout and x rows
    // [y_begin, y_end); a rank passes base pointers shifted by its slab start
    const double *rin;
    double *rout, *x;
};

__global__ void __launch_bounds__(mcs::NT, 2)
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

    // row loader: thread -> two (field, local column incl. guards) entries;
    // rows are fetched while row <= rmax (rows only grow), the rest are zero
    const int rmax = min(Yhi, n1 - 1);
    int lx[2], lf[2];
    bool lact[2];
    double *ldst[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int t = tid + e * NT;
        lf[e] = t >= STRIDE;
        const int lc = t - lf[e] * STRIDE;
        lx[e] = xl - 1 + lc;
        lact[e] = t < 2 * STRIDE && lx[e] >= xl && lx[e] < xr;
        ldst[e] = t < 2 * STRIDE ? reinterpret_cast<double *>(ring) + 2 * lc + lf[e] : nullptr;
    }
    auto slot0 = [&](int y) { return ((y - Ylo) % RING + RING) % RING; };
    auto fetch = [&](int e, int y) -> double {
        return lact[e] && y >= 0 && y <= rmax
                   ? __ldg(P.rin + lf[e] * NI + (int64_t)y * n1 + lx[e])
                   : 0.0;
    };
    for (int y = Ylo - 1; y <= Ylo + 1; ++y)
#pragma unroll
        for (int e = 0; e < 2; ++e)
            if (ldst[e]) ldst[e][2 * STRIDE * slot0(y)] = fetch(e, y);
    // steady state: one pointer per entry advanced a row per step, and the
    // rows still to fetch counted down (rows only grow; past rmax: zeros)
    int lrow = Ylo + 2;  // next row to fetch
    double pf[PF][2];    // rows s+2 .. s+1+PF in flight
#pragma unroll
    for (int i = 0; i < PF; ++i) {
#pragma unroll
        for (int e = 0; e < 2; ++e) pf[i][e] = fetch(e, lrow);
        ++lrow;
    }
    const double *lsrc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e)
        lsrc[e] = P.rin + lf[e] * NI + (int64_t)lrow * n1 + lx[e];
    int lleft = lrow <= rmax ? rmax - lrow + 1 : 0;  // valid rows left to fetch
    int lslot = slot0(Ylo + 2);  // ring slot of row Ylo+s+2

    // compute role: warp q = position q of the sweep
    const int colour = P.forward ? q : NC - 1 - q;
    const int f0 = P.forward ? 0 : 1;  // first field of each vertex
    const int mg = 2 * (NC - 1 - q) + 1;  // margin whose result reaches the tile
    const int cxl = max(xl, X0 - mg), cxr = min(xr, X1 + mg);
    const int cyl = max(Ylo, Y0 - mg), cyh = min(Yhi, Y1 + mg);
    // interior coefficients in shared memory (see node_update_s)
    __shared__ __align__(16) double sci[2][30];
    if (tid < 58) sci[tid / 29][tid % 29] = P.ci[tid / 29][tid % 29];
    const unsigned sci0 = (unsigned)__cvta_generic_to_shared(&sci[f0][0]);
    const unsigned sci1 = (unsigned)__cvta_generic_to_shared(&sci[1 - f0][0]);
    // this lane's vertex at step s: row y = Ylo + s - 3q, column
    // x = xl + o + 7 lane with o = (colour - xl - 2y) mod 7, so o(y+1) = o(y) - 2
    int y = Ylo - 3 * q;
    int o = (colour - xl - 2 * y) % 7;
    o += o < 0 ? 7 : 0;
    int sy = slot0(y);
    const int64_t FX = P.fs_x;
    double *xrow = P.x + (int64_t)y * n1 + xl + 7 * lane;
    const int xbase = xl + 7 * lane;
    auto owned = [&](int yy, int xx) {
        return yy >= Y0 && yy < Y1 && xx >= X0 && xx < X1;
    };
    // x of the vertex two steps ahead (row y+2, o - 4 mod 7), both fields
    double xa[2], xb[2];
    {
        const int o1 = o - 2 < 0 ? o + 5 : o - 2;
        const bool w0 = owned(y, xbase + o), w1 = owned(y + 1, xbase + o1);
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            xa[f] = w0 ? xrow[f * FX + o] : 0.0;
            xb[f] = w1 ? xrow[f * FX + n1 + o1] : 0.0;
        }
    }
    __syncthreads();
    // store role: thread -> two (field, output column) entries; row
    // Ylo+s-STORE_LAG leaves at step s, i.e. steps [s_st0, s_st1)
    const double *ssrc[2];
    double *sdst[2];
    bool sact[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int t = tid + e * NT;
        const int sf = t / W, sx = X0 + (t - sf * W);
        sact[e] = t < 2 * W && sx < X1;
        ssrc[e] = reinterpret_cast<const double *>(ring) + 2 * (sx - xl + 1) + sf;
        sdst[e] = P.rout + sf * P.fs_out + (int64_t)Y0 * n1 + sx;
    }
    const int s_st0 = Y0 - Ylo + STORE_LAG, s_st1 = Y1 - Ylo + STORE_LAG;

    const int nsteps = (Yhi - Ylo) + STORE_LAG;
    for (int s = 0; s < nsteps; ++s) {
        double lnew[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            lnew[e] = lact[e] && lleft > 0 ? __ldg(lsrc[e]) : 0.0;
            lsrc[e] += n1;
        }
        lleft -= lleft > 0 ? 1 : 0;
        double xcur[2];
        {
            const int o2 = o + 3 >= 7 ? o - 4 : o + 3;
            const bool w2 = owned(y + 2, xbase + o2);
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                xcur[f] = xa[f];
                xa[f] = xb[f];
                xb[f] = w2 ? xrow[f * FX + 2 * (int64_t)n1 + o2] : 0.0;
            }
        }
        if (s >= s_st0 && s < s_st1) {
            const int ss = lslot + (RING - 2 - STORE_LAG) % RING;  // slot of row Ylo+s-STORE_LAG
            const int slot = ss >= RING ? ss - RING : ss;
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (sact[e]) {
                    *sdst[e] = ssrc[e][2 * STRIDE * slot];
                    sdst[e] += n1;
                }
        }
        const int x = xbase + o;
        if (y >= cyl && y < cyh && x >= cxl && x < cxr) {
            const int c0 = x - xl + 1;
            const int sb = sy == 0 ? RING - 1 : sy - 1;
            const int su = sy == RING - 1 ? 0 : sy + 1;
            double2 *rb = ring + sb * STRIDE + c0, *rc = ring + sy * STRIDE + c0,
                    *ru = ring + su * STRIDE + c0;
            double2 *const adr[7] = {rb - 1, rb, rc - 1, rc, rc + 1, ru, ru + 1};
            double2 v[7];
#pragma unroll
            for (int d = 0; d < 7; ++d) v[d] = *adr[d];
            double p[2];
            if (y >= 3 && y <= n1 - 4 && x >= 3 && x <= n1 - 4) {
                // coefficients straight from the parameter bank (indexed LDC:
                // the constant cache, not the shared-memory pipe)
                p[f0] = node_update_s(v, sci0);
                p[1 - f0] = node_update_s(v, sci1);
            } else {
                const int cls = 7 * p1_axis_class(y, n1) + p1_axis_class(x, n1);
                p[f0] = node_update(v, P.C + (cls * 2 + f0) * 29);
                p[1 - f0] = node_update(v, P.C + (cls * 2 + 1 - f0) * 29);
            }
#pragma unroll
            for (int d = 0; d < 7; ++d) *adr[d] = v[d];
            if (owned(y, x)) {
                xrow[o] = __dadd_rn(xcur[0], p[0]);
                xrow[FX + o] = __dadd_rn(xcur[1], p[1]);
            }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e)
            if (ldst[e]) ldst[e][2 * STRIDE * lslot] = pf[0][e];
#pragma unroll
        for (int i = 0; i + 1 < PF; ++i) {
            pf[i][0] = pf[i + 1][0];
            pf[i][1] = pf[i + 1][1];
        }
        pf[PF - 1][0] = lnew[0];
        pf[PF - 1][1] = lnew[1];
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
// segments per strip so that the grid fills the SMs (two CTAs each) once
struct McsPlan {
    int nstrips = 0, base = 0, rem = 0, grid = 0;
};

inline McsPlan mcs_plan(int n1, int sm_count, int rows = -1) {
    McsPlan p;
    if (rows < 0) rows = n1;
    p.nstrips = (n1 + mcs::W - 1) / mcs::W;
    // segments much shorter than the pipeline fill (2H + STORE_LAG rows) waste steps
    const int max_seg = std::max(1, rows / 24);
    const int total = std::max(p.nstrips, std::min(2 * sm_count, p.nstrips * max_seg));
    p.base = total / p.nstrips;
    p.rem = total % p.nstrips;
    p.grid = p.nstrips * (p.base + (p.rem ? 1 : 0));
    return p;
}

}  // namespace ocmg
