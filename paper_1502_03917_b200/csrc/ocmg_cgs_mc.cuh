// One-launch 3-colour CGS sweep on a structured P1 level (the multicolour
// mode of ocmg_cgs.cuh in a single launch, bit-identical to its six-launch
// form).
//
// Colour c = (ix + iy) mod 3 is a distance-1 colouring; a vertex reads only
// its own residual and writes its neighbours' (rows y-1 .. y+1).  Colour q+1
// at row y' needs colour q finished on rows <= y'+1, so a CTA streams its rows
// bottom to top running colour q on row s - 3q at step s: the three
// colour-rows of a step touch disjoint rows.  Every r_j receives its
// colour-c updates from the rows below it first, i.e. in increasing vertex
// index, the order of the six-launch gather.  The live rows (s-7 .. s+1) sit
// in a small shared-memory ring of (state, adjoint) pairs.
//
// Decomposition as in ocmg_p1_mc.cuh: a CTA owns W columns x seg_h rows,
// loads a halo of H = 3 (1 per colour) on every side, computes the halo
// vertices only where their updates reach the tile, writes only its tile of
// r (out of place) and x (in place).
#pragma once

#include "ocmg_p1_mc.cuh"

namespace ocmg {
namespace cgsm {
constexpr int H = 3;
constexpr int RING = 12;              // rows s-8 .. s+3
constexpr int W = 224;                // owned columns per CTA
constexpr int STRIDE = W + 2 * H + 2;
constexpr int PER = (W + 2 * H + 2) / 3;  // colour vertices per row (<= 77)
constexpr int WPC = (PER + 31) / 32;      // warps per colour
constexpr int NT = 3 * WPC * 32;
constexpr int SMEM = RING * STRIDE * 16;
constexpr int PF = 4;
static_assert(2 * STRIDE <= 2 * NT, "two row values per thread at most");
}  // namespace cgsm

struct CgsmParams {
    int n1, nstrips, base, rem;
    double alpha;
    // per position class: m = M_ii, k = K_ii, -m/alpha, det = -m m/alpha - k k
    // (formed on the host with the same IEEE operations as the reference)
    double mk[49][4];
    double a24[28];   // A rows of the interior class (constant-bank reads)
    const double *T;  // class tables (A rows)
    const double *rin;
    double *rout, *x;
};

__global__ void __launch_bounds__(cgsm::NT, 2)
    k_p1_cgs_mc_sweep(const __grid_constant__ CgsmParams P) {
    using namespace cgsm;
    extern __shared__ double2 ring[];  // [RING][STRIDE]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n1 = P.n1;
    const int64_t N = (int64_t)n1 * n1;
    const int strip = blockIdx.x % P.nstrips, seg = blockIdx.x / P.nstrips;
    const int nseg = P.base + (strip < P.rem ? 1 : 0);
    if (seg >= nseg) return;
    const int seg_h = (n1 + nseg - 1) / nseg;
    const int X0 = strip * W, X1 = min(n1, X0 + W);
    const int Y0 = seg * seg_h, Y1 = min(n1, Y0 + seg_h);
    if (Y0 >= Y1) return;
    const int xl = max(0, X0 - H), xr = min(n1, X1 + H);
    const int Ylo = max(0, Y0 - H), Yhi = min(n1, Y1 + H);

    // row loader: thread t handles entries t and t + NT of the 2*STRIDE row
    const int rmax = min(Yhi, n1 - 1);
    auto slot0 = [&](int yy) { return ((yy - Ylo) % RING + RING) % RING; };
    auto fetch = [&](int e, int yy) -> double {
        const int f = e >= STRIDE, lc = e - f * STRIDE, lx = xl - 1 + lc;
        if (e < 2 * STRIDE && lx >= xl && lx < xr && yy >= 0 && yy <= rmax && yy >= Ylo - 1)
            return __ldg(P.rin + f * N + (int64_t)yy * n1 + lx);
        return 0.0;
    };
    auto put = [&](int e, int yy, double v) {
        if (e < 2 * STRIDE) {
            const int f = e >= STRIDE, lc = e - f * STRIDE;
            reinterpret_cast<double *>(ring + slot0(yy) * STRIDE + lc)[f] = v;
        }
    };
    for (int yy = Ylo - 1; yy <= Ylo + 1; ++yy) {
        put(tid, yy, fetch(tid, yy));
        put(tid + NT, yy, fetch(tid + NT, yy));
    }
    double pf[PF][2];  // rows s+2 .. s+1+PF
#pragma unroll
    for (int i = 0; i < PF; ++i) {
        pf[i][0] = fetch(tid, Ylo + 2 + i);
        pf[i][1] = fetch(tid + NT, Ylo + 2 + i);
    }

    // compute role: warps [q*WPC, (q+1)*WPC) = colour q of the sweep
    const int q = warp / WPC, m = (warp - q * WPC) * 32 + lane;
    const int mg = (2 - q) + 1;  // margin whose updates reach the tile
    const int cxl = max(xl, X0 - mg), cxr = min(xr, X1 + mg);
    const int cyl = max(Ylo, Y0 - mg), cyh = min(Yhi, Y1 + mg);
    // x of this lane's vertex, prefetched two steps ahead (row y+2): the
    // read-modify-write would otherwise hold every step for an HBM round trip
    const int c = q;  // sweep position = colour (forward order)
    auto colx = [&](int yy) { return xl + (((c - xl - yy) % 3) + 3) % 3 + 3 * m; };
    auto owned = [&](int xx, int yy) {
        return q < 3 && xx >= X0 && xx < X1 && yy >= Y0 && yy < Y1;
    };
    auto xload = [&](int yy, int f) -> double {
        const int xx = colx(yy);
        return owned(xx, yy) ? P.x[f * N + (int64_t)yy * n1 + xx] : 0.0;
    };
    double xa[2], xb[2];
    {
        const int y0 = Ylo - 3 * q;
        for (int f = 0; f < 2; ++f) {
            xa[f] = xload(y0, f);
            xb[f] = xload(y0 + 1, f);
        }
    }
    __syncthreads();
    // store role: thread -> (field, output column) pairs
    const int ow = X1 - X0;

    const int nsteps = (Yhi - Ylo) + 3 * 2 + 3;
    for (int s = 0; s < nsteps; ++s) {
        const double ln0 = fetch(tid, Ylo + s + 2 + PF), ln1 = fetch(tid + NT, Ylo + s + 2 + PF);
        // final row leaves: colour 2 at step s touches rows >= Ylo+s-7
        const int ys = Ylo + s - 8;
        if (ys >= Y0 && ys < Y1) {
            const double2 *src = ring + slot0(ys) * STRIDE;
            for (int e = tid; e < 2 * ow; e += NT) {
                const int f = e >= ow, xx = X0 + e - f * ow;
                P.rout[f * N + (int64_t)ys * n1 + xx] =
                    reinterpret_cast<const double *>(src + (xx - xl + 1))[f];
            }
        }
        const int y = Ylo + s - 3 * q;
        double xcur[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            xcur[f] = xa[f];
            xa[f] = xb[f];
            xb[f] = xload(y + 2, f);
        }
        if (y >= cyl && y < cyh && q < 3) {
            // colour q's vertices in row y: x = first + 3 m
            const int xx = colx(y);
            if (xx >= cxl && xx < cxr) {
                const int sy = slot0(y);
                const int sb = sy == 0 ? RING - 1 : sy - 1;
                const int su = sy == RING - 1 ? 0 : sy + 1;
                const int c0 = xx - xl + 1;
                double2 *rb = ring + sb * STRIDE + c0, *rc = ring + sy * STRIDE + c0,
                        *ru = ring + su * STRIDE + c0;
                double2 *const adr[7] = {rb - 1, rb, rc - 1, rc, rc + 1, ru, ru + 1};
                const bool l = xx > 0, rr = xx < n1 - 1, dn = y > 0, up = y < n1 - 1;
                const bool ex[7] = {l && dn, dn, l, true, rr, up, rr && up};
                const int cls = 7 * p1_axis_class(y, n1) + p1_axis_class(xx, n1);
                const double *A = cls == 24 ? P.a24 : P.T + kP1OffA + cls * 28;
                const double mm = P.mk[cls][0], kk = P.mk[cls][1];
                const double mda = P.mk[cls][2], det = P.mk[cls][3];
                const double2 own = *rc;
                const double sv =
                    __ddiv_rn(__dsub_rn(__dmul_rn(mda, own.x), __dmul_rn(kk, own.y)), det);
                const double tv =
                    __ddiv_rn(__dadd_rn(__dmul_rn(-kk, own.x), __dmul_rn(mm, own.y)), det);
                const int64_t xi = (int64_t)y * n1 + xx;
                if (owned(xx, y)) {
                    P.x[xi] = __dadd_rn(xcur[0], sv);
                    P.x[N + xi] = __dadd_rn(xcur[1], tv);
                }
#pragma unroll
                for (int d = 0; d < 7; ++d)
                    if (ex[d]) {
                        double2 v = *adr[d];
                        // A symmetric: A_{j b, i f} = row i, block f, column
                        // block b, offset d = A[f][7 b + d]
                        v.x = __dsub_rn(__dsub_rn(v.x, __dmul_rn(A[d], sv)),
                                        __dmul_rn(A[14 + d], tv));
                        v.y = __dsub_rn(__dsub_rn(v.y, __dmul_rn(A[7 + d], sv)),
                                        __dmul_rn(A[21 + d], tv));
                        *adr[d] = v;
                    }
            }
        }
        put(tid, Ylo + s + 2, pf[0][0]);
        put(tid + NT, Ylo + s + 2, pf[0][1]);
#pragma unroll
        for (int i = 0; i + 1 < PF; ++i) {
            pf[i][0] = pf[i + 1][0];
            pf[i][1] = pf[i + 1][1];
        }
        pf[PF - 1][0] = ln0;
        pf[PF - 1][1] = ln1;
        __syncthreads();
    }
}

struct CgsmPlan {
    int nstrips = 0, base = 0, rem = 0, grid = 0;
};

inline CgsmPlan cgsm_plan(int n1, int sm_count) {
    CgsmPlan p;
    p.nstrips = (n1 + cgsm::W - 1) / cgsm::W;
    const int max_seg = std::max(1, n1 / 16);
    const int total = std::max(p.nstrips, std::min(2 * sm_count, p.nstrips * max_seg));
    p.base = total / p.nstrips;
    p.rem = total % p.nstrips;
    p.grid = p.nstrips * (p.base + (p.rem ? 1 : 0));
    return p;
}

}  // namespace ocmg
