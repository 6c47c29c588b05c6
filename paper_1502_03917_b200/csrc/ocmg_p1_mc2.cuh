// Distance-2 multicolour NE-GS sweep in ONE launch, rolling-window form
// (EXPERIMENTAL: opt-in with OCMG_MC_SWEEP=roll; k_p1_mc_sweep stays the
// default, see "Measured" below).
//
// Same smoother, order, arithmetic and tile decomposition as k_p1_mc_sweep
// (ocmg_p1_mc.cuh: colour c = (ix + 2 iy) mod 7, colours 0..6 forward, 6..0
// backward, a vertex's two unknowns in turn, node_update arithmetic,
// kernels.py:57-64), bit-identical to the 7-pass form.  What changes is who
// holds the residual between colours.
//
// An r entry e is touched by exactly one vertex per colour, and in colour
// order those are (relative to e) (-1,-1), (0,-1), (-1,0), (0,0), (1,0),
// (0,1), (1,1): runs of consecutive columns on rows y-1, y, y+1.  So a lane
// that walks a row's segment of 7 consecutive columns -- colours 0..6 in
// order, starting where (x + 2y) mod 7 = 0 -- keeps 4 of the 7 entries of a
// vertex's neighbourhood in registers from one colour to the next and moves
// 3 entries in and 3 out per vertex (k_p1_mc_sweep: 7 in, 7 out; its
// shared-memory pipe is 56% busy).
//
// Schedule.  Colour position q of row y runs at step y + 3 q (colour q+1 at
// row y needs colour q finished on rows y-2 .. y+2).  Row y belongs to warp
// y mod 21 for all seven colours, lane m its m-th segment, so a warp computes
// every third step and the 21 row warps form three groups of 7.  The steps
// are chained by three mbarriers (the 7 row warps and the boundary warp of
// step S arrive, those of step S + 1 wait); between its compute steps a group
// does its duties off that chain: it retires a finished row (r to r_out,
// x += delta, a thread per column, x staged by cp.async one duty earlier) and
// issues the cp.async of a new row.  The deltas of a row's vertices wait for
// the row's retirement in a second ring.  A 22nd warp takes the vertices of
// the boundary columns (class rows from shared memory, loads pipelined ahead
// of their use) and the three boundary rows at each end of the domain (class
// rows from the global table), full neighbourhood in and out.
//
// A lane's window is inherited only from its own previous vertex: where
// that vertex was not the lane's to compute (outside the colour's valid
// region, or a boundary column) the neighbourhood is loaded in full, and
// stored in full where the next one is not.  scripts/mc2_emulate.py runs
// this schedule on the CPU (masks, inheritance, slots, duties) against a
// plain colour-by-colour sweep.
//
// Measured (B200, L12; bench.py --quick under OCMG_MC_SWEEP=roll, scripts/
// mc2_prof.py per-warp cycle counters with -DMC2_PROF, scripts/micro_node.cu,
// micro_dfma_lat.cu): 0.411 ms per sweep (40% of HBM) against k_p1_mc_sweep's
// 0.350 ms.  A vertex update is a 20-deep dependent FP64 chain (DFMA 8.3
// cycles): 217 cycles on one warp, 250 for 7 warps with the 3 + 3
// shared-memory accesses, ~400 with a CTA barrier per step.  The kernel's
// step takes ~1060 cycles: ~600-700 of compute phase and ~300 between one
// group's last store and the next group's first load (mbarrier, hardware
// named barriers and a CTA barrier all measure the same).  Found on the way,
// each worth 10-40%: register-staged x spilled and turned the prefetch into
// a blocking load (x is staged by cp.async); any value in local memory costs
// ~300 cycles per reload because L1 is nearly all shared memory (the loop
// is at the 80-register limit of 22 warps: setup-only state is parked in
// shared memory, the boundary warp recomputes its lane state each step);
// divergent regions around one or two lanes' extra loads / stores cost the
// warp ~50 cycles each (predicated PTX now); a code copy per colour position
// (static window slots, no register moves) was slower than one copy with 16
// moves; one-warp duties (lane = column mod 32) are latency-bound at
// 2200-4100 cycles a row; __threadfence_block before an arrive is a
// MEMBAR.SC (~300 cycles).  What would be next is a dependency chain per row
// warp (row y at step S only needs rows y+2, y+1 at S-1, S-2) instead of a
// barrier per step, which would also let the warps of a group drift apart.
// Two rows per warp and step (two independent chains) would need a 46-row
// ring, more shared memory than an SM has at this tile width.
#pragma once

#include "ocmg_p1_mc.cuh"

// timing experiments (dev): -DMC2_X=<bits> switches roles off (1 compute,
// 2 retire, 4 load, 8 boundary columns); results are then wrong
#ifndef MC2_X
#define MC2_X 0
#endif

namespace ocmg {
#ifdef MC2_PROF
// per (CTA, warp): cycles waiting for the step barrier, computing, in duties, total
__device__ unsigned long long mc2_prof[256 * 24 * 4];
#define MC2_T(v) const long long v = clock64()
#else
#define MC2_T(v)
#endif
namespace mc2 {
using mcs::CROW;
using mcs::H;
using mcs::NC;
using mcs::NU;
#ifndef MC2_W
#define MC2_W 171
#endif
constexpr int W = MC2_W;            // owned columns per CTA (at most)
constexpr int NWARP = 3 * NC;       // a row stays with its warp for 3 * 7 steps
constexpr int NT = 32 * (NWARP + 1);  // + the boundary-column warp
constexpr int GT = 32 * NC;         // threads of a phase group
constexpr int GL = 8;               // guard columns left of xl in a ring row
constexpr int STRIDE = 234;         // ring row: columns xl - 8 .. xl + 225
constexpr int RS = STRIDE * 16;     // r ring row bytes ((state, adjoint) pairs)
constexpr int DS = W * 16;          // delta ring row bytes (owned columns)
constexpr int AHEAD = 7;            // step S loads relative row S + AHEAD
constexpr int RETIRE = 3 * (NC - 1) + 3;  // relative row ry leaves in the window after step ry + RETIRE - 1
// ring rows; slot of relative row ry is (ry + 1) % RING.  A slot is reloaded
// (row ry + RING, in the window after step ry + RING - AHEAD - 2) only after
// the group that retired row ry (window after step ry + RETIRE - 1) has
// arrived at its next step's barrier (ry + RETIRE + 2) and the loading group
// has waited for it: RING - AHEAD - 2 >= RETIRE + 3
constexpr int RING = AHEAD + RETIRE + 5;
constexpr int D_OFF = RING * RS;
constexpr int DRING = RETIRE + 3;   // delta ring rows (slot (ry + 1) % DRING): written at steps ry .. ry + 18,
                                    // read in the window after step ry + RETIRE - 1, rewritten (row ry + DRING)
                                    // by a group that has waited for the reader's next arrival (ry + RETIRE + 2)
constexpr int XSLOTS = 6;           // x staging rows (row % 6): a group may stage row R + 6 before the
                                    // group retiring row R + 2 has read its x
constexpr int X_OFF = D_OFF + DRING * DS;
constexpr int CLS_OFF = X_OFF + XSLOTS * DS;
constexpr int MB_OFF = CLS_OFF + 7 * 2 * CROW * 8;  // three step mbarriers
constexpr int SMEM = MB_OFF + 32;
constexpr int LCOLS = GT;           // ring columns a row load covers (one per loader thread)
static_assert(W + 2 * H + 6 <= 224, "32 segments of 7 columns cover the tile and its halo");
static_assert(GL + 224 + 2 <= STRIDE, "ring row covers every neighbour of every segment");
static_assert(GL + W + 2 * H <= LCOLS, "a row load covers the tile and its halo");
constexpr int RCH = (W + 31) / 32;   // 32-column chunks of a retiring row
static_assert(SMEM + 1024 <= 228 * 1024, "one CTA per SM");

__device__ __forceinline__ void sts2(unsigned a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
// predicated forms (no branch: a divergent region around one or two lanes'
// extra loads or stores cost the whole warp ~50 cycles each, four of them per
// vertex ~200 of the compute phase's 650)
__device__ __forceinline__ void lds2_if(double2 &v, unsigned a, bool p) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.s32 q, %3, 0;\n@q ld.shared.v2.f64 {%0, %1}, [%2];\n}"
                 : "+d"(v.x), "+d"(v.y)
                 : "r"(a), "r"((int)p)
                 : "memory");
}
__device__ __forceinline__ void sts2_if(unsigned a, double2 v, bool p) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.s32 q, %3, 0;\n@q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a),
                 "d"(v.x), "d"(v.y), "r"((int)p)
                 : "memory");
}
__device__ __forceinline__ double lds1(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double ldg1(const double *p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
// node_update (same operations, same order) with every coefficient loaded
// next to its use: the boundary paths must not hold a class row in registers
// on top of the lane's window.  LD(i): coefficient i of the row (W 0-13,
// A 14-27, 1/n_diag 28).
template <class LD>
__device__ __forceinline__ double node_update_ld(double2 (&v)[7], LD ld) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = __fma_rn(ld(d), v[d].x, s0);
        s1 = __fma_rn(ld(7 + d), v[d].y, s1);
    }
    const double p = __dmul_rn(__dadd_rn(s0, s1), ld(28));
#pragma unroll
    for (int d = 0; d < 7; ++d)
        v[d] = make_double2(__fma_rn(-ld(14 + d), p, v[d].x), __fma_rn(-ld(21 + d), p, v[d].y));
    return p;
}
// The steps are chained by three mbarriers in shared memory (step S uses
// number S % 3, phase parity (S / 3) & 1): each of the 8 warps of step S (7
// row warps and the boundary warp) arrives once when its vertices are
// stored, the warps of step S + 1 poll it.  Hardware barriers (bar.sync /
// bar.arrive, also as producer / consumer pairs) cost 300-400 cycles a step
// here while the duty warps' global stores and cp.asyncs were in flight.
#ifndef MC2_BAR
#define MC2_BAR 0
#endif
__device__ __forceinline__ void mb_init(unsigned a, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive_warp(unsigned a) {  // one arrival per warp
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
        asm volatile("{\n.reg .b64 t;\nmbarrier.arrive.release.cta.shared::cta.b64 t, [%0];\n}" ::"r"(a)
                     : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned a, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// Both unknowns of a vertex with the class rows in shared memory (ca: the
// row of the first unknown, cb: of the second; node_update's operations in
// its order).  The 58 coefficients are loaded in the order of their use, each
// LOOK uses ahead, so that a load's latency hides behind the dependent FMAs
// before it and only LOOK coefficients are held at a time.
__device__ __forceinline__ void node_update_pair_s(double2 (&v)[7], unsigned ca, unsigned cb,
                                                   double &pa, double &pb) {
    constexpr int LOOK = 6, N = 58;
    // use i of an unknown (0..28): W_d, W_{7+d} alternating (0..13), 1/n_diag (14), A_d, A_{7+d} (15..28)
    auto slot = [](int i) {
        const int t = i % 29;
        return t < 14 ? ((t & 1) ? 7 + (t >> 1) : (t >> 1)) : t == 14 ? 28
                      : (((t - 15) & 1) ? 21 + ((t - 15) >> 1) : 14 + ((t - 15) >> 1));
    };
    double q[LOOK];
#pragma unroll
    for (int i = 0; i < LOOK; ++i) q[i] = lds1((i < 29 ? ca : cb) + 8u * slot(i));
    double s0 = 0.0, s1 = 0.0, p = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double cf = q[i % LOOK];
        if (i + LOOK < N) q[i % LOOK] = lds1((i + LOOK < 29 ? ca : cb) + 8u * slot(i + LOOK));
        const int t = i % 29;
        if (t < 14) {
            if (t == 0) s0 = s1 = 0.0;
            if (t & 1) s1 = __fma_rn(cf, v[t >> 1].y, s1);
            else s0 = __fma_rn(cf, v[t >> 1].x, s0);
        } else if (t == 14) {
            p = __dmul_rn(__dadd_rn(s0, s1), cf);
            if (i < 29) pa = p; else pb = p;
        } else {
            const int d = (t - 15) >> 1;
            if ((t - 15) & 1) v[d].y = __fma_rn(-cf, p, v[d].y);
            else v[d].x = __fma_rn(-cf, p, v[d].x);
        }
    }
}
__device__ __forceinline__ int pmod7(int a) {  // a mod 7 in 0..6, a > -700000
    return (a + 700000) % 7;
}
}  // namespace mc2

// One vertex of a boundary row (y < 3 or y > n1 - 4): its class row comes
// from the global table, its neighbourhood is loaded and stored in full.
// The boundary warp's.
template <bool FWD>
__device__ __forceinline__ void mc2_boundary_row_vertex(const double *Cc, unsigned b, unsigned c,
                                                     unsigned u, unsigned ad, bool owned) {
    using namespace mc2;
    double2 v[7];
    v[0] = lds2(b - 16); v[1] = lds2(b);
    v[2] = lds2(c - 16); v[3] = lds2(c); v[4] = lds2(c + 16);
    v[5] = lds2(u); v[6] = lds2(u + 16);
    const double *Ca = Cc + (FWD ? 0 : 29), *Cb = Cc + (FWD ? 29 : 0);
    const double pa = node_update_ld(v, [&](int i) { return ldg1(Ca + i); });
    const double pb = node_update_ld(v, [&](int i) { return ldg1(Cb + i); });
    sts2(b - 16, v[0]); sts2(b, v[1]);
    sts2(c - 16, v[2]); sts2(c, v[3]); sts2(c + 16, v[4]);
    sts2(u, v[5]); sts2(u + 16, v[6]);
    if (owned) sts2(ad, make_double2(FWD ? pa : pb, FWD ? pb : pa));
}

template <bool FWD>
__global__ void __launch_bounds__(mc2::NT, 1) k_p1_mc_roll(const __grid_constant__ McsParams P) {
    using namespace mc2;
    extern __shared__ __align__(16) double2 ring2[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n1 = P.n1;
    const int strip = blockIdx.x % P.nstrips, seg = blockIdx.x / P.nstrips;
    // the extra row segments go to the edge strips first: their boundary
    // warp's steps are the longer ones
    const int pri = strip == 0 ? 0 : strip == P.nstrips - 1 ? 1 : strip + 1;
    const int nseg = P.base + (pri < P.rem ? 1 : 0);
    if (seg >= nseg) return;
    const int rows = P.y_end - P.y_begin;
    const int seg_h = (rows + nseg - 1) / nseg;
    const int X0 = strip * n1 / P.nstrips, X1 = (strip + 1) * n1 / P.nstrips;
    const int Y0 = P.y_begin + seg * seg_h, Y1 = min(P.y_end, Y0 + seg_h);
    if (Y0 >= Y1) return;
    const int xl = max(0, X0 - H), xr = min(n1, X1 + H);
    const int Ylo = max(0, Y0 - H), Yhi = min(n1, Y1 + H);
    const unsigned sm = (unsigned)__cvta_generic_to_shared(ring2);
    {   // class rows (3, c), c = 0..6 = global classes 21..27
        double *ct = reinterpret_cast<double *>(reinterpret_cast<char *>(ring2) + CLS_OFF);
        for (int i = tid; i < 7 * 2 * 29; i += NT) ct[(i / 29) * CROW + i % 29] = P.C[21 * 58 + i];
    }
    // ring columns 224 .. STRIDE-1 are guards no row load covers: zero once
    for (int i = tid; i < RING * (STRIDE - LCOLS); i += NT)
        sts2(sm + (unsigned)(i / (STRIDE - LCOLS)) * RS +
                 (unsigned)(LCOLS + i % (STRIDE - LCOLS)) * 16u,
             make_double2(0.0, 0.0));
    const int rmax = min(Yhi, n1 - 1);

    // one row of r into its ring slot: ring column lc (global xl - GL + lc)
    // of both fields, zero outside [xl, xr) and outside the domain's rows
    auto load_col = [&](int lc, int lry, unsigned slot) {
        const int gx = xl - GL + lc, row = Ylo + lry;
        const bool ok = gx >= xl && gx < xr && row >= 0 && row <= rmax;
        const unsigned dst = sm + slot * RS + (unsigned)lc * 16u;
        const double *src = ok ? P.rin + (int64_t)row * n1 + gx : P.rin;
        mcs_cp8(dst, src, ok);
        mcs_cp8(dst + 8, ok ? src + P.fs_in : P.rin, ok);
    };
    for (int e = tid; e < (AHEAD + 1) * LCOLS; e += NT)
        load_col(e % LCOLS, e / LCOLS - 1, (unsigned)(e / LCOLS));
    mcs_commit();
    const int S_end = (Y1 - 1 - Ylo) + RETIRE + 1;
    const unsigned mb = sm + MB_OFF;
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mb_init(mb + 8u * i, NC + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    mcs_wait<0>();
    __syncthreads();

    if (w == NWARP) {
        // ---- the boundary warp (no window to keep: its own loop, the same
        // step barriers).  Lane (side, q) takes the vertex of colour position
        // q (row S - 3q) in the three boundary columns at that side of an
        // interior row, with its class row from shared memory.  The loop
        // carries only the lane's window of steps; everything else is
        // recomputed where there is work (state pushed into local memory
        // costs ~300 cycles a reload here -- L1 is nearly all shared memory
        // --, which made this the slowest warp of every step).
        const int side = lane / NC, q = lane - side * NC;
        int Slo = 0, Sw = 0;  // steps at which position q has an interior row in its valid range
        if (lane < 2 * NC && !(MC2_X & 8) && (side == 0 ? xl == 0 : xr == n1)) {
            const int mg = 2 * (NC - 1 - q) + 1;
            const int ylo_q = max(max(Ylo, Y0 - mg), 3), yhi_q = min(min(Yhi, Y1 + mg), n1 - 3);
            Slo = ylo_q - Ylo + 3 * q;
            Sw = max(yhi_q - ylo_q, 0);
        }
        const bool brows = (Ylo < 3 || Yhi > n1 - 3) && !(MC2_X & 16);
        // the loop's per-lane state lives in shared memory, and the step
        // counter is parked there across the work (the register allocator
        // otherwise keeps them in local memory for the whole loop)
        __shared__ int bw_state[3 * 32];
        bw_state[lane] = Slo;
        bw_state[32 + lane] = Sw;
        const unsigned bw_base = (unsigned)__cvta_generic_to_shared(bw_state);  // CTA-uniform
        auto lds_i = [](unsigned a) {
            int v;
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
            return v;
        };
#ifdef MC2_PROF
        long long pw = 0, pc = 0, pa = 0;
        const long long pstart = clock64();
#endif
#pragma unroll 1
        for (int S = 0; S < S_end; ++S) {
            MC2_T(t0);
            if (S > 0) mb_wait(mb + 8u * ((S - 1) % 3), (unsigned)(((S - 1) / 3) & 1));
            MC2_T(t1);
            // (lane-derived values are recomputed from %laneid each step
            // rather than carried: carried, they went to local memory)
            unsigned lid;
            asm volatile("mov.u32 %0, %%laneid;" : "=r"(lid));
            const unsigned bws = bw_base + 4u * lid;
            const int lane = (int)lid, side = lane / NC, q = lane - side * NC;
            asm volatile("st.shared.s32 [%0], %1;" ::"r"(bws + 256u), "r"(S) : "memory");
            if ((unsigned)(S - lds_i(bws)) < (unsigned)lds_i(bws + 128u)) {
                const int colour = FWD ? q : NC - 1 - q;
                const int mg = 2 * (NC - 1 - q) + 1;
                const int c0 = side == 0 ? 0 : n1 - 3;
                const int xlo_q = max(xl, X0 - mg), xhi_q = min(xr, X1 + mg);
                const unsigned cls_s = sm + CLS_OFF;
                const int rq = S - 3 * q, yb = Ylo + rq;
                const int ob = pmod7(colour - 2 * yb - c0);
                const int xb = c0 + ob;
                if (ob < 3 && xb >= xlo_q && xb < xhi_q) {
                    const unsigned cb = (unsigned)(xb - xl + GL) * 16u;
                    const int sl = rq % RING;  // slot of row yb - 1
                    const unsigned bB = sm + (unsigned)sl * RS + cb;
                    const unsigned bC = sm + (unsigned)((sl + 1) % RING) * RS + cb;
                    const unsigned bU = sm + (unsigned)((sl + 2) % RING) * RS + cb;
                    double2 u[7];
                    u[0] = lds2(bB - 16); u[1] = lds2(bB);
                    u[2] = lds2(bC - 16); u[3] = lds2(bC); u[4] = lds2(bC + 16);
                    u[5] = lds2(bU); u[6] = lds2(bU + 16);
                    const unsigned cs = cls_s + (unsigned)(p1_axis_class(xb, n1) * 2) * (CROW * 8);
                    const unsigned ca = cs + (FWD ? 0 : CROW * 8), cb2 = cs + (FWD ? CROW * 8 : 0);
                    double pa, pb;
                    node_update_pair_s(u, ca, cb2, pa, pb);
                    sts2(bB - 16, u[0]); sts2(bB, u[1]);
                    sts2(bC - 16, u[2]); sts2(bC, u[3]); sts2(bC + 16, u[4]);
                    sts2(bU, u[5]); sts2(bU + 16, u[6]);
                    if ((unsigned)(yb - Y0) < (unsigned)(Y1 - Y0) &&
                        (unsigned)(xb - X0) < (unsigned)(X1 - X0))
                        sts2(sm + D_OFF + (unsigned)((rq + 1) % DRING) * DS + (unsigned)(xb - X0) * 16u,
                             make_double2(FWD ? pa : pb, FWD ? pb : pa));
                }
            }
            // a boundary row (y < 3 or y > n1 - 4) among the rows computed
            // this step: at most one per end of the domain (they are 3
            // apart), and only in the first 3 + 3 * 7 steps of a CTA at the
            // bottom, from row n1 - 3 on at the top.  Lane = segment, every
            // column with its own class row.
            if (brows && (Ylo + S < 3 + 3 * NC || Ylo + S >= n1 - 3)) {
                for (int qq = 0; qq < NC; ++qq) {
                        const int rr = S - 3 * qq, y = Ylo + rr;
                        if (rr < 0 || y >= Yhi || (unsigned)(y - 3) <= (unsigned)(n1 - 7)) continue;
                        const int mgq = 2 * (NC - 1 - qq) + 1;
                        if (y < max(Ylo, Y0 - mgq) || y >= min(Yhi, Y1 + mgq)) continue;
                        const int x = xl - pmod7(xl + 2 * y) + 7 * lane + (FWD ? qq : 6 - qq);
                        if (x >= max(xl, X0 - mgq) && x < min(xr, X1 + mgq)) {
                            const unsigned cb = (unsigned)(x - xl + GL) * 16u;
                            const int sl = rr % RING;  // slot of row y - 1
                            const unsigned s1 = (unsigned)((sl + 1) % RING);
                            const double *Cc =
                                P.C + (7 * p1_axis_class(y, n1) + p1_axis_class(x, n1)) * 58;
                            mc2_boundary_row_vertex<FWD>(
                                Cc, sm + (unsigned)sl * RS + cb, sm + s1 * RS + cb,
                                sm + (unsigned)((sl + 2) % RING) * RS + cb,
                                sm + D_OFF + (unsigned)((rr + 1) % DRING) * DS + (unsigned)(x - X0) * 16u,
                                (unsigned)(y - Y0) < (unsigned)(Y1 - Y0) &&
                                    (unsigned)(x - X0) < (unsigned)(X1 - X0));
                        }
                    }
            }
            unsigned lid2;  // (again: not carried across the work)
            asm volatile("mov.u32 %0, %%laneid;" : "=r"(lid2));
            S = lds_i(bw_base + 256u + 4u * lid2);
            MC2_T(t2);
            mb_arrive_warp(mb + 8u * (S % 3));
#ifdef MC2_PROF
            pw += t1 - t0;
            pc += t2 - t1;
            pa += clock64() - t2;
#endif
        }
#ifdef MC2_PROF
        if (lane == 0) {
            unsigned long long *o = mc2_prof + ((size_t)blockIdx.x * 24 + w) * 4;
            o[0] = pw; o[1] = pc; o[2] = pa; o[3] = clock64() - pstart;
        }
#endif
        return;
    }

    // ---- the 21 row warps.  Group grp = w % 3 computes at steps S = grp
    // (mod 3), retires a row at the step after and loads one at the step
    // after that.
    const int grp = w % 3, m = w / 3;
    // this lane's segment: the rows of a warp are 21 apart, 2 * 21 = 0 (mod
    // 7), so it starts at the same column in every row
    // columns: positions of the segment that are the lane's (in a colour's
    // valid region, not a boundary column) and that the tile owns
    // (packed: bits 0-6 the lane's, 8-14 owned)
    unsigned cm = 0;  // (built here, parked in shared memory below)
    {
        const int xs0 = xl - pmod7(xl + 2 * (Ylo + w)) + 7 * lane;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int x = FWD ? xs0 + q : xs0 + 6 - q, mg = 2 * (NC - 1 - q) + 1;
            const bool okc = x >= max(xl, X0 - mg) && x < min(xr, X1 + mg);
            cm |= (unsigned)(okc && x >= 3 && x <= n1 - 4) << q;
            cm |= (unsigned)(x >= X0 && x < X1) << (8 + q);
        }
    }
    // ring column (bytes) of position 0; the delta column is db_u further
    const unsigned cb0_ =
        (unsigned)(xl - pmod7(xl + 2 * (Ylo + w)) + 7 * lane + (FWD ? 0 : 6) - xl + GL) * 16u;
    // what only the per-row setup needs is parked in shared memory per thread
    // (2 x 4 bytes): the loop is at the register limit of 22 warps (80), and
    // a value pushed into local memory costs ~300 cycles per reload
    __shared__ unsigned park[2 * NWARP * 32];
    park[tid] = cm;
    park[NWARP * 32 + tid] = cb0_;
    const unsigned park_a = (unsigned)__cvta_generic_to_shared(park) + 4u * tid;
    const unsigned db_u = (unsigned)(xl - GL - X0) * 16u;

    // compute state
    int ry = m ? w - NWARP : w;  // relative row (y = Ylo + ry); a virtual one first for m > 0
    unsigned mask2 = 0, omask = 0;   // bit q + 1 / bit q: position q is the lane's / owned
    unsigned aB = 0, aC = 0, aU = 0, aD = 0;  // ring addresses of position 0
    bool rowact = false;
    // the window: v[0..6] = (x-1,y-1) (x,y-1) (x-1,y) (x,y) (x+1,y) (x,y+1) (x+1,y+1).
    // The position is a run-time value and the four inherited entries are
    // moved between positions (16 register moves): one copy of the vertex
    // code for all 21 row warps.  With a copy per position (static window
    // slots, no moves) the warps of a scheduler ran 7 different code paths
    // plus the duties, more than its instruction cache holds, and a compute
    // step took 650 cycles instead of the ~250 of its dependent chain.
    double2 v[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) v[d] = make_double2(0.0, 0.0);

    auto setup = [&]() {  // masks and addresses of row ry
        unsigned cm, cb0;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cm) : "r"(park_a) : "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cb0) : "r"(park_a + 4u * NWARP * 32) : "memory");
        const int y = Ylo + ry;
        // (the boundary rows y < 3, y > n1 - 4 are the boundary warp's)
        rowact = ry >= 0 && y < Yhi && (unsigned)(y - 3) <= (unsigned)(n1 - 7);
        // rows: colour position q is valid in [max(Ylo, Y0 - 13 + 2q), min(Yhi, Y1 + 13 - 2q))
        const int qr = min((y - Y0 + 13 + 300) / 2 - 150, (Y1 + 12 - y + 300) / 2 - 150);
        const unsigned rmask = qr >= 6 ? 0x7Fu : qr < 0 ? 0u : (2u << qr) - 1u;
        const unsigned mk = rowact ? (cm & rmask) : 0u;
        mask2 = mk << 1;
        omask = (unsigned)(y - Y0) < (unsigned)(Y1 - Y0) ? (mk & (cm >> 8)) : 0u;
        const unsigned cslot = (unsigned)((ry + RING) % RING);  // slot of row y - 1
        const unsigned s1 = cslot + 1 >= RING ? cslot + 1 - RING : cslot + 1;
        const unsigned s2 = s1 + 1 >= RING ? s1 + 1 - RING : s1 + 1;
        aB = sm + cslot * RS + cb0;
        aC = sm + s1 * RS + cb0;
        aU = sm + s2 * RS + cb0;
        aD = sm + D_OFF + (unsigned)((ry + 1 + DRING) % DRING) * DS + cb0 + db_u;
    };

    auto compute = [&](int k) {
        if (!rowact || (MC2_X & 1)) return;  // warp-uniform
        const unsigned dk = (unsigned)((FWD ? k : -k) * 16);
        // (MC2_X timing experiments: 64 every lane owns and inherits, 32 no
        // window moves, 256 no vertex updates)
        const bool own = (MC2_X & 64) ? true : (bool)((mask2 >> (k + 1)) & 1u);
        const bool prev = (MC2_X & 64) ? true : (bool)((mask2 >> k) & 1u);
        const bool next = (MC2_X & 64) ? true : (bool)((mask2 >> (k + 2)) & 1u);
        const unsigned b = aB + dk, c = aC + dk, u = aU + dk;
        // the three entries that enter the window are loaded by every lane
        // (always inside the ring), so that only the four inherited ones are
        // live from one position to the next
        const bool full = own && !prev;  // the window is not inherited: load all of it
        if (FWD) {
            if (!(MC2_X & 32)) { v[0] = v[1]; v[2] = v[3]; v[3] = v[4]; v[5] = v[6]; }
            v[1] = lds2(b); v[4] = lds2(c + 16); v[6] = lds2(u + 16);
            lds2_if(v[0], b - 16, full); lds2_if(v[2], c - 16, full);
            lds2_if(v[3], c, full); lds2_if(v[5], u, full);
        } else {
            if (!(MC2_X & 32)) { v[6] = v[5]; v[4] = v[3]; v[3] = v[2]; v[1] = v[0]; }
            v[0] = lds2(b - 16); v[2] = lds2(c - 16); v[5] = lds2(u);
            lds2_if(v[1], b, full); lds2_if(v[3], c, full);
            lds2_if(v[4], c + 16, full); lds2_if(v[6], u + 16, full);
        }
        double pa = v[3].x, pb = v[3].y;
        if (!(MC2_X & 256)) {
            pa = mcs::node_update_u<FWD ? 0 : 1>(v, P.cu);
            pb = mcs::node_update_u<FWD ? 1 : 0>(v, P.cu);
        }
        const bool rest = own && !next;  // the next vertex does not inherit: store all of it
        if (FWD) {
            sts2_if(b - 16, v[0], own); sts2_if(c - 16, v[2], own); sts2_if(u, v[5], own);
            sts2_if(b, v[1], rest); sts2_if(c, v[3], rest);
            sts2_if(c + 16, v[4], rest); sts2_if(u + 16, v[6], rest);
        } else {
            sts2_if(b, v[1], own); sts2_if(c + 16, v[4], own); sts2_if(u + 16, v[6], own);
            sts2_if(b - 16, v[0], rest); sts2_if(c - 16, v[2], rest);
            sts2_if(c, v[3], rest); sts2_if(u, v[5], rest);
        }
        sts2_if(aD + dk, make_double2(FWD ? pa : pb, FWD ? pb : pa),
                ((omask >> k) & 1u) && !(MC2_X & 128));
    };

    // A thread per column: gt = the thread's index in its group.
    const int gt = m * 32 + lane;
    auto retire = [&](int S) {
        const int R = Ylo + S - RETIRE;
        const unsigned rslot = (unsigned)(S + RING - RETIRE + 1) % RING;
        mcs_wait<1>();
        if (gt < X1 - X0 && !(MC2_X & 2)) {
            if (R >= Y0 && R < Y1) {
                const double2 rv = lds2(sm + rslot * RS + (unsigned)(X0 - xl + GL + gt) * 16u);
                const double2 dv =
                    lds2(sm + D_OFF + (unsigned)((S - RETIRE + 1) % DRING) * DS + (unsigned)gt * 16u);
                const double2 xv = lds2(sm + X_OFF + (unsigned)(R % XSLOTS) * DS + (unsigned)gt * 16u);
                const int64_t idx = (int64_t)R * n1 + X0 + gt;
                P.rout[idx] = rv.x;
                P.rout[P.fs_out + idx] = rv.y;
                P.x[idx] = __dadd_rn(xv.x, dv.x);
                P.x[P.fs_x + idx] = __dadd_rn(xv.y, dv.y);
            }
            const int R3 = R + 3;  // this thread's next retiring row: stage its x
            if (R3 >= Y0 && R3 < Y1) {
                const double *src = P.x + (int64_t)R3 * n1 + X0 + gt;
                const unsigned dst = sm + X_OFF + (unsigned)(R3 % XSLOTS) * DS + (unsigned)gt * 16u;
                mcs_cp8(dst, src, true);
                mcs_cp8(dst + 8, src + P.fs_x, true);
            }
        }
        mcs_commit();
    };

    // ---- load relative row S + AHEAD: this thread's ring column (the
    // group's previous row has had three steps to land and the group's next
    // arrival at a step barrier publishes it; the x staged just before may
    // still be in flight)
    auto load = [&](int S) {
        const unsigned lslot = (unsigned)(S + AHEAD + 1) % RING;
        mcs_wait<1>();
        if (Ylo + S + AHEAD <= Yhi && !(MC2_X & 4)) load_col(gt, S + AHEAD, lslot);
        mcs_commit();
    };

    int S = 0;
    auto step = [&]() {
        ++S;
    };
    // the duties of a group run between its compute steps, off the chain of
    // step barriers; they are written for "step S" = the step they would
    // take in a lock-step schedule (retire: the step after the group's
    // compute, load: the one after that)
    if (grp == 2) {
        retire(S);
        step();
    }
    if (grp >= 1) {
        load(S);
        step();
    }
    // S == grp: the warp's first compute step.  Warp w = grp + 3m computes
    // row ry at S = ry + 3k, so it enters at position (7 - m) % 7 of the
    // virtual row w - 21 (m > 0).
    setup();
    int k = (NC - m) % NC;
#ifdef MC2_PROF
    long long pw = 0, pc = 0, pd = 0;
    const long long pstart = clock64();
#endif
    for (;;) {
        if (S >= S_end) break;
        MC2_T(t0);
        if (S > 0) mb_wait(mb + 8u * ((unsigned)(S + 2) % 3), (unsigned)(((S - 1) / 3) & 1));
        MC2_T(t1);
        compute(k);
        mb_arrive_warp(mb + 8u * ((unsigned)S % 3));
        MC2_T(t2);
#ifdef MC2_PROF
        pw += t1 - t0;
        pc += t2 - t1;
#endif
        step();
        if (S >= S_end) break;
        retire(S);
        step();
        if (S >= S_end) break;
        load(S);
        if (++k == NC) {  // the next row's masks and addresses
            k = 0;
            ry += NWARP;
            setup();
        }
        step();
#ifdef MC2_PROF
        pd += clock64() - t2;
#endif
    }
#ifdef MC2_PROF
    if (lane == 0) {
        unsigned long long *o = mc2_prof + ((size_t)blockIdx.x * 24 + w) * 4;
        o[0] = pw; o[1] = pc; o[2] = pd; o[3] = clock64() - pstart;
    }
#endif
    mcs_wait<0>();
}

// Which one-launch kernel the multicolour sweep uses: k_p1_mc_sweep, unless
// OCMG_MC_SWEEP=roll asks for the rolling-window kernel of this file (both
// are bit-identical to the 7-pass form).  Measured at L12 on a B200
// (bench.py --quick): ring 0.350 ms, roll 0.411 ms per sweep -- see the
// notes at the top of this file and DESIGN.md section 3 for why it is not the
// default.
inline bool mc_use_roll() {
    static const bool v = [] {
        const char *e = std::getenv("OCMG_MC_SWEEP");
        return e && std::strcmp(e, "roll") == 0;
    }();
    return v;
}

inline McsPlan mc_plan(int n1, int sm_count, int rows = -1) {
    if (!mc_use_roll()) return mcs_plan(n1, sm_count, rows);
    McsPlan p;
    if (rows < 0) rows = n1;
    p.nstrips = (n1 + mc2::W - 1) / mc2::W;
    const int max_seg = std::max(1, rows / MCS_MIN_SEG_ROWS);
    const int total = std::max(p.nstrips, std::min(sm_count, p.nstrips * max_seg));
    p.base = total / p.nstrips;
    p.rem = total % p.nstrips;
    p.grid = p.nstrips * (p.base + (p.rem ? 1 : 0));
    return p;
}

inline void mc_launch(const McsParams &P, int grid, cudaStream_t s) {
    if (!mc_use_roll()) return mcs_launch(P, grid, s);
    // a strip next to the first / last one must not reach the boundary columns
    OCMG_REQUIRE(P.nstrips == 1 || P.n1 / P.nstrips >= mcs::H + 3,
                 "level too narrow for the strip decomposition");
    OCMG_REQUIRE(((uintptr_t)P.rin & 7) == 0 && ((uintptr_t)P.rout & 7) == 0 &&
                     ((uintptr_t)P.x & 7) == 0,
                 "vectors must be 8-byte aligned");
    if (P.forward)
        OCMG_LAUNCH(k_p1_mc_roll<true>, grid, mc2::NT, mc2::SMEM, s, P);
    else
        OCMG_LAUNCH(k_p1_mc_roll<false>, grid, mc2::NT, mc2::SMEM, s, P);
}

inline void mc2_set_smem() {
    OCMG_CUDA(cudaFuncSetAttribute(k_p1_mc_roll<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mc2::SMEM));
    OCMG_CUDA(cudaFuncSetAttribute(k_p1_mc_roll<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mc2::SMEM));
}

}  // namespace ocmg
