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
// Pipelining.  Colour q at row y reads r on rows y-1..y+1 and writes the
// same rows; colour q+1 at row y' needs colour q finished on rows <= y'+2.
// A CTA streams its rows bottom to top in supersteps of K = 2 rows: colour
// q updates rows K S - C q + {0, 1} at superstep S (skew C = K + 2 rows), so
// the 14 colour-rows of a superstep touch disjoint rows and are independent;
// one __syncthreads per superstep.  Warp q owns colour q; its lane m the
// m-th vertex of that colour in each of the two rows (7 columns apart), so
// every lane has two independent vertex updates per superstep.
//
// Shared memory (one CTA per SM, 8 compute warps + 6 duty warps, 211 KB):
//  * the r ring: 34 rows of (state, adjoint) pairs over the tile plus halo;
//    a neighbour is one 16-byte access and a vertex's two unknown updates
//    share one load and one store of its neighbourhood;
//  * the x ring: the owned columns of the same rows.  x is loaded with the
//    row (coalesced) and written back with it when the row is final, so a
//    lane never touches x in global memory (a warp's vertices are 56 bytes
//    apart: 13 cache lines per access when it did);
//  * the class rows (3, c) of the boundary columns.
// Rows arrive by cp.async two supersteps ahead (zero-filled outside the
// domain) and leave, r to r_out and x in place, LAG = 27 rows behind.
//
// Boundary classes.  In interior rows only columns 0..2 and n1-3..n1-1 have
// other classes.  Their vertices belong to the eighth warp: its lane
// (side, q, i) takes the (at most one) vertex of colour-warp q, row i in the
// three columns at that side, with the class row from shared memory, while
// the colour warps run the interior class on every lane (lanes outside the
// computed region discard their results).  So the edge strips cost what the
// others do.  The top and bottom three rows read per-lane class rows from
// the global table.
//
// Decomposition.  A CTA owns W = 176 columns (balanced strips) x seg_h rows.
// The valid region of r shrinks by 2 columns (rows) per colour, so it loads
// its tile plus a halo of H = 14 on every side, recomputes the halo (only
// where the result can reach the tile: margin 2(6-q)+1 for colour q) and
// writes only its own tile.  Halos are read from r_in and the tile is
// written to r_out (out of place: neighbours read what this CTA
// overwrites); x is updated in place by the owning CTA.  Strips get base or
// base+1 row segments so the grid fills the SMs once.
#pragma once

#include "ocmg_p1.cuh"

namespace ocmg {
namespace mcs {
#ifndef MCS_K
#define MCS_K 2
#endif
#ifndef MCS_D
#define MCS_D 2
#endif
#ifndef MCS_W
#define MCS_W 176
#endif
constexpr int NC = kMcColours;     // 7
constexpr int H = 2 * NC;          // 2 columns (rows) per colour
constexpr int K = MCS_K;           // rows per colour and superstep
constexpr int C = K + 2;           // row skew between consecutive colours
// superstep S stores rows Ylo + K S - LAG + i (i < K): final once colour 6
// has passed them
constexpr int LAG = (NC - 1) * C + 1 + K;
constexpr int D = MCS_D;           // cp.async prefetch distance (supersteps)
// live rows: the K leaving (LAG behind) .. the K D + K rows in flight
constexpr int RING = K * D + K + LAG + 1;
#ifndef MCS_WPC
#define MCS_WPC 1
#endif
// warps per colour: each takes K / WPC of the colour's K rows per superstep.
// WPC = 2 (15 warps of 128 registers instead of 8 of 240) measured the same
// 0.439 ms at L12 as WPC = 1: the superstep is bound by the shared-memory
// pipe (~1100 wavefronts of ~2150 cycles) and issue, not by latency hiding
constexpr int WPC = MCS_WPC;
constexpr int KW = K / WPC;          // rows per colour warp and superstep
static_assert(K % WPC == 0, "rows per superstep split evenly over a colour's warps");
#ifndef MCS_ND
#define MCS_ND 6
#endif
// duty warps: they load the rows (cp.async) and write the final ones back
// while the colour warps compute.  With MCS_ND = 0 every thread shares the
// duties before its vertex updates, as in round 1: ncu's source page put 37%
// of a colour warp's time into that part (200 instructions of predicates,
// selects and 64-bit pointer arithmetic in front of the 200 of the update).
constexpr int ND = MCS_ND;
constexpr int NCW = NC * WPC + 1;        // colour warps + the boundary-column warp
constexpr int NT = 32 * (NCW + ND);
constexpr int NDT = ND ? 32 * ND : NT;   // threads that share the duties
constexpr int W = MCS_W;           // owned columns per CTA (at most)
constexpr int STRIDE = W + 2 * H + 2;  // r ring row: columns xl-1 .. xr
constexpr int RS = STRIDE * 16;    // r ring row bytes: (state, adjoint) pairs
constexpr int XS = W * 16;         // x ring row bytes: owned columns' pairs
constexpr int CROW = 30;           // class row: W (14), A (14), 1/n_diag, pad
// r ring, x ring (slots of the r ring, owned columns), the class rows (3, c)
// of boundary columns in interior rows.  Lanes outside the tile read (and
// discard) up to 19 r entries past a row end, inside the x ring at worst.
constexpr int X_OFF = RING * RS;
constexpr int CLS_OFF = X_OFF + RING * XS;
constexpr int FLG_OFF = CLS_OFF + 7 * 2 * CROW * 8;  // progress counters (MCS_CHAIN)
constexpr int SMEM = FLG_OFF + 64;
#ifndef MCS_CHAIN
#define MCS_CHAIN 0
#endif
// MCS_CHAIN = 1 (measured, not the default): no CTA barrier per superstep.
// Every warp publishes the number of supersteps it has finished (release
// store to a shared counter) and polls only what it reads: colour q at
// superstep S for colour q-1 (and the boundary warp) at S-1, colour 0 for the
// rows' loads, the write-back of rows for colour 6, the boundary warp for all
// colours at S-1.  The idea was that the warps drift apart by up to a
// superstep, so that one warp's shared-memory burst overlaps another's FMA
// chains (with the CTA barrier all 7 bursts come first, then all chains:
// 784 + ~480 cycles).  Bit-identical (L7-L12, strips, fused block), and
// slower: 0.478 ms per L12 sweep against 0.349 ms -- the release store costs
// a colour warp ~230 cycles per superstep (ncu: long_sb at the store after
// MEMBAR.ALL.CTA) and the warps still wait ~200 cycles per superstep for
// their predecessor, as they did at the barrier.  (With one polling lane per
// warp it was 0.66 ms: the warp stayed split in two after the poll and
// executed every superstep twice.)
constexpr bool CHAIN = MCS_CHAIN != 0 && ND != 0;
// counters (32-bit, shared): done[q] (q < 7), boundary warp (7), loads landed per duty warp (8 ..)
constexpr int F_BW = 7, F_LD = 8;
static_assert(F_LD + ND <= 16, "flag words");
constexpr int NLD = (2 * STRIDE + 2 * W + NDT - 1) / NDT;  // row-load entries per duty thread
constexpr int NST = (2 * W + NDT - 1) / NDT;               // row-store pairs per duty thread
static_assert((W + 2 * H + 6) / 7 <= 31, "one warp per colour-row, lane 31 free");
static_assert(SMEM + 1024 <= 228 * 1024, "one CTA per SM");

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

// The interior class (3,3) row has the stencil's symmetry bitwise: M has a
// centre and one neighbour value, K a centre, an axis and a diagonal value
// (d = 0 and 6 are the SW-NE diagonal neighbours, d = 3 the vertex).  So the
// 58 interior coefficients are 19 distinct doubles: A values {m1, m0, kd, ka,
// k0, -m1/a, -m0/a} (0-6), state-unknown W {M nbr, M centre, K diag, K axis,
// K centre} (7-11), adjoint-unknown W {K diag, K axis, K centre, M nbr,
// M centre} (12-16), 1/n_diag state, adjoint (17, 18).  umap(f, i) is the
// distinct index of slot i (node_update layout) of field f; the host checks
// every slot against it (mcs_fill_cu).
constexpr int NU = 19;
__host__ __device__ constexpr int mcls(int d) { return d == 3 ? 1 : 0; }
__host__ __device__ constexpr int kcls(int d) { return d == 3 ? 2 : (d == 0 || d == 6) ? 0 : 1; }
__host__ __device__ constexpr int umap(int f, int i) {
    return f == 0 ? (i < 7 ? 7 + mcls(i) : i < 14 ? 9 + kcls(i - 7) : i < 21 ? mcls(i - 14)
                     : i < 28 ? 2 + kcls(i - 21) : 17)
                  : (i < 7 ? 12 + kcls(i) : i < 14 ? 15 + mcls(i - 7) : i < 21 ? 2 + kcls(i - 14)
                     : i < 28 ? 5 + mcls(i - 21) : 18);
}
// node_update on the interior class, coefficients from the distinct set
// (same operations in the same order, hence bit-identical)
template <int F>
__device__ __forceinline__ double node_update_u(double2 (&v)[7], const double (&u)[NU]) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        s0 = __fma_rn(u[umap(F, d)], v[d].x, s0);
        s1 = __fma_rn(u[umap(F, 7 + d)], v[d].y, s1);
    }
    const double p = __dmul_rn(__dadd_rn(s0, s1), u[umap(F, 28)]);
#pragma unroll
    for (int d = 0; d < 7; ++d)
        v[d] = make_double2(__fma_rn(-u[umap(F, 14 + d)], p, v[d].x),
                            __fma_rn(-u[umap(F, 21 + d)], p, v[d].y));
    return p;
}
}  // namespace mcs

struct McsParams {
    int n1, nstrips, base, rem, forward;
    int y_begin, y_end;        // rows this launch owns (a rank's strip; 0, n1)
    int64_t fs_in, fs_out, fs_x;  // field strides of rin / rout / x
    double cu[mcs::NU];  // interior class (3,3), distinct values (mcs::umap)
    const double *C;   // [49][2][29]: W row, A row, 1/n_diag per (class, field)
    // addressed by global vertex index y*n1+x (+ field * fs_*): rin must hold
    // rows [y_begin-15, y_end+15) of the domain, rout and x rows
    // [y_begin, y_end); a rank passes base pointers shifted by its slab start
    const double *rin;
    double *rout, *x;
};

// cp.async of one double (zero-filled when !valid): ring rows are filled
// without passing through registers
__device__ __forceinline__ void mcs_cp8(unsigned dst, const double *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void mcs_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void mcs_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double2 mcs_lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void mcs_sts2(unsigned a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// predicated store (no branch: a divergent region around the stores of the
// lanes at a tile's edge costs the whole warp ~50 cycles)
__device__ __forceinline__ void mcs_sts2_if(unsigned a, double2 v, bool p) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.s32 q, %3, 0;\n@q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a),
                 "d"(v.x), "d"(v.y), "r"((int)p)
                 : "memory");
}
// progress counters in shared memory: one warp publishes (its lanes' earlier
// shared-memory accesses ordered before it through __syncwarp + release), any
// warp polls
__device__ __forceinline__ void mcs_flag_set(unsigned a, int v) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
#ifndef MCS_DUTY_RELEASE
#define MCS_DUTY_RELEASE 0
#endif
#ifndef MCS_POLL_NS
#define MCS_POLL_NS 0
#endif
// the same without a fence of the publishing thread: for a warp whose data
// was made visible by a barrier it has just passed (the duty warps: a
// release fence there also waits for their global stores, ~1 us a superstep)
__device__ __forceinline__ void mcs_flag_set_relaxed(unsigned a, int v) {
    if ((threadIdx.x & 31) == 0)
        asm volatile("st.relaxed.cta.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void mcs_flag_wait(unsigned a, int need) {
    int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    while (v < need) {
        if (MCS_POLL_NS) __nanosleep(MCS_POLL_NS);
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    }
}
// node_update with the coefficient row in shared memory (cs: its address,
// 16-byte aligned; asm volatile keeps the 15 loads next to their use)
__device__ __forceinline__ double node_update_s(double2 (&v)[7], unsigned cs) {
    double c[30];
#pragma unroll
    for (int i = 0; i < 15; ++i) {
        const double2 t = mcs_lds2(cs + 16 * i);
        c[2 * i] = t.x;
        c[2 * i + 1] = t.y;
    }
    return mcs::node_update(v, c);
}

template <bool FWD>
__global__ void __launch_bounds__(mcs::NT, 1) k_p1_mc_sweep(const __grid_constant__ McsParams P) {
    using namespace mcs;
    extern __shared__ __align__(16) double2 ring[];
    const int tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
    const int n1 = P.n1;
    const int strip = blockIdx.x % P.nstrips, seg = blockIdx.x / P.nstrips;
    const int nseg = P.base + (strip < P.rem ? 1 : 0);
    if (seg >= nseg) return;
    const int rows = P.y_end - P.y_begin;
    const int seg_h = (rows + nseg - 1) / nseg;
    // balanced strips of at most W columns
    const int X0 = strip * n1 / P.nstrips, X1 = (strip + 1) * n1 / P.nstrips;
    const int Y0 = P.y_begin + seg * seg_h, Y1 = min(P.y_end, Y0 + seg_h);
    if (Y0 >= Y1) return;
    const int xl = max(0, X0 - H), xr = min(n1, X1 + H);
    const int Ylo = max(0, Y0 - H), Yhi = min(n1, Y1 + H);
    const unsigned sm = (unsigned)__cvta_generic_to_shared(ring);
    char *const smc = reinterpret_cast<char *>(ring);
    auto wrap = [](int j) { return j >= RING ? j - RING : j; };
    if (tid < 16) reinterpret_cast<int *>(smc + FLG_OFF)[tid] = tid >= F_LD ? 1 : 0;  // rows of superstep 0 land before the first barrier
    {   // class rows (3, c), c = 0..6 = global classes 21..27
        double *ct = reinterpret_cast<double *>(smc + CLS_OFF);
        for (int i = tid; i < 7 * 2 * 29; i += NT) ct[(i / 29) * CROW + i % 29] = P.C[21 * 58 + i];
    }

    // ---- loader: row Ylo-1+m lives in slot m mod RING of both rings.
    // Entries [0, 2 STRIDE): r (field, local column incl. guards), zero
    // outside [xl, xr) and for rows past rmax; [2 STRIDE, 2 STRIDE + 2 W): x
    // (field, owned column), rows Y0 .. Y1-1 only.
    const int rmax = min(Yhi, n1 - 1);
    const bool duty = ND == 0 || q >= NCW;          // this thread shares the duties
    const int dt = ND ? tid - 32 * NCW : tid;       // its index among the duty threads
    bool lisx[NLD], lact[NLD], lhas[NLD];
    unsigned loff[NLD];
    const double *lp[NLD];  // entry's element in row Ylo-1 (a valid address if inactive)
#pragma unroll
    for (int e = 0; e < NLD; ++e) {
        const int t = dt + e * NDT;
        lhas[e] = duty && t < 2 * STRIDE + 2 * W;
        lisx[e] = t >= 2 * STRIDE;
        if (!lisx[e]) {
            const int f = t >= STRIDE, lc = t - f * STRIDE, gx = xl - 1 + lc;
            lact[e] = gx >= xl && gx < xr;
            loff[e] = sm + (unsigned)(2 * lc + f) * 8u;
            lp[e] = P.rin + (lact[e] ? f * P.fs_in + (int64_t)(Ylo - 1) * n1 + gx : 0);
        } else {
            const int v = t - 2 * STRIDE, f = v >= W, c = v - f * W, gx = X0 + c;
            lact[e] = lhas[e] && gx < X1;
            loff[e] = sm + X_OFF + (unsigned)(2 * c + f) * 8u;
            lp[e] = P.x + (lact[e] ? f * P.fs_x + (int64_t)(Ylo - 1) * n1 + gx : 0);
        }
    }
    int lrow = Ylo - 1;  // next row to load
    int lslot = 0;       // its slot
    auto load_row = [&]() {
        const bool okr = lrow >= 0 && lrow <= rmax, okx = lrow >= Y0 && lrow < Y1;
#pragma unroll
        for (int e = 0; e < NLD; ++e) {
            if (lhas[e]) {
                const bool ok = lact[e] && (lisx[e] ? okx : okr);
                mcs_cp8(loff[e] + (unsigned)lslot * (lisx[e] ? XS : RS), ok ? lp[e] : P.rin, ok);
            }
            if (lact[e]) lp[e] += n1;
        }
        ++lrow;
        lslot = wrap(lslot + 1);
    };
    // prologue: rows Ylo-1 .. Ylo+K (superstep 0), then K rows per superstep
    // 1 .. D-1, one commit group per superstep
    if (duty) {
        for (int j = 0; j < K + 2; ++j) load_row();
        mcs_commit();
        for (int g = 1; g < D; ++g) {
#pragma unroll
            for (int i = 0; i < K; ++i) load_row();
            mcs_commit();
        }
    }

    // ---- store role: thread -> NST entries t of each leaving row: t < W an
    // r pair (column X0+t), W <= t < 2W an x pair (column X0+t-W)
    bool sact[NST];
    double *sp[NST];
    int64_t sfs[NST];
    unsigned soff[NST], srs[NST];
#pragma unroll
    for (int e = 0; e < NST; ++e) {
        const int t = dt + e * NDT;
        const bool isx = t >= W;
        const int c = isx ? t - W : t;
        sact[e] = duty && t < 2 * W && X0 + c < X1;
        sp[e] = (isx ? P.x : P.rout) + (int64_t)(Ylo - LAG) * n1 + X0 + c;
        sfs[e] = isx ? P.fs_x : P.fs_out;
        soff[e] = isx ? sm + X_OFF + (unsigned)c * 16u : sm + (unsigned)(X0 - xl + 1 + c) * 16u;
        srs[e] = isx ? XS : RS;
    }
    int srow = Ylo - LAG;                          // next row to leave
    int sslot = (RING - (LAG - 1) % RING) % RING;  // its slot

    const int S_end = (Y1 - Ylo + LAG + K - 1) / K;
    auto duties = [&]() {
        // 1. the rows superstep S + D needs first
#pragma unroll
        for (int i = 0; i < K; ++i) load_row();
        mcs_commit();
        // 2. final rows leave (r pairs, x pairs)
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (srow >= Y0 && srow < Y1) {  // CTA-uniform
#pragma unroll
                for (int e = 0; e < NST; ++e)
                    if (sact[e]) {
                        const double2 v = mcs_lds2(soff[e] + (unsigned)sslot * srs[e]);
                        sp[e][0] = v.x;
                        sp[e][sfs[e]] = v.y;
                    }
            }
#pragma unroll
            for (int e = 0; e < NST; ++e) sp[e] += n1;
            ++srow;
            sslot = wrap(sslot + 1);
        }
    };
    const unsigned flg = sm + FLG_OFF;
    // the tile touches a side of the domain: the boundary warp has work
    const bool hb = xl == 0 || xr == n1;
    if (ND != 0 && q >= NCW) {
        // ---- the duty warps' loop
        mcs_wait<D - 1>();
        __syncthreads();
        for (int S = 0; S < S_end; ++S) {
            if (!CHAIN) {
                duties();
                mcs_wait<D - 1>();
                __syncthreads();
                continue;
            }
            // rows for superstep S + D in (their slots were freed by the
            // write-back of superstep S - 1: the duty warps' barrier below)
#pragma unroll
            for (int i = 0; i < K; ++i) load_row();
            mcs_commit();
            // final rows out: final once colour 6 (and the boundary warp) has finished S - 1
            // (every lane polls, the same word: with one polling lane the warp
            // stayed split in two for the rest of the iteration and executed
            // everything twice)
            mcs_flag_wait(flg + 4u * (NC - 1), S);
            if (hb) mcs_flag_wait(flg + 4u * F_BW, S);
#pragma unroll
            for (int i = 0; i < K; ++i) {
                if (srow >= Y0 && srow < Y1) {  // CTA-uniform
#pragma unroll
                    for (int e = 0; e < NST; ++e)
                        if (sact[e]) {
                            const double2 v = mcs_lds2(soff[e] + (unsigned)sslot * srs[e]);
                            sp[e][0] = v.x;
                            sp[e][sfs[e]] = v.y;
                        }
                }
#pragma unroll
                for (int e = 0; e < NST; ++e) sp[e] += n1;
                ++srow;
                sslot = wrap(sslot + 1);
            }
            mcs_wait<D - 1>();  // the rows of superstep S + 1 have landed (this thread's part)
            asm volatile("bar.sync 1, %0;" ::"n"(32 * (ND ? ND : 1)) : "memory");
#if MCS_DUTY_RELEASE
            mcs_flag_set(flg + 4u * (F_LD + (q - NCW)), S + 2);
#else
            mcs_flag_set_relaxed(flg + 4u * (F_LD + (q - NCW)), S + 2);
#endif
        }
        mcs_wait<0>();
        return;
    }

    // ---- compute roles.  Colour warp q = position q of the sweep (colour q
    // forward, 6 - q backward); at superstep S it updates rows
    // y_i = Ylo + K S - C q + i (i < K), its lane the vertex at column
    // xbase + o_i, o_i = (colour - xl - 2 y_i) mod 7.  Vertices of a
    // boundary column (x < 3 or x > n1-4) in an interior row belong to warp
    // 7 (the boundary warp): its lane (side, q', i) takes the one vertex of
    // colour-warp q' row i in the three columns at that side, with the
    // class row from shared memory.
    const bool bw = q == NC * WPC;
    const int qq = bw ? (lane % 14) / 2 : q / WPC;     // the colour (warp) emulated
    const int i0 = bw ? 0 : (q % WPC) * KW;            // colour warp: its first row
    const int bi = bw ? lane & 1 : 0;                  // boundary warp: its row i
    const int side = bw ? (lane < 14 ? 0 : lane < 28 ? 1 : 2) : 0;  // left, right, none
    const bool bside = bw && ((side == 0 && xl == 0) || (side == 1 && xr == n1));
    const int colour = FWD ? qq : NC - 1 - qq;
    const int mg = 2 * (NC - 1 - qq) + 1;  // margin whose result reaches the tile
    const int cxl = max(xl, X0 - mg), cxr = min(xr, X1 + mg);
    const int cyl = max(Ylo, Y0 - mg), cyh = min(Yhi, Y1 + mg);
    int y = Ylo - C * qq;  // y_0
    int o = (colour - xl - 2 * y) % 7;
    o += o < 0 ? 7 : 0;
    const int xbase = xl + 7 * lane;
    int sl = (RING - (C * qq) % RING) % RING;  // slot of row y_0 - 1
    double cu[NU];  // interior coefficients (uniform registers)
#pragma unroll
    for (int i = 0; i < NU; ++i) cu[i] = P.cu[i];
    const unsigned cls_s = sm + CLS_OFF;
    // The common superstep of a colour warp -- both rows interior and inside
    // the colour's valid rows -- runs on loop-carried state: the ring
    // addresses of rows y-1 .. y+2 and of the x rows, the two column offsets
    // (mod 7 by compare), and the lane's column windows relative to xbase
    // (its computed columns, its owned columns).  The general path below
    // recomputes all of it from y, o and sl each superstep (75 dependent
    // integer instructions in front of the first load, ~340 cycles).
    constexpr bool kFast = K == 2 && WPC == 1;
    const int fyA = max(cyl, 3), fyW = max(min(cyh, n1 - 3) - 1 - fyA, 0);  // y_0 range of a fast superstep
    const int fxlo = max(cxl, 3) - xbase, fxw = max(min(cxr, n1 - 3) - max(cxl, 3), 0);
    const int oxlo = X0 - xbase, oxw = X1 - X0;
    const unsigned cb = (unsigned)(xbase - xl + 1) * 16u, xb16 = (unsigned)(xbase - X0) * 16u;
    const unsigned r_end = sm + RING * RS, x_end = sm + X_OFF + RING * XS;
    auto nxt_r = [&](unsigned a) { return a + RS == r_end ? sm : a + RS; };
    auto nxt_x = [&](unsigned a) { return a + XS == x_end ? sm + X_OFF : a + XS; };
    unsigned ra0 = sm + (unsigned)sl * RS, ra1 = nxt_r(ra0), ra2 = nxt_r(ra1), ra3 = nxt_r(ra2);
    unsigned xa0 = sm + X_OFF + (unsigned)wrap(sl + 1) * XS, xa1 = nxt_x(xa0);
    mcs_wait<D - 1>();
    __syncthreads();
    if (CHAIN && bw && !hb) return;  // no boundary columns in this tile

    for (int S = 0; S < S_end; ++S) {
        if (ND == 0) duties();  // 1. rows for superstep S + D in, 2. final rows out
        if (CHAIN) {
            // (warp-uniform control flow: every lane polls the same words)
            if (bw) {  // every colour has finished S - 1
#pragma unroll
                for (int j = 0; j < NC; ++j) mcs_flag_wait(flg + 4u * j, S);
            } else {   // the colour before (and the boundary warp) has finished S - 1
                if (q > 0) mcs_flag_wait(flg + 4u * (q - 1), S);
                if (hb) mcs_flag_wait(flg + 4u * F_BW, S);
                // colour 0: the rows of this superstep have landed
                if (q == 0) {
#pragma unroll
                    for (int j = 0; j < ND; ++j) mcs_flag_wait(flg + 4u * (F_LD + j), S + 1);
                }
            }
        }
        if (kFast && !bw && (unsigned)(y - fyA) < (unsigned)fyW) {
            int o1 = o + 5;
            o1 -= o1 >= 7 ? 7 : 0;
            const unsigned c0 = cb + (unsigned)o * 16u, c1 = cb + (unsigned)o1 * 16u;
            double2 v0[7], v1[7];
            v0[0] = mcs_lds2(ra0 + c0 - 16); v0[1] = mcs_lds2(ra0 + c0);
            v0[2] = mcs_lds2(ra1 + c0 - 16); v0[3] = mcs_lds2(ra1 + c0); v0[4] = mcs_lds2(ra1 + c0 + 16);
            v0[5] = mcs_lds2(ra2 + c0); v0[6] = mcs_lds2(ra2 + c0 + 16);
            v1[0] = mcs_lds2(ra1 + c1 - 16); v1[1] = mcs_lds2(ra1 + c1);
            v1[2] = mcs_lds2(ra2 + c1 - 16); v1[3] = mcs_lds2(ra2 + c1); v1[4] = mcs_lds2(ra2 + c1 + 16);
            v1[5] = mcs_lds2(ra3 + c1); v1[6] = mcs_lds2(ra3 + c1 + 16);
            const unsigned xe0 = xa0 + xb16 + (unsigned)o * 16u, xe1 = xa1 + xb16 + (unsigned)o1 * 16u;
            const double2 xo0 = mcs_lds2(xe0), xo1 = mcs_lds2(xe1);
            const double pa0 = node_update_u<FWD ? 0 : 1>(v0, cu);
            const double pa1 = node_update_u<FWD ? 0 : 1>(v1, cu);
            const double pb0 = node_update_u<FWD ? 1 : 0>(v0, cu);
            const double pb1 = node_update_u<FWD ? 1 : 0>(v1, cu);
            const bool a0 = (unsigned)(o - fxlo) < (unsigned)fxw, a1 = (unsigned)(o1 - fxlo) < (unsigned)fxw;
            mcs_sts2_if(ra0 + c0 - 16, v0[0], a0); mcs_sts2_if(ra0 + c0, v0[1], a0);
            mcs_sts2_if(ra1 + c0 - 16, v0[2], a0); mcs_sts2_if(ra1 + c0, v0[3], a0);
            mcs_sts2_if(ra1 + c0 + 16, v0[4], a0);
            mcs_sts2_if(ra2 + c0, v0[5], a0); mcs_sts2_if(ra2 + c0 + 16, v0[6], a0);
            mcs_sts2_if(ra1 + c1 - 16, v1[0], a1); mcs_sts2_if(ra1 + c1, v1[1], a1);
            mcs_sts2_if(ra2 + c1 - 16, v1[2], a1); mcs_sts2_if(ra2 + c1, v1[3], a1);
            mcs_sts2_if(ra2 + c1 + 16, v1[4], a1);
            mcs_sts2_if(ra3 + c1, v1[5], a1); mcs_sts2_if(ra3 + c1 + 16, v1[6], a1);
            mcs_sts2_if(xe0,
                        make_double2(__dadd_rn(xo0.x, FWD ? pa0 : pb0), __dadd_rn(xo0.y, FWD ? pb0 : pa0)),
                        a0 && (unsigned)(y - Y0) < (unsigned)(Y1 - Y0) &&
                            (unsigned)(o - oxlo) < (unsigned)oxw);
            mcs_sts2_if(xe1,
                        make_double2(__dadd_rn(xo1.x, FWD ? pa1 : pb1), __dadd_rn(xo1.y, FWD ? pb1 : pa1)),
                        a1 && (unsigned)(y + 1 - Y0) < (unsigned)(Y1 - Y0) &&
                            (unsigned)(o1 - oxlo) < (unsigned)oxw);
        } else {
        // 3. vertex updates (independent: same colour, distance >= 3)
        auto rrow = [&](int j) {  // r ring row j (slot sl + j) as double2*
            return reinterpret_cast<double2 *>(smc + wrap(sl + j) * RS);
        };
        auto xent = [&](int i, int x) {  // x ring entry of (y_i, x)
            return reinterpret_cast<double2 *>(smc + X_OFF + wrap(sl + i + 1) * XS) + (x - X0);
        };
        auto load_v = [&](int i, int x, double2 (&v)[7]) {
            const int col = x - xl + 1;
            const double2 *rb = rrow(i) + col, *rc = rrow(i + 1) + col, *ru = rrow(i + 2) + col;
            v[0] = rb[-1]; v[1] = rb[0];
            v[2] = rc[-1]; v[3] = rc[0]; v[4] = rc[1];
            v[5] = ru[0]; v[6] = ru[1];
        };
        auto store_v = [&](int i, int x, const double2 (&v)[7]) {
            const int col = x - xl + 1;
            double2 *rb = rrow(i) + col, *rc = rrow(i + 1) + col, *ru = rrow(i + 2) + col;
            rb[-1] = v[0]; rb[0] = v[1];
            rc[-1] = v[2]; rc[0] = v[3]; rc[1] = v[4];
            ru[0] = v[5]; ru[1] = v[6];
        };
        auto x_update = [&](int i, int x, double pa, double pb) {
            double2 *xp = xent(i, x);
            const double2 xo = *xp;
            *xp = make_double2(__dadd_rn(xo.x, FWD ? pa : pb), __dadd_rn(xo.y, FWD ? pb : pa));
        };
        auto owned = [&](int i, int x) {
            return (unsigned)(y + i - Y0) < (unsigned)(Y1 - Y0) &&
                   (unsigned)(x - X0) < (unsigned)(X1 - X0);
        };
        auto in_rows = [&](int i) { return (unsigned)(y + i - cyl) < (unsigned)(cyh - cyl); };
        auto int_row = [&](int i) { return (unsigned)(y + i - 3) <= (unsigned)(n1 - 7); };
        auto int_col = [&](int x) { return (unsigned)(x - 3) <= (unsigned)(n1 - 7); };
        if (!bw) {
            int xi[KW];
            bool act[KW];
            bool allint = true;
#pragma unroll
            for (int ii = 0; ii < KW; ++ii) {
                const int i = i0 + ii;
                const int oi = (o - 2 * i + 7 * K) % 7;
                xi[ii] = xbase + oi;
                act[ii] = in_rows(i) && (unsigned)(xi[ii] - cxl) < (unsigned)(cxr - cxl);
                allint = allint && int_row(i);
                // boundary columns of interior rows: the boundary warp's
                act[ii] = act[ii] && (!int_row(i) || int_col(xi[ii]));
            }
            if (allint) {  // warp-uniform: every computed lane has the interior class
                double2 v[KW][7];
#pragma unroll
                for (int ii = 0; ii < KW; ++ii) load_v(i0 + ii, xi[ii], v[ii]);
                // x of the vertices, loaded with their neighbourhoods so that
                // the x update at the end is an add and a store (a halo
                // vertex reads some other entry of the rings and drops it)
                double2 xo[KW];
#pragma unroll
                for (int ii = 0; ii < KW; ++ii) xo[ii] = *xent(i0 + ii, xi[ii]);
                double pa[KW], pb[KW];  // first / second unknown in sweep order
#pragma unroll
                for (int ii = 0; ii < KW; ++ii) pa[ii] = node_update_u<FWD ? 0 : 1>(v[ii], cu);
#pragma unroll
                for (int ii = 0; ii < KW; ++ii) pb[ii] = node_update_u<FWD ? 1 : 0>(v[ii], cu);
#pragma unroll
                for (int ii = 0; ii < KW; ++ii)
                    if (act[ii]) {
                        store_v(i0 + ii, xi[ii], v[ii]);
                        if (owned(i0 + ii, xi[ii]))
                            *xent(i0 + ii, xi[ii]) =
                                make_double2(__dadd_rn(xo[ii].x, FWD ? pa[ii] : pb[ii]),
                                             __dadd_rn(xo[ii].y, FWD ? pb[ii] : pa[ii]));
                    }
            } else {  // a boundary row: per-lane class rows from the global table
#pragma unroll
                for (int ii = 0; ii < KW; ++ii) {
                    const int i = i0 + ii;
                    if (!in_rows(i)) continue;  // warp-uniform
                    double2 v[7];
                    load_v(i, xi[ii], v);
                    double pa, pb;
                    if (int_row(i)) {
                        pa = node_update_u<FWD ? 0 : 1>(v, cu);
                        pb = node_update_u<FWD ? 1 : 0>(v, cu);
                    } else {
                        const int xc = min(max(xi[ii], 0), n1 - 1);
                        const int yc = min(max(y + i, 0), n1 - 1);
                        const double *Cc =
                            P.C + (7 * p1_axis_class(yc, n1) + p1_axis_class(xc, n1)) * 58;
                        pa = node_update(v, Cc + (FWD ? 0 : 29));
                        pb = node_update(v, Cc + (FWD ? 29 : 0));
                    }
                    if (act[ii]) {
                        store_v(i, xi[ii], v);
                        if (owned(i, xi[ii])) x_update(i, xi[ii], pa, pb);
                    }
                }
            }
        } else if (bside) {
            // this lane's vertex: row y_bi of colour warp qq, the column in
            // 0..2 (left) or n1-3..n1-1 (right) with that colour, if any
            const int yb = y + bi;
            const int c0 = side == 0 ? 0 : n1 - 3;
            const int ob = ((colour - 2 * yb - c0) % 7 + 7) % 7;  // column offset from c0
            const int xb = c0 + ob;
            if (ob < 3 && in_rows(bi) && int_row(bi) &&
                (unsigned)(xb - cxl) < (unsigned)(cxr - cxl)) {
                double2 v[7];
                load_v(bi, xb, v);
                const unsigned cs = cls_s + (unsigned)(p1_axis_class(xb, n1) * 2) * (CROW * 8);
                const double pa = node_update_s(v, cs + (FWD ? 0 : CROW * 8));
                const double pb = node_update_s(v, cs + (FWD ? CROW * 8 : 0));
                store_v(bi, xb, v);
                if (owned(bi, xb)) x_update(bi, xb, pa, pb);
            }
        }
        }
        // advance K rows
        y += K;
        sl = wrap(sl + K);
        o = (o - 2 * K + 7 * K) % 7;
        if (kFast) {
            ra0 = ra2;
            ra1 = ra3;
            ra2 = nxt_r(ra3);
            ra3 = nxt_r(ra2);
            xa0 = nxt_x(xa1);
            xa1 = nxt_x(xa0);
        }
        if (CHAIN) {
            mcs_flag_set(flg + 4u * (bw ? F_BW : qq), S + 1);
        } else {
            mcs_wait<D - 1>();
            __syncthreads();
        }
    }
    mcs_wait<0>();
}

// host side: the distinct interior values from ci58 = [state row (29),
// adjoint row (29)] (node_update layout); false if a slot differs bitwise
// from its distinct value (the symmetry mcs::umap assumes does not hold)
inline bool mcs_fill_cu(double (&cu)[mcs::NU], const double *ci58) {
    bool set[mcs::NU] = {};
    for (int f = 0; f < 2; ++f)
        for (int i = 0; i < 29; ++i) {
            const int u = mcs::umap(f, i);
            if (!set[u]) cu[u] = ci58[29 * f + i], set[u] = true;
            if (std::memcmp(&cu[u], &ci58[29 * f + i], sizeof(double)) != 0) return false;
        }
    for (bool b : set)
        if (!b) return false;
    return true;
}

inline void mcs_set_smem() {
    OCMG_CUDA(cudaFuncSetAttribute(k_p1_mc_sweep<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mcs::SMEM));
    OCMG_CUDA(cudaFuncSetAttribute(k_p1_mc_sweep<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mcs::SMEM));
}
inline void mcs_launch(const McsParams &P, int grid, cudaStream_t s) {
    OCMG_REQUIRE(((uintptr_t)P.rin & 7) == 0 && ((uintptr_t)P.rout & 7) == 0 &&
                     ((uintptr_t)P.x & 7) == 0,
                 "vectors must be 8-byte aligned");
    if (P.forward)
        OCMG_LAUNCH(k_p1_mc_sweep<true>, grid, mcs::NT, mcs::SMEM, s, P);
    else
        OCMG_LAUNCH(k_p1_mc_sweep<false>, grid, mcs::NT, mcs::SMEM, s, P);
}

// host-side launch geometry: strips of W columns; base or base+1 row
// segments per strip so that the grid fills the SMs (two CTAs each) once
struct McsPlan {
    int nstrips = 0, base = 0, rem = 0, grid = 0;
};

// rows per segment at least: shorter segments only add pipeline fill (55 rows
// of halo and lag per CTA), but on the small levels of a cycle (L7-L9) more,
// shorter CTAs still shorten the sweep while SMs are idle (24 -> 8: L7 41 ->
// 34 us, L8 44 -> 36, L9 46 -> 37 per sweep; config 3 multicolour 0.297 ->
// 0.264 s)
#ifndef MCS_MIN_SEG_ROWS
#define MCS_MIN_SEG_ROWS 8
#endif
inline McsPlan mcs_plan(int n1, int sm_count, int rows = -1) {
    McsPlan p;
    if (rows < 0) rows = n1;
    p.nstrips = (n1 + mcs::W - 1) / mcs::W;  // balanced widths <= W (kernel)
    // segments much shorter than the pipeline fill (H + STORE_LAG rows) waste steps
    const int max_seg = std::max(1, rows / MCS_MIN_SEG_ROWS);
    const int total = std::max(p.nstrips, std::min(sm_count, p.nstrips * max_seg));
    p.base = total / p.nstrips;
    p.rem = total % p.nstrips;
    p.grid = p.nstrips * (p.base + (p.rem ? 1 : 0));
    return p;
}

}  // namespace ocmg
