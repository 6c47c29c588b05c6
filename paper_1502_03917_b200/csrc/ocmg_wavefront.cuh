// Exact-order (wavefront) NE-GS sweep of a structured P1 level in ONE
// cooperative launch: the reference's sweep order (kernels.lsgs_sweep,
// kernels.py:43-66), all state unknowns lexicographically, then all adjoint
// unknowns (backward: the reverse).
//
// Algebra (delta form).  With N = A^T L^-1 A and
// G = A^T L^-1 r_entry the sequential sweep computes, unknown by unknown,
//     p_i = (G_i - sum_{k earlier, k ~ i} N_ik p_k) / N_ii ,
// which is the reference's q = sum_j A_ij r_j / L_j on the current residual.
// Forward order is every state unknown, then every adjoint one, so a sweep is
// two triangular "chains" separated by residual updates:
//     G1 = W_F1 r_entry                       chain 1:  p1 = (G1 - N1 p1) / n
//     u  = r_entry - A[:, F1] p1              G2 = W_F2 u
//     chain 2:  p2 = (G2 - N2 p2) / n         r  = u - A[:, F2] p2,  x += p
// (F1 = state, F2 = adjoint; the backward sweep runs on the point-reflected
// grid with the fields swapped and the "upper" N coefficients).  A node
// (x, y) of a chain depends on its 9 earlier neighbours at graph distance
// <= 2, which sit on wavefront levels x + 2y - 1 ... x + 2y - 6.  Rounding
// differs from the reference (FMA, one residual fold per chain); tests hold
// the result to 1e-12 of the reference order.
//
// Execution.  One CTA per band of REAL = 29 grid rows; lane i of every warp
// is band row i (rows 29..31 are the next band's first rows, recomputed
// bit-identically so that u, G2 and r of the band's own rows need nothing
// from below; rows -1, -2 come from the band above).  Every stage walks the
// band in *skewed* time: at step tau, lane i handles column x = tau - 2 i
// (minus the stage's lag), so a wavefront level is one step for all lanes.
// Shared-memory windows are indexed by the skewed slot x + 2 i, so the 32
// lanes of a step touch one slot of 32 rows (an odd row stride keeps that
// conflict-free) and a window only has to span the stages' lags, not the
// 62-column skew.  Warps (all lane = row):
//   0  chain 1    8 steps per iteration, incremental: the two terms from
//                 level t-1 (own row's last p, the row above's last p by
//                 shuffle) are the only ones on the critical path; the
//                 others are folded into a 7-deep accumulator window as
//                 soon as they exist
//   1  chain 2    the same on G2, 36 steps behind
//   2  G1         16 steps ahead of chain 1        (stencil on r_entry)
//   3  u          11 steps behind, x_F1 += p1      (stencil on p1)
//   4  G2         22 steps behind                  (stencil on u)
//   5  r          47 steps behind, x_F2 += p2      (stencil on p2)
//   6  loader     cp.async of r_entry (rows 0..32) and x 59 steps ahead
//   7  writer     r and x of finished columns back to HBM (coalesced)
//   8  scout      waits for the band above and stages its rows -2, -1
// then one CTA barrier per iteration of CW = 8 steps and a release of the
// band's progress counter.  The band above publishes p1, u and p2 of its
// rows 27-28 into a per-band hand-off array (indexed by its slot; a row of
// band b sits 58 slots earlier in band b+1's frame), and r_entry of its row
// 28 (G1 of band b+1's row 0 needs it, and band b overwrites r in place).
// Band b starts iteration c+1 once band b-1 has completed c + DOWN.  Nothing
// flows upwards: band b reads r_entry of band b+1's first rows (its ghost
// rows) long before band b+1, DOWN iterations behind, overwrites them.
//
// Table layout appended after the P1 tables (see ocmg_p1.cuh):
//   WF[49][38]: per position class
//     [ 0.. 8] N^{yy}_{ik} for the 9 earlier ("lower") state neighbours k
//     [ 9..17] N^{ll}_{ik} for the 9 earlier adjoint neighbours
//     [18..26] N^{yy} for the 9 later ("upper") neighbours (backward sweep)
//     [27..35] N^{ll} for the 9 later neighbours
//     [36], [37] 1 / n_diag for the state / adjoint unknown
//   lower offsets m = 0..8 in increasing index order:
//     (-2,-2) (-1,-2) (0,-2) (-2,-1) (-1,-1) (0,-1) (1,-1) (-2,0) (-1,0);
//   upper offset m is the negation of lower offset m.
#pragma once

#include "ocmg_common.cuh"
#include "ocmg_p1.cuh"

#ifndef WF_REL_WARP
#define WF_REL_WARP 0
#endif

namespace ocmg {

constexpr int kWfStride = 38;
constexpr int kWfTableDoubles = 49 * kWfStride;

namespace wf {
constexpr int REAL = 29;            // rows owned by a band
constexpr int CW = 8;               // steps per iteration
constexpr int WL = 128, SL = WL + 1;  // long windows (r_entry / u / r, x)
constexpr int WS = 32, SS = WS + 1;   // short windows (G1, p1, G2, p2)
constexpr int D = 5;                // cp.async groups in flight
// a stage at iteration c handles steps [CW c - OFF, CW c - OFF + CW)
constexpr int OFF_G1 = -16, OFF_C1 = 0, OFF_U = 11, OFF_G2 = 22, OFF_C2 = 36,
              OFF_R = 47, OFF_WR = 55, OFF_LD = -(CW * D + 19);
constexpr int SKEW = 2 * REAL;      // slot shift from band b-1 to band b
constexpr int DOWN = 9;             // iteration c+1 needs band b-1 through c+DOWN
// rows each stage produces (lanes 0..n-1)
constexpr int ROWS_C1 = 32, ROWS_U = 31, ROWS_G2 = 30, ROWS_C2 = 30;
constexpr int RE_ROWS = 34;         // r_entry / u / r rows -1..32
constexpr int P1_ROWS = 34;         // p1 rows -2..31
constexpr int P2_ROWS = 32;         // p2 rows -2..29
constexpr int HO = 8;               // hand-off doubles per slot
constexpr int SO = 160;             // slot offset of the hand-off array
constexpr int NWARPS = 9, NTHREADS = 32 * NWARPS;
constexpr int FLAG_STRIDE = 64;     // ints between band counters (256 B)
// shared memory (doubles)
constexpr int SM_AW = kP1Classes * 28 * 2;  // A then W
constexpr int SM_N = kWfTableDoubles;
constexpr int SM_RE = 2 * RE_ROWS * SL;
constexpr int SM_X = 2 * REAL * SL;
constexpr int SM_G1 = ROWS_C1 * SS, SM_P1 = P1_ROWS * SS;
constexpr int SM_G2 = ROWS_G2 * SS, SM_P2 = P2_ROWS * SS;
constexpr int SM_TOTAL = SM_AW + SM_N + SM_RE + SM_X + SM_G1 + SM_P1 + SM_G2 + SM_P2;
constexpr size_t SM_BYTES = SM_TOTAL * sizeof(double);
static_assert(SM_BYTES <= 227 * 1024, "one CTA per SM");
// window spans (see the stage comments): the long windows hold slots from
// the loader's (CW c - OFF_LD + CW) down to the writer's (CW c - OFF_WR)
static_assert(OFF_WR - OFF_LD + CW <= WL, "long window too short");
static_assert(OFF_C1 - OFF_G1 + 6 + CW <= WS, "G1 window too short");
}  // namespace wf

struct WfParams {
    int n1, nb, c0, c1;         // iterations c0 .. c1-1
    const double *T;            // P1 tables (device)
    const double *WF;           // delta tables (device)
    double *x, *r;
    double *ho;                 // [nb][nslot][HO] hand-off values
    int nslot;
    int *iter;                  // [nb * FLAG_STRIDE] completed iterations
    unsigned long long *prof;   // OCMG_WF_PROFILE: [nb][niter][NWARPS][3] ns
};

namespace wfd {
__device__ __forceinline__ void cp8(unsigned dst, const double *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
}  // namespace wfd

// per-CTA constants, shared by the stage functions
struct WfBand {
    double *hsink;  // this band's dummy hand-off slots: non-publishing lanes
                    // store there unconditionally (a guarded store cost the
                    // chain 30-40 cycles per step)
    int n1, b, iy0, nreal;
    int64_t N;
    const double *sA, *sW, *sN;  // shared tables
    double *re, *xw, *g1, *p1, *g2, *p2;  // shared windows
};

template <bool BWD>
__device__ __forceinline__ int wf_cls(const WfBand &B, int x, int i) {
    // position class of processing-frame node (x, band row i), clamped into
    // the domain (callers never use the value outside it)
    const int xc = min(max(x, 0), B.n1 - 1);
    const int yc = min(max(B.iy0 + i, 0), B.n1 - 1);
    const int cx = p1_axis_class(xc, B.n1), cy = p1_axis_class(yc, B.n1);
    return BWD ? 7 * (6 - cy) + (6 - cx) : 7 * cy + cx;
}
__device__ __forceinline__ bool wf_col_int(int x, int n1) { return x >= 3 && x <= n1 - 4; }
// the two halves of wf_cls: 7 * (row class) of band row i, and the column
// class of processing-frame column x (the boundary paths add them per node)
template <bool BWD>
__device__ __forceinline__ int wf_rowbase(const WfBand &B, int i) {
    const int cy = p1_axis_class(min(max(B.iy0 + i, 0), B.n1 - 1), B.n1);
    return 7 * (BWD ? 6 - cy : cy);
}
template <bool BWD>
__device__ __forceinline__ int wf_colcls(int x, int n1) {
    const int cx = p1_axis_class(min(max(x, 0), n1 - 1), n1);
    return BWD ? 6 - cx : cx;
}

// c ? a : b without a branch.  On values loaded from shared memory the
// compiler turns a ternary into a divergent branch with the load sunk into
// it; on the chain's critical path that cost ~190 of ~215 cycles per step
// (scripts/micro_chain.cu: 213 -> 24 cycles per step).
__device__ __forceinline__ double wf_sel(bool c, double a, double b) {
    const long long m = -(long long)c;
    return __longlong_as_double((__double_as_longlong(a) & m) | (__double_as_longlong(b) & ~m));
}

// guarded stores (kept as plain C++: inline asm with a memory clobber stopped
// the compiler from moving the next loads above them, 15-30 cycles per step)
__device__ __forceinline__ void wf_sts(double *p, double v, bool pred) {
    // a plain guarded store: the compiler predicates it, and (unlike inline
    // asm with a memory clobber) may still move the next loads above it
    if (pred) *p = v;
}
__device__ __forceinline__ void wf_stg(double *p, double v, bool pred) {
    if (pred) *p = v;
}

// window accessors (processing-frame band row i, slot s)
__device__ __forceinline__ double &wf_re(const WfBand &B, int f, int i, int s) {
    return B.re[(f * wf::RE_ROWS + i + 1) * wf::SL + (s & (wf::WL - 1))];
}
__device__ __forceinline__ double &wf_xw(const WfBand &B, int f, int i, int s) {
    return B.xw[(f * wf::REAL + i) * wf::SL + (s & (wf::WL - 1))];
}

// ---------------------------------------------------------------------------
// chain: CW steps of one triangular chain.  acc[k] is the partial q of
// column x + k; at step x the 9 lower neighbours of columns x .. x+6 arrive
// as (own row) p(x), (row above, shuffle) v1 = p(x+2, i-1), (two above)
// v2 = p(x+4, i-2):
//   x+6: init G, m0 v2   x+5: m1 v2   x+4: m3 v1, m2 v2   x+3: m4 v1
//   x+2: m7 p, m5 v1     x+1: next step, critical: m8 p, m6 v1
// ---------------------------------------------------------------------------
struct WfChain {
    double acc[7];
    double pprev, v1prev;
};

template <bool BWD, bool FAST>
__device__ __forceinline__ void wf_chain(const WfBand &B, WfChain &S, const double (&K)[10],
                                         int tau0, int nb, int invo, int nrows,
                                         const double *gw, double *pw, double *ho,
                                         int hoff) {
    using namespace wf;
    const int i = threadIdx.x & 31, n1 = B.n1;
    const bool rowok = i < nrows && B.iy0 + i < n1;
    const double *Ntab = B.sN;
    // boundary path: column classes of the targets x0 .. x0 + CW + 5 once per
    // call; a coefficient comes from the table only where the target's
    // column class is not the interior one (K holds this row's interior-
    // column coefficients; targets outside the domain never matter: their
    // p is forced to 0)
    int cxw[CW + 6];
    if (!FAST) {
        const int x0 = tau0 - 2 * i;
#pragma unroll
        for (int k = 0; k < CW + 6; ++k) cxw[k] = wf_colcls<BWD>(x0 + k, n1);
    }
    const int rb = FAST ? 0 : wf_rowbase<BWD>(B, i);
    auto Nc = [&](int s, int k, int m) {  // -N_m of target (x + k, i) at step s
        if (FAST) return K[m];
        const int cx = cxw[s + k];
        return wf_sel(cx == 3, K[m], -Ntab[(rb + cx) * kWfStride + nb + m]);
    };
    // everything this iteration reads, before any store: G of columns x+6
    // and the band above's rows -1, -2 (staged by the scout; lanes 0, 1)
    double g[CW], e1[CW], e2[CW];
#pragma unroll
    for (int s = 0; s < CW; ++s) {
        const int sl = (tau0 + s) & (WS - 1);
        g[s] = gw[i * SS + ((tau0 + s + 6) & (WS - 1))];
        e1[s] = pw[1 * SS + sl];
        e2[s] = pw[0 * SS + sl];
    }
    double pout[CW];
#pragma unroll
    for (int s = 0; s < CW; ++s) {
        const int tau = tau0 + s;
        const int x = tau - 2 * i;
        // 1/n_diag, or 0 outside the domain (the accumulators stay finite
        // there: every window starts zeroed)
        const double inv = wf_sel(rowok && (unsigned)x < (unsigned)n1,
                                  FAST ? K[9]
                                       : wf_sel(cxw[s] == 3, K[9], Ntab[(rb + cxw[s]) * kWfStride + invo]),
                                  0.0);
        double a = fma(Nc(s, 0, 8), S.pprev, S.acc[0]);
        a = fma(Nc(s, 0, 6), S.v1prev, a);
        const double p = a * inv;
        pout[s] = p;
        const double u1 = __shfl_up_sync(0xffffffffu, p, 1);
        const double u2 = __shfl_up_sync(0xffffffffu, p, 2);
        const double v1 = wf_sel(i == 0, e1[s], u1);
        const double v2 = wf_sel(i == 0, e2[s], wf_sel(i == 1, e1[s], u2));
        double a2 = fma(Nc(s, 2, 7), p, S.acc[2]);
        a2 = fma(Nc(s, 2, 5), v1, a2);
        const double a3 = fma(Nc(s, 3, 4), v1, S.acc[3]);
        double a4 = fma(Nc(s, 4, 3), v1, S.acc[4]);
        a4 = fma(Nc(s, 4, 2), v2, a4);
        const double a5 = fma(Nc(s, 5, 1), v2, S.acc[5]);
        const double a6 = fma(Nc(s, 6, 0), v2, g[s]);
        S.acc[0] = S.acc[1];
        S.acc[1] = a2;
        S.acc[2] = a3;
        S.acc[3] = a4;
        S.acc[4] = a5;
        S.acc[5] = a6;
        S.pprev = p;
        S.v1prev = v1;
    }
    const int ip = min(i, nrows - 1);
#pragma unroll
    for (int s = 0; s < CW; ++s) wf_sts(pw + (ip + 2) * SS + ((tau0 + s) & (WS - 1)), pout[s], i < nrows);
    if (ho) {
        const bool pub = i == REAL - 2 || i == REAL - 1;
        double *h = pub ? ho + (int64_t)(tau0 + SO) * HO + hoff + (i - (REAL - 2)) : B.hsink;
#pragma unroll
        for (int s = 0; s < CW; ++s) h[s * HO] = pout[s];
    }
}

// ---------------------------------------------------------------------------
// G stage: gw(i, tau) = sum_f sum_e W[F][f][d(e)] src_f(neighbour e) for rows
// i < nrows, src = the long window (r_entry for G1, u for G2).  Processing
// frame neighbour e = 0:(-1,-1) 1:(0,-1) 2:(-1,0) 3:(0,0) 4:(1,0) 5:(0,1)
// 6:(1,1) at slots tau-3, tau-2 (row i-1), tau-1, tau, tau+1 (row i),
// tau+2, tau+3 (row i+1); the reflected frame reads table entry 6 - e.
// Two halves of H = 4 steps: all loads, then H independent sums, then the
// stores (no load waits behind a store to the same window).
// ---------------------------------------------------------------------------
template <bool BWD, bool FAST>
__device__ __forceinline__ void wf_gstage(const WfBand &B, int F, int tau0, int nrows,
                                          double *gw, double *ho) {
    using namespace wf;
    constexpr int H = CW;  // one pass of 8 outputs (67 vs 73 cycles/step for two of 4)
    const int i = threadIdx.x & 31;
    const int ii = min(i, nrows - 1);  // address row (idle lanes read a valid row)
    // this lane's row class with an interior column class (FAST: every
    // column of the call is interior, the row may be a boundary row)
    const int rb = wf_rowbase<BWD>(B, i);
    const double *Wi = B.sW + (rb + 3) * 28 + F * 14;
    double w[2][7];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int e = 0; e < 7; ++e) w[f][e] = Wi[f * 7 + (BWD ? 6 - e : e)];
#pragma unroll
    for (int h = 0; h < CW / H; ++h) {
        const int t0 = tau0 + h * H;
        // row i-1: slots t0-3 .. t0+H-3; row i: t0-1 .. t0+H; row i+1: t0+2 .. t0+H+2
        double up[2][H + 1], md[2][H + 2], dn[2][H + 1];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
#pragma unroll
            for (int k = 0; k <= H; ++k) {
                up[f][k] = wf_re(B, f, ii - 1, t0 - 3 + k);
                dn[f][k] = wf_re(B, f, ii + 1, t0 + 2 + k);
            }
#pragma unroll
            for (int k = 0; k < H + 2; ++k) md[f][k] = wf_re(B, f, ii, t0 - 1 + k);
        }
        double out[H];
#pragma unroll
        for (int s = 0; s < H; ++s) {
            const int cx = FAST ? 3 : wf_colcls<BWD>(t0 + s - 2 * i, B.n1);
            const double *wc = B.sW + (rb + cx) * 28 + F * 14;
            auto W = [&](int f, int e) {
                return FAST ? w[f][e] : wf_sel(cx == 3, w[f][e], wc[f * 7 + (BWD ? 6 - e : e)]);
            };
            double g = 0.0;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                g = fma(W(f, 0), up[f][s], g);
                g = fma(W(f, 1), up[f][s + 1], g);
                g = fma(W(f, 2), md[f][s], g);
                g = fma(W(f, 3), md[f][s + 1], g);
                g = fma(W(f, 4), md[f][s + 2], g);
                g = fma(W(f, 5), dn[f][s], g);
                g = fma(W(f, 6), dn[f][s + 1], g);
            }
            out[s] = g;
        }
#pragma unroll
        for (int s = 0; s < H; ++s) wf_sts(gw + ii * SS + ((t0 + s) & (WS - 1)), out[s], i < nrows);
        if (ho) {  // G1 only: r_entry of row 28 for band b+1
            double *h = i == REAL - 1 ? ho + (int64_t)(t0 + SO) * HO + 6 : B.hsink;
#pragma unroll
            for (int s = 0; s < H; ++s) {
                h[s * HO] = md[0][s + 1];
                h[s * HO + 1] = md[1][s + 1];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// apply stage: out_f = base_f - sum_e A[f][FP][d(e)] p(neighbour e), in place
// in the long window (r_entry -> u for chain 1's field FP, u -> r for chain
// 2's), rows i < nrows inside the domain; x_FP += p on the real rows.
// pw: the chain's p window (rows -2..); halves of 4 steps like the G stage.
// ---------------------------------------------------------------------------
template <bool BWD, bool FAST>
__device__ __forceinline__ void wf_astage(const WfBand &B, int FP, int tau0, int nrows,
                                          const double *pw, int prow_max, double *ho,
                                          int hoff) {
    using namespace wf;
    constexpr int H = CW / 2;
    const int i = threadIdx.x & 31, n1 = B.n1;
    const int ii = min(i, prow_max - 2);  // idle lanes read rows that exist
    const bool rowok = i < nrows && B.iy0 + i < n1;
    const bool real = rowok && i < B.nreal;
    const int ib = min(i, REAL - 1);  // x row (read-only on idle lanes)
    auto Pv = [&](int row, int s) { return pw[(row + 2) * SS + (s & (WS - 1))]; };
    const int rb = wf_rowbase<BWD>(B, i);
    const double *Ai = B.sA + (rb + 3) * 28;  // see wf_gstage
    double a[2][7];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int e = 0; e < 7; ++e) a[f][e] = -Ai[f * 14 + FP * 7 + (BWD ? 6 - e : e)];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t0 = tau0 + h * H;
        double up[H + 1], md[H + 2], dn[H + 1], base[2][H], xo[H];
#pragma unroll
        for (int k = 0; k <= H; ++k) {
            up[k] = Pv(ii - 1, t0 - 3 + k);
            dn[k] = Pv(ii + 1, t0 + 2 + k);
        }
#pragma unroll
        for (int k = 0; k < H + 2; ++k) md[k] = Pv(ii, t0 - 1 + k);
#pragma unroll
        for (int s = 0; s < H; ++s) {
            base[0][s] = wf_re(B, 0, i, t0 + s);
            base[1][s] = wf_re(B, 1, i, t0 + s);
            xo[s] = wf_xw(B, FP, ib, t0 + s);
        }
        double out[2][H];
#pragma unroll
        for (int s = 0; s < H; ++s) {
            const int cx = FAST ? 3 : wf_colcls<BWD>(t0 + s - 2 * i, n1);
            const double *ac = B.sA + (rb + cx) * 28;
            auto A = [&](int f, int e) {
                return FAST ? a[f][e]
                            : wf_sel(cx == 3, a[f][e], -ac[f * 14 + FP * 7 + (BWD ? 6 - e : e)]);
            };
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                double w = base[f][s];
                w = fma(A(f, 0), up[s], w);
                w = fma(A(f, 1), up[s + 1], w);
                w = fma(A(f, 2), md[s], w);
                w = fma(A(f, 3), md[s + 1], w);
                w = fma(A(f, 4), md[s + 2], w);
                w = fma(A(f, 5), dn[s], w);
                w = fma(A(f, 6), dn[s + 1], w);
                out[f][s] = w;
            }
        }
#pragma unroll
        for (int s = 0; s < H; ++s) {
            const int tau = t0 + s;
            const bool ok = rowok && (unsigned)(tau - 2 * i) < (unsigned)n1;
            wf_sts(&wf_re(B, 0, i, tau), out[0][s], ok);
            wf_sts(&wf_re(B, 1, i, tau), out[1][s], ok);
            if (ho) {
                double *h = ok && i == REAL - 1 ? ho + (int64_t)(tau + SO) * HO + hoff : B.hsink;
                h[0] = out[0][s];
                h[1] = out[1][s];
            }
            wf_sts(&wf_xw(B, FP, ib, tau), xo[s] + md[s + 1], ok && real);
        }
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <bool BWD>
__global__ void __launch_bounds__(wf::NTHREADS, 1) k_wavefront(const __grid_constant__ WfParams P) {
    using namespace wf;
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WfBand B;
    B.n1 = P.n1;
    B.b = blockIdx.x;
    B.iy0 = blockIdx.x * REAL;
    B.nreal = min(REAL, P.n1 - B.iy0);
    B.N = (int64_t)P.n1 * P.n1;
    B.sA = sm;
    B.sW = sm + kP1Classes * 28;
    B.sN = sm + SM_AW;
    B.re = sm + SM_AW + SM_N;
    B.xw = B.re + SM_RE;
    B.g1 = B.xw + SM_X;
    B.p1 = B.g1 + SM_G1;
    B.g2 = B.p1 + SM_P1;
    B.p2 = B.g2 + SM_G2;
    // chain 1 works on field F1, chain 2 on F2 (0 state, 1 adjoint)
    constexpr int F1 = BWD ? 1 : 0, F2 = 1 - F1;
    constexpr int NB1 = BWD ? 27 : 0, NB2 = BWD ? 18 : 9;
    constexpr int INV1 = 36 + F1, INV2 = 36 + F2;

    for (int t = threadIdx.x; t < SM_AW; t += NTHREADS) sm[t] = P.T[t];
    for (int t = threadIdx.x; t < SM_N; t += NTHREADS) sm[SM_AW + t] = P.WF[t];
    for (int t = threadIdx.x; t < SM_TOTAL - SM_AW - SM_N; t += NTHREADS) B.re[t] = 0.0;
    __syncthreads();

    const int n1 = P.n1, b = B.b;
    double *const ho_out = b + 1 < P.nb ? P.ho + (int64_t)b * P.nslot * HO : nullptr;
    B.hsink = P.ho + ((int64_t)b * P.nslot + P.nslot - 2 * CW) * HO;
    const double *const ho_in = b > 0 ? P.ho + (int64_t)(b - 1) * P.nslot * HO : nullptr;
    // chain state and interior coefficients (negated N, then 1/n_diag)
    WfChain S;
#pragma unroll
    for (int k = 0; k < 7; ++k) S.acc[k] = 0.0;
    S.pprev = S.v1prev = 0.0;
    double K[10];
    {
        const int nb = warp == 1 ? NB2 : NB1, io = warp == 1 ? INV2 : INV1;
        const int lc = wf_cls<BWD>(B, n1 / 2, lane) * kWfStride;  // row class, interior column
#pragma unroll
        for (int m = 0; m < 9; ++m) K[m] = -B.sN[lc + nb + m];
        K[9] = B.sN[lc + io];
    }
    // FAST: every column a stage touches this iteration (tau0 - 2*31 + lo ..
    // tau0 + CW - 1 + hi) has the interior column class; each lane then
    // holds its own row's coefficients (boundary rows included)
    auto fast = [&](int tau0, int lo, int hi) {
        return wf_col_int(tau0 - 62 + lo, n1) && wf_col_int(tau0 + CW - 1 + hi, n1);
    };
    const unsigned sre = (unsigned)__cvta_generic_to_shared(B.re);
    const unsigned sxw = (unsigned)__cvta_generic_to_shared(B.xw);

#ifdef OCMG_WF_PROFILE
    auto gtimer = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
    unsigned long long t_begin = 0;
    long long c_begin = 0, t_mid = 0;
    auto prof_begin = [&]() {
        t_begin = gtimer();
        c_begin = clock64();
        t_mid = 0;
    };
#else
    auto prof_begin = []() {};
#endif
    // end of iteration c: every warp, from its own role loop (the roles are
    // separate loops so that the two warps of a role share one copy of the
    // code: the instruction cache, not the arithmetic, bounded the first
    // version with one loop and a role switch)
    auto iteration_end = [&](int c) {
#ifdef OCMG_WF_PROFILE
        if (lane == 0 && P.prof) {
            unsigned long long *pp =
                P.prof + (((int64_t)blockIdx.x * (P.c1 - P.c0) + (c - P.c0)) * NWARPS + warp) * 3;
            const long long ce = clock64();
            pp[0] = t_begin;
            pp[1] = warp == 8 ? (unsigned long long)t_mid
                              : (unsigned long long)((t_mid ? t_mid : ce) - c_begin);
            pp[2] = (unsigned long long)(ce - c_begin);
        }
#endif
        asm volatile("bar.sync 0, %0;" ::"n"(NTHREADS) : "memory");
        // the release (a gpu-scope fence, then the flag) is issued by a lane
        // of warp WF_REL_WARP: after the barrier it covers every warp's
        // hand-off stores, and whichever warp issues it starts its next
        // iteration that much later (measured at L9 / L10 / L12: warp 0
        // 0.487 / 0.938 / 4.28 ms, the loader 0.482 / 0.940 / 4.70, the
        // writer 0.485 / 0.933 / 4.46, the scout 0.500 / 0.962 / 4.33: the
        // iteration period is not set by this fence)
        if (threadIdx.x == 32 * WF_REL_WARP) {
            wfd::st_release(P.iter + b * FLAG_STRIDE, c - P.c0 + 1);
#ifdef OCMG_WF_PROFILE
            if (P.prof)  // warp 0's mid slot: when this release was issued (ns)
                P.prof[(((int64_t)blockIdx.x * (P.c1 - P.c0) + (c - P.c0)) * NWARPS) * 3 + 1] =
                    gtimer();
#endif
        }
    };

    if (warp < 2) {
        // chains: warp 0 chain 1 on G1, warp 1 chain 2 on G2
        const int off = warp ? OFF_C2 : OFF_C1, nb = warp ? NB2 : NB1, io = warp ? INV2 : INV1;
        const int nrows = warp ? ROWS_C2 : ROWS_C1, hoff = warp ? 4 : 0;
        double *const gw = warp ? B.g2 : B.g1;
        double *const pw = warp ? B.p2 : B.p1;
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            const int t0 = CW * c - off;
            if (fast(t0, -2, 6))
                wf_chain<BWD, true>(B, S, K, t0, nb, io, nrows, gw, pw, ho_out, hoff);
            else
                wf_chain<BWD, false>(B, S, K, t0, nb, io, nrows, gw, pw, ho_out, hoff);
            iteration_end(c);
        }
    } else if (warp == 2 || warp == 4) {
        // G stages: warp 2 G1 (on r_entry, publishes r_entry of row 28),
        // warp 4 G2 (on u)
        const bool one = warp == 2;
        const int off = one ? OFF_G1 : OFF_G2, F = one ? F1 : F2;
        const int nrows = one ? ROWS_C1 : ROWS_G2;
        double *const gw = one ? B.g1 : B.g2;
        double *const ho = one ? ho_out : nullptr;
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            const int t0 = CW * c - off;
            if (fast(t0, -1, 1))
                wf_gstage<BWD, true>(B, F, t0, nrows, gw, ho);
            else
                wf_gstage<BWD, false>(B, F, t0, nrows, gw, ho);
            iteration_end(c);
        }
    } else if (warp == 3 || warp == 5) {
        // apply stages: warp 3 u = r_entry - A[:, F1] p1 (publishes u of row
        // 28), warp 5 r = u - A[:, F2] p2
        const bool one = warp == 3;
        const int off = one ? OFF_U : OFF_R, FP = one ? F1 : F2;
        const int nrows = one ? ROWS_U : REAL, prow = one ? 32 : 30;
        const double *const pw = one ? B.p1 : B.p2;
        double *const ho = one ? ho_out : nullptr;
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            const int t0 = CW * c - off;
            if (fast(t0, -1, 1))
                wf_astage<BWD, true>(B, FP, t0, nrows, pw, prow, ho, 2);
            else
                wf_astage<BWD, false>(B, FP, t0, nrows, pw, prow, ho, 2);
            iteration_end(c);
        }
    } else if (warp == 6) {
        // loader: slots [t0, t0 + CW) of r_entry rows 0..32 and x rows 0..28,
        // both fields, zero outside the domain (row -1 comes from the band
        // above).  Lane = (segment group, slot): 4 row segments of CW slots
        // per warp instruction
        const int sub = lane >> 3;
        const int N = n1 * n1;
        constexpr int LR = RE_ROWS - 1;
        constexpr int TR = (2 * LR + 3) / 4, TX = (2 * REAL + 3) / 4;
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            const int slot = CW * c - OFF_LD + (lane & 7), sw = slot & (WL - 1);
#pragma unroll
            for (int t = 0; t < TR; ++t) {
                const int q = sub + 4 * t;
                const int f = q >= LR, row = q - f * LR;
                const int x = slot - 2 * row, y = B.iy0 + row;
                const bool ok = (unsigned)x < (unsigned)n1 && (unsigned)y < (unsigned)n1;
                const int g = f * N + (BWD ? N - 1 - (y * n1 + x) : y * n1 + x);
                if (t < TR - 1 || q < 2 * LR)
                    wfd::cp8(sre + (unsigned)(((f * RE_ROWS + row + 1) * SL + sw) * 8),
                             P.r + (ok ? g : 0), ok);
            }
#pragma unroll
            for (int t = 0; t < TX; ++t) {
                const int q = sub + 4 * t;
                const int f = q >= REAL, row = q - f * REAL;
                const int x = slot - 2 * row, y = B.iy0 + row;
                const bool ok = (unsigned)x < (unsigned)n1 && row < B.nreal;
                const int g = f * N + (BWD ? N - 1 - (y * n1 + x) : y * n1 + x);
                if (t < TX - 1 || q < 2 * REAL)
                    wfd::cp8(sxw + (unsigned)(((f * REAL + row) * SL + sw) * 8), P.x + (ok ? g : 0), ok);
            }
            wfd::commit();
#ifdef OCMG_WF_PROFILE
            t_mid = clock64();
#endif
            wfd::wait_group<D - 1>();
            iteration_end(c);
        }
        wfd::wait_group<0>();
    } else if (warp == 7) {
        // writer: r and x of the real rows at slots [t0, t0 + CW); lane =
        // (segment group, slot).  All loads first, then predicated stores:
        // no branch regions, the loads overlap
        const int sub = lane >> 3;
        const int N = n1 * n1;
        constexpr int NT = (2 * REAL + 3) / 4;  // 15 segments per lane and array
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            const int slot = CW * c - OFF_WR + (lane & 7);
#pragma unroll
            for (int arr = 0; arr < 2; ++arr) {
                double v[NT];
                int g[NT];
                bool ok[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int q = min(sub + 4 * t, 2 * REAL - 1);
                    const int f = q >= REAL, row = q - f * REAL;
                    const int x = slot - 2 * row, y = B.iy0 + row;
                    ok[t] = sub + 4 * t < 2 * REAL && (unsigned)x < (unsigned)n1 && row < B.nreal;
                    g[t] = f * N + (BWD ? N - 1 - (y * n1 + x) : y * n1 + x);
                    v[t] = arr ? wf_xw(B, f, row, slot) : wf_re(B, f, row, slot);
                }
#pragma unroll
                for (int t = 0; t < NT; ++t) wf_stg((arr ? P.x : P.r) + (ok[t] ? g[t] : 0), v[t], ok[t]);
            }
            iteration_end(c);
        }
    } else {
        // scout: progress of the band above, then its rows -2, -1 for the
        // next iteration
        for (int c = P.c0; c < P.c1; ++c) {
            prof_begin();
            if (b > 0) {
                if (lane == 0) {
                    // a schedule bug would spin forever: trap after ~10 s instead
                    unsigned spins = 0;
                    const int need = min(c + DOWN, P.c1 - 1) - P.c0 + 1;
                    // a busy poll (one L2 round trip per try)
                    while (wfd::ld_relaxed(P.iter + (b - 1) * FLAG_STRIDE) < need)
                        if (++spins > (1u << 25)) __trap();
                    wfd::fence_acq_rel();
#ifdef OCMG_WF_PROFILE
                    t_mid = (long long)gtimer();  // scout: poll success (ns)
#endif
                }
                __syncwarp();
                // 64 values: lane -> (kind, slot); kind 0/1 p1 rows -2/-1 for
                // chain 1 at c+1, 2/3 u row -1 fields 0/1 (G2 at c+1), 4/5 p2
                // rows -2/-1 for chain 2 at c+1, 6/7 r_entry row -1 fields 0/1
                // (G1 at c+1 reads slots from CW (c+1) - OFF_G1 - 3 on)
#pragma unroll
                for (int e0 = 0; e0 < HO * CW; e0 += 32) {
                    const int e = e0 + lane, kind = e / CW, s = e % CW;
                    const int base = kind < 2 ? CW * (c + 1) - OFF_C1
                                   : kind < 4 ? CW * c
                                   : kind < 6 ? CW * (c + 1) - OFF_C2
                                              : CW * (c + 1) - OFF_G1 - 2;
                    const int slot = base + s;
                    const double v = __ldcg(ho_in + (int64_t)(slot + SKEW + SO) * HO + kind);
                    double *dst = kind < 2   ? B.p1 + kind * SS + (slot & (WS - 1))
                                  : kind < 4 ? &wf_re(B, kind - 2, -1, slot)
                                  : kind < 6 ? B.p2 + (kind - 4) * SS + (slot & (WS - 1))
                                             : &wf_re(B, kind - 6, -1, slot);
                    *dst = v;
                }
            }
            iteration_end(c);
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct P1Wavefront {
    int k = 0, n1 = 0, nb = 0, c0 = 0, c1 = 0, nslot = 0;
    const double *T = nullptr;
    const double *tab = nullptr;  // device WF tables
    DevBuf<double> ho;
    DevBuf<int> iter;
    DevBuf<unsigned long long> prof;
    bool ok = false;

    void init(int k_, int n1_, const double *T_, const double *wf_tab) {
        using namespace wf;
        k = k_;
        n1 = n1_;
        T = T_;
        tab = wf_tab;
        nb = (n1 + REAL - 1) / REAL;
        // first iteration: chain 1 starts at iteration -1 (steps -8..-1, every
        // lane left of the domain, its accumulators 6 columns ahead); G1 has
        // to cover its slots from -2, the loader the slots G1 reads (-3).
        // Last: the writer passes the last real slot n1 - 1 + 2 (REAL - 1).
        auto fdiv = [](int a, int q) { return a >= 0 ? a / q : -((-a + q - 1) / q); };
        const int cg = fdiv(-CW + 6 + OFF_G1, CW);        // first G1 iteration
        const int re_first = CW * cg - OFF_G1 - 3;         // first slot it reads
        c0 = fdiv(re_first + OFF_LD, CW);
        c1 = (n1 + 2 * (REAL - 1) + OFF_WR + CW) / CW + 1;
        // hand-off slots: written from CW c0 - OFF_C2 on, read up to
        // CW c1 - OFF_G1 - 2 + CW + SKEW
        nslot = CW * (c1 + 1) - OFF_G1 + SKEW + SO + CW + 2 * CW;  // + the dummy slots
        OCMG_REQUIRE(CW * c0 - OFF_C2 + SO >= 0, "hand-off offset too small");
        int dev = 0, sms = 0, coop = 0;
        OCMG_CUDA(cudaGetDevice(&dev));
        OCMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        OCMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        OCMG_CUDA(cudaFuncSetAttribute(k_wavefront<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_BYTES));
        OCMG_CUDA(cudaFuncSetAttribute(k_wavefront<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_BYTES));
        int per_sm = 0;
        OCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wavefront<false>,
                                                                NTHREADS, SM_BYTES));
        if (!coop || per_sm < 1 || nb > sms * per_sm) return;  // level too big
        // slots nobody writes stay zero (the consumer's last iterations read
        // past the producer's last step, outside the domain)
        ho.alloc((size_t)nb * nslot * HO);
        OCMG_CUDA(cudaMemset(ho.p, 0, ho.n * sizeof(double)));
        iter.alloc((size_t)nb * FLAG_STRIDE);
#ifdef OCMG_WF_PROFILE
        prof.alloc((size_t)nb * (c1 - c0) * NWARPS * 3);
#endif
        ok = true;
    }
    bool ready() const { return ok; }
    int niter() const { return c1 - c0; }

    void sweep(bool forward, double *x, double *r, cudaStream_t s) const {
        WfParams P;
        P.n1 = n1;
        P.nb = nb;
        P.c0 = c0;
        P.c1 = c1;
        P.T = T;
        P.WF = tab;
        P.x = x;
        P.r = r;
        P.ho = ho.p;
        P.nslot = nslot;
        P.iter = iter.p;
        P.prof = prof.p;
        OCMG_CUDA(cudaMemsetAsync(iter.p, 0, iter.n * sizeof(int), s));
        void *args[] = {&P};
        launch_counter().fetch_add(1, std::memory_order_relaxed);
        OCMG_CUDA(cudaLaunchCooperativeKernel(
            forward ? (const void *)k_wavefront<false> : (const void *)k_wavefront<true>,
            dim3(nb), dim3(wf::NTHREADS), args, wf::SM_BYTES, s));
    }
};

}  // namespace ocmg
