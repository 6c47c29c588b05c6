// Fused wavefront NE-GS for structured P1 levels, in the reference's sweep
// order (kernels.lsgs_sweep, kernels.py:43-66), one cooperative launch per
// sweep.
//
// Algebra (delta form).  With N = A^T L^-1 A and
// G = A^T L^-1 r_entry, the sequential sweep computes, unknown by unknown,
//     p_i = (G_i - sum_{k earlier, k ~ i} N_ik p_k) / N_ii ,
// which is exactly the reference's q = sum_j A_ij r_j / L_j on the current
// residual.  Forward order is all state unknowns (lexicographic) then all
// adjoint unknowns, so a sweep is two triangular "chains":
//     chain 1 (state):   p_y = (G_y - N^yy_low p_y) / N_ii,  G_y = W_y r0
//     u = r0 - A[:, y] p_y                         (residual after chain 1)
//     chain 2 (adjoint): p_l = (G_l - N^ll_low p_l) / N_ii,  G_l = W_l u
//     r = u - A[:, l] p_l ,   x += p
// Every node of chain k depends on its 9 earlier neighbours at graph
// distance <= 2; node (ix, iy) sits at wavefront level ix + 2 iy.  The
// backward sweep is the same computation on the point-reflected grid with
// the fields swapped (adjoint chain first) and the "upper" N coefficients.
// Arithmetic differs from the reference only by rounding (FMA, residual
// folded once per sweep); tests hold it to 1e-12 per cycle.
//
// Execution.  One CTA per band of REAL = 29 grid rows.  Warp lanes map to
// 32 consecutive rows: the band's 29 rows plus 3 "ghost" rows of the band
// above, recomputed bit-identically, so that everything a band needs for its
// own rows (u needs chain-1 values one row up, G2 needs u one row up, r needs
// chain-2 values one row up) is produced inside the band: data flows only
// from band b-1 to band b.  Columns go in chunks of 32; iteration c runs, in
// parallel warps, every pipeline stage on a different chunk:
//   warp 0      chain 1 on chunk c        (lane l at column 32c - 2l + s,
//   warp 1      chain 2 on chunk c - A     s = 0..31: the skewed wavefront)
//   warp 2      scout: waits for band b-1's progress needed by iteration
//               c+1 and stages its top rows into smem
//   warps 3-6   G1 for chunk c + 1        (stencil on r_entry)
//   warps 7-10  u for chunk c - U, x += p1 (stencil on p1)
//   warps 11-14 G2 for chunk c - G        (stencil on u)
//   warps 15-18 r for chunk c - R, x += p2 (stencil on p2)
// then a CTA barrier and a release of the band's iteration counter.  Band b
// starts iteration c once band b-1 has completed c + DOWN iterations; the
// only upward coupling is a loose bound (band b+1 at most UP iterations
// behind) that keeps ring slots and r_entry alive for their readers.  p1,
// p2 and u live in per-band global ring buffers (L2-resident); r is
// overwritten in place by the final r stage only.
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

namespace ocmg {

constexpr int kWfStride = 38;
constexpr int kWfTableDoubles = 49 * kWfStride;

namespace wf {
constexpr int ROWS = 32;            // lanes = band rows incl. ghosts
constexpr int REAL = 29;            // rows owned by a band
constexpr int CW = 32;              // columns per chunk
constexpr int RING = 16;            // global ring depth, chunks
constexpr int RW = RING * CW;       // 512
constexpr int WIN = 4 * CW;         // smem window / G ring width (128)
constexpr int LAG_U = 4, LAG_G = 6, LAG_A = 7, LAG_R = 10;
constexpr int DOWN = 3, UP = 8;
constexpr int FLAG_STRIDE = 64;     // ints between band counters (256 B)
// rows produced per stage (lanes 0..n-1): chain 1 all 32, u 31, G2 30,
// chain 2 30, r 29 (= REAL)
constexpr int ROWS_U = REAL + 2, ROWS_G2 = REAL + 1, ROWS_C2 = REAL + 1;
constexpr int HR = 8;               // rows per helper warp
constexpr int HPS = ROWS / HR;      // helper warps per stage (4 stages)
constexpr int NWARPS = 3 + 4 * HPS;
constexpr int NTHREADS = NWARPS * 32;
// shared memory (doubles)
constexpr int SM_AW = kP1Classes * 28 * 2;     // A and W tables
constexpr int SM_WF = kWfTableDoubles;
constexpr int SM_WIN = ROWS * WIN;              // one chain window
constexpr int SM_EXT = 2 * WIN;                 // rows -2, -1 of one chain
constexpr int SM_G = ROWS * WIN;                // one G ring
constexpr int EDGE_W = 2 * (HR + 2) * 2 * 2;    // per helper warp edge slots
constexpr int SM_EDGE = (NWARPS - 3) * EDGE_W;
constexpr int SM_TOTAL =
    SM_AW + SM_WF + 2 * SM_WIN + 2 * SM_EXT + 2 * SM_G + SM_EDGE;
constexpr size_t SM_BYTES = SM_TOTAL * sizeof(double);
}  // namespace wf

struct WfParams {
    int n1, nb, nch, niter;
    const double *T;    // P1 tables (device)
    const double *WF;   // delta tables (device)
    double *x, *r;
    double *ring1, *ring2;  // [nb][ROWS][RW]
    double *ringu;          // [nb][2][ROWS][RW]
    int *iter;              // [nb * FLAG_STRIDE] completed iterations
    unsigned long long *prof;  // OCMG_WF_PROFILE: [nb][niter][NWARPS][2] ns
};

namespace wfd {

__device__ __forceinline__ void cp_async8_ca(double *s, const double *g) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(g)
                 : "memory");
}
// 16-byte copy that bypasses L1 (ring data is rewritten by other CTAs)
__device__ __forceinline__ void cp_async16_cg(double *s, const double *g) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(g)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool BWD>
struct Geo {
    int n1;
    int64_t N;
    __device__ __forceinline__ int ax(int i) const { return BWD ? n1 - 1 - i : i; }
    // actual linear vertex index of reflected coordinates
    __device__ __forceinline__ int64_t vid(int ixr, int iyr) const {
        return (int64_t)ax(iyr) * n1 + ax(ixr);
    }
    __device__ __forceinline__ int cls(int ixr, int iyr) const {
        return 7 * p1_axis_class(ax(iyr), n1) + p1_axis_class(ax(ixr), n1);
    }
    __device__ __forceinline__ bool in(int ixr, int iyr) const {
        return ixr >= 0 && ixr < n1 && iyr >= 0 && iyr < n1;
    }
};

}  // namespace wfd

// ---------------------------------------------------------------------------
// device-side context (one copy in shared memory, read by every stage)
// ---------------------------------------------------------------------------
struct WfCtx {
    WfParams P;
    int b, iy0, nreal;
    int64_t N, ps1, psu;
    const double *sAW;  // A then W tables (smem)
    const double *sWF;  // delta tables (smem)
};

template <bool BWD>
__device__ __forceinline__ int64_t wf_vid(const WfCtx *C, int ixr, int iyr) {
    const int n1 = C->P.n1;
    const int ax = BWD ? n1 - 1 - ixr : ixr, ay = BWD ? n1 - 1 - iyr : iyr;
    return (int64_t)ay * n1 + ax;
}
template <bool BWD>
__device__ __forceinline__ int wf_cls(const WfCtx *C, int ixr, int iyr) {
    const int n1 = C->P.n1;
    const int ax = BWD ? n1 - 1 - ixr : ixr, ay = BWD ? n1 - 1 - iyr : iyr;
    return 7 * p1_axis_class(ay, n1) + p1_axis_class(ax, n1);
}
__device__ __forceinline__ bool wf_in(const WfCtx *C, int ixr, int iyr) {
    const int n1 = C->P.n1;
    return ixr >= 0 && ixr < n1 && iyr >= 0 && iyr < n1;
}

// ring element of band-relative row i (row -1 is band b-1's lane REAL-1;
// rows >= 0 are this band's lanes below `rowlimit`), nullptr outside
__device__ __forceinline__ double *wf_ring_ptr(const WfCtx *C, double *ring,
                                               int64_t pstride, int i, int xr,
                                               int rowlimit) {
    using namespace wf;
    const int iyr = C->iy0 + i, n1 = C->P.n1;
    if (xr < 0 || xr >= n1 || iyr < 0 || iyr >= n1 || i >= rowlimit)
        return nullptr;
    int bb = C->b, ii = i;
    if (i < 0) {
        bb -= 1;
        ii = REAL + i;
    }
    if (bb < 0) return nullptr;
    return ring + (int64_t)bb * pstride + (int64_t)ii * RW + (xr & (RW - 1));
}

// source of a G stage: kind 0 = r_entry (reference layout), 1 = u ring
template <bool BWD>
__device__ __forceinline__ const double *wf_gsrc(const WfCtx *C, int kind,
                                                 int i, int xr, int f) {
    using namespace wf;
    if (kind == 0) {
        const int iyr = C->iy0 + i;
        return wf_in(C, xr, iyr) ? C->P.r + f * C->N + wf_vid<BWD>(C, xr, iyr)
                                 : nullptr;
    }
    return wf_ring_ptr(C, C->P.ringu + (int64_t)f * ROWS * RW, C->psu, i, xr,
                       ROWS_U);
}

// ---- scout: wait for iteration `it`'s neighbour progress, stage ext ------
template <bool BWD>
__device__ __noinline__ void wf_scout(const WfCtx *C, int it, double *ext1,
                                      double *ext2) {
    using namespace wf;
    const int lane = threadIdx.x & 31, b = C->b, nb = C->P.nb, n1 = C->P.n1;
    if (lane == 0) {
        const int need_dn = min(it + DOWN, C->P.niter);
        const int need_up = it - UP;
        if (b > 0)
            while (wfd::ld_relaxed(C->P.iter + (b - 1) * FLAG_STRIDE) < need_dn)
                __nanosleep(100);
        if (b + 1 < nb && need_up > 0)
            while (wfd::ld_relaxed(C->P.iter + (b + 1) * FLAG_STRIDE) < need_up)
                __nanosleep(100);
        wfd::fence_acquire();
    }
    __syncwarp();
    if (b == 0) return;
    // band b-1's lanes REAL-2, REAL-1 (rows -2, -1) for chunks it, it+1
    // (chain 1) and it-A, it-A+1 (chain 2): 256 values, 8 per lane
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = lane + 32 * k;
        const int chain = q >> 7, row = (q >> 6) & 1, col = q & 63;
        const int ch = (chain == 0 ? it : it - LAG_A) + (col >> 5);
        const int ixr = ch * CW + (col & 31);
        v[k] = 0.0;
        if (ch >= 0 && ixr < n1) {
            const double *ring = chain == 0 ? C->P.ring1 : C->P.ring2;
            v[k] = __ldcg(ring + (int64_t)(b - 1) * C->ps1 +
                          (int64_t)(REAL - 2 + row) * RW + (ixr & (RW - 1)));
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = lane + 32 * k;
        const int chain = q >> 7, row = (q >> 6) & 1, col = q & 63;
        const int ch = (chain == 0 ? it : it - LAG_A) + (col >> 5);
        const int ixr = ch * CW + (col & 31);
        double *ext = chain == 0 ? ext1 : ext2;
        if (ixr >= 0) ext[row * WIN + (ixr & (WIN - 1))] = v[k];
    }
}

// ---- chain: 32 skewed wavefront steps of one chunk ------------------------
template <bool BWD>
__device__ __noinline__ void wf_chain(const WfCtx *C, int jc, int nbase,
                                      int inv, int nrows, double *win,
                                      const double *ext, const double *gring,
                                      double *ring) {
    using namespace wf;
    const int i = threadIdx.x & 31, n1 = C->P.n1;
    const int iyr = C->iy0 + i;
    const bool rowok = iyr < n1 && i < nrows;
    const double *rm1 = i >= 1 ? win + (i - 1) * WIN : ext + WIN;
    const double *rm2 = i >= 2 ? win + (i - 2) * WIN : ext + i * WIN;
    double *own = win + i * WIN;
    const double *gi = gring + i * WIN;
    double *rg = ring + (int64_t)C->b * C->ps1 + (int64_t)i * RW;
    const double *sWF = C->sWF;
    for (int s = 0; s < CW; ++s) {
        const int ixr = jc * CW - 2 * i + s;
        double p = 0.0;
        if (rowok && ixr >= 0 && ixr < n1) {
            const int c = wf_cls<BWD>(C, ixr, iyr);
            const double *Nc = sWF + c * kWfStride + nbase;
            const int m2 = (ixr - 2) & (WIN - 1), m1 = (ixr - 1) & (WIN - 1);
            const int z0 = ixr & (WIN - 1), p1 = (ixr + 1) & (WIN - 1);
            double q = gi[z0];
            q = fma(-Nc[0], rm2[m2], q);
            q = fma(-Nc[1], rm2[m1], q);
            q = fma(-Nc[2], rm2[z0], q);
            q = fma(-Nc[3], rm1[m2], q);
            q = fma(-Nc[4], rm1[m1], q);
            q = fma(-Nc[5], rm1[z0], q);
            q = fma(-Nc[7], own[m2], q);
            q = fma(-Nc[6], rm1[p1], q);
            q = fma(-Nc[8], own[m1], q);
            p = q * sWF[c * kWfStride + inv];
            rg[ixr & (RW - 1)] = p;
        }
        if (ixr >= -2 * CW) own[ixr & (WIN - 1)] = p;
        __syncwarp();
    }
}

// ---- helper stencils: lane = column, HR rows per warp ---------------------
// Every load of a tile (HR+2 rows of the own column) is issued before any
// arithmetic, so a stage costs one L2 round trip; the lane-0 / lane-31 edge
// columns go through a per-warp smem buffer filled by cp.async (left and
// right edges in disjoint halves of `ebuf`).
__device__ __forceinline__ double wf_ld(const double *p) {
    return p ? __ldcg(p) : 0.0;
}
__device__ __forceinline__ void wf_edge_fetch(double *slot, const double *p,
                                              bool ring, int lane) {
    if (!p) {
        slot[0] = 0.0;
        slot[1] = 0.0;
    } else if (ring) {
        wfd::cp_async16_cg(slot, lane == 0 ? p - 1 : p);
    } else {
        wfd::cp_async8_ca(slot + (lane == 0 ? 1 : 0), p);
    }
}

// G for chain field F on chunk j, rows [rlo, rlo+HR) below `nrows`:
// gring <- W_F . src  (src kind 0: r_entry, 1: u ring)
template <bool BWD>
__device__ __noinline__ void wf_stage_G(const WfCtx *C, int j, int F,
                                        double *gring, int kind, int rlo,
                                        int nrows, double *ebuf) {
    using namespace wf;
    const int lane = threadIdx.x & 31;
    const bool edge = lane == 0 || lane == 31;
    const int ixr = j * CW + lane, xe = ixr + (lane == 0 ? -1 : 1);
    const int eo = lane == 0 ? 1 : 0;
    double v[HR + 2][2];
#pragma unroll
    for (int t = 0; t < HR + 2; ++t)
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            v[t][f] = wf_ld(wf_gsrc<BWD>(C, kind, rlo - 1 + t, ixr, f));
            if (edge)
                wf_edge_fetch(ebuf + 2 * (2 * t + f),
                              wf_gsrc<BWD>(C, kind, rlo - 1 + t, xe, f),
                              kind != 0, lane);
        }
    wfd::cp_async_wait_all();
    __syncwarp();
    const double *W = C->sAW + kP1Classes * 28 + F * 14;
#pragma unroll
    for (int t = 1; t <= HR; ++t) {
        const int i = rlo - 1 + t;
        const int iyr = C->iy0 + i;
        double lp[2], lc[2], rc[2], rn[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const double a = __shfl_up_sync(0xffffffffu, v[t - 1][f], 1);
            const double bq = __shfl_up_sync(0xffffffffu, v[t][f], 1);
            const double cq = __shfl_down_sync(0xffffffffu, v[t][f], 1);
            const double d = __shfl_down_sync(0xffffffffu, v[t + 1][f], 1);
            lp[f] = lane == 0 ? ebuf[2 * (2 * (t - 1) + f) + eo] : a;
            lc[f] = lane == 0 ? ebuf[2 * (2 * t + f) + eo] : bq;
            rc[f] = lane == 31 ? ebuf[2 * (2 * t + f) + eo] : cq;
            rn[f] = lane == 31 ? ebuf[2 * (2 * (t + 1) + f) + eo] : d;
        }
        if (i < nrows && wf_in(C, ixr, iyr)) {
            const double *w = W + wf_cls<BWD>(C, ixr, iyr) * 28;
            double g = 0.0;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const double *wf_ = w + 7 * f;
                g = fma(wf_[BWD ? 6 : 0], lp[f], g);
                g = fma(wf_[BWD ? 5 : 1], v[t - 1][f], g);
                g = fma(wf_[BWD ? 4 : 2], lc[f], g);
                g = fma(wf_[3], v[t][f], g);
                g = fma(wf_[BWD ? 2 : 4], rc[f], g);
                g = fma(wf_[BWD ? 1 : 5], v[t + 1][f], g);
                g = fma(wf_[BWD ? 0 : 6], rn[f], g);
            }
            gring[i * WIN + (ixr & (WIN - 1))] = g;
        }
    }
}

// out_f = base_f - A[f, FP] p  for both fields f (rows below `nrows`), and
// x_FP += p on the band's real rows.  p from ring1 (which=0) or ring2;
// base kind 0: r_entry, 1: u ring; out kind 0: u ring, 1: r.
template <bool BWD>
__device__ __noinline__ void wf_stage_apply(const WfCtx *C, int j, int FP,
                                            int which, int prows, int bkind,
                                            int okind, int rlo, int nrows,
                                            double *ebuf) {
    using namespace wf;
    const int lane = threadIdx.x & 31;
    const bool edge = lane == 0 || lane == 31;
    const int ixr = j * CW + lane, xe = ixr + (lane == 0 ? -1 : 1);
    const int eo = lane == 0 ? 1 : 0;
    double *pring = which == 0 ? C->P.ring1 : C->P.ring2;
    const int64_t N = C->N;
    double pv[HR + 2], bv[HR][2], xv[HR];
#pragma unroll
    for (int t = 0; t < HR + 2; ++t) {
        pv[t] = wf_ld(wf_ring_ptr(C, pring, C->ps1, rlo - 1 + t, ixr, prows));
        if (edge)
            wf_edge_fetch(ebuf + 2 * t,
                          wf_ring_ptr(C, pring, C->ps1, rlo - 1 + t, xe, prows),
                          true, lane);
    }
#pragma unroll
    for (int t = 0; t < HR; ++t) {
        const int i = rlo + t;
        const int iyr = C->iy0 + i;
        const bool ok = i < nrows && wf_in(C, ixr, iyr);
#pragma unroll
        for (int f = 0; f < 2; ++f)
            bv[t][f] = ok ? wf_ld(wf_gsrc<BWD>(C, bkind, i, ixr, f)) : 0.0;
        xv[t] = (ok && i < C->nreal) ? C->P.x[FP * N + wf_vid<BWD>(C, ixr, iyr)]
                                     : 0.0;
    }
    wfd::cp_async_wait_all();
    __syncwarp();
#pragma unroll
    for (int t = 1; t <= HR; ++t) {
        const int i = rlo - 1 + t;
        const int iyr = C->iy0 + i;
        const double su = __shfl_up_sync(0xffffffffu, pv[t - 1], 1);
        const double sc = __shfl_up_sync(0xffffffffu, pv[t], 1);
        const double dc = __shfl_down_sync(0xffffffffu, pv[t], 1);
        const double dn = __shfl_down_sync(0xffffffffu, pv[t + 1], 1);
        const double lp = lane == 0 ? ebuf[2 * (t - 1) + eo] : su;
        const double lc = lane == 0 ? ebuf[2 * t + eo] : sc;
        const double rc = lane == 31 ? ebuf[2 * t + eo] : dc;
        const double rn = lane == 31 ? ebuf[2 * (t + 1) + eo] : dn;
        if (i < nrows && wf_in(C, ixr, iyr)) {
            const double *a = C->sAW + wf_cls<BWD>(C, ixr, iyr) * 28 + FP * 7;
            const int64_t v = wf_vid<BWD>(C, ixr, iyr);
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const double *af = a + 14 * f;
                double w = bv[t - 1][f];
                w = fma(-af[BWD ? 6 : 0], lp, w);
                w = fma(-af[BWD ? 5 : 1], pv[t - 1], w);
                w = fma(-af[BWD ? 4 : 2], lc, w);
                w = fma(-af[3], pv[t], w);
                w = fma(-af[BWD ? 2 : 4], rc, w);
                w = fma(-af[BWD ? 1 : 5], pv[t + 1], w);
                w = fma(-af[BWD ? 0 : 6], rn, w);
                if (okind == 0)
                    C->P.ringu[(int64_t)C->b * C->psu + (int64_t)f * ROWS * RW +
                               (int64_t)i * RW + (ixr & (RW - 1))] = w;
                else
                    C->P.r[f * N + v] = w;
            }
            if (i < C->nreal) C->P.x[FP * N + v] = xv[t - 1] + pv[t];
        }
    }
}

// ---------------------------------------------------------------------------
// interior fast paths.  When every node a call touches has the interior
// position class (axis class 3 on both axes; true for ~97% of the tiles of
// a large level), coefficients are loop-invariant (held in registers),
// every neighbour exists, and addresses are plain strides: the calls below
// do the same arithmetic as the generic versions without any per-node
// class lookup or bounds logic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool wf_interior_rows(const WfCtx *C, int r0, int r1) {
    return C->iy0 + r0 >= 3 && C->iy0 + r1 <= C->P.n1 - 4;
}
__device__ __forceinline__ bool wf_interior_cols(const WfCtx *C, int c0, int c1) {
    return c0 >= 3 && c1 <= C->P.n1 - 4;
}
constexpr int kMidClass = 7 * 3 + 3;

template <bool BWD>
__device__ __noinline__ void wf_chain_fast(const WfCtx *C, int jc, int nbase,
                                           int inv, double *win,
                                           const double *ext,
                                           const double *gring, double *ring) {
    using namespace wf;
    const int i = threadIdx.x & 31;
    const double *rm1 = i >= 1 ? win + (i - 1) * WIN : ext + WIN;
    const double *rm2 = i >= 2 ? win + (i - 2) * WIN : ext + i * WIN;
    double *own = win + i * WIN;
    const double *gi = gring + i * WIN;
    double *rg = ring + (int64_t)C->b * C->ps1 + (int64_t)i * RW;
    const double *Nc = C->sWF + kMidClass * kWfStride + nbase;
    const double n0 = -Nc[0], n1c = -Nc[1], n2 = -Nc[2], n3 = -Nc[3], n4 = -Nc[4],
                 n5 = -Nc[5], n6 = -Nc[6], n7 = -Nc[7], n8 = -Nc[8];
    const double ninv = C->sWF[kMidClass * kWfStride + inv];
    int ixr = jc * CW - 2 * i;
    double o1 = own[(ixr - 1) & (WIN - 1)], o2 = own[(ixr - 2) & (WIN - 1)];
#pragma unroll 4
    for (int s = 0; s < CW; ++s, ++ixr) {
        const int m2 = (ixr - 2) & (WIN - 1), m1 = (ixr - 1) & (WIN - 1);
        const int z0 = ixr & (WIN - 1), p1 = (ixr + 1) & (WIN - 1);
        double q = gi[z0];
        q = fma(n0, rm2[m2], q);
        q = fma(n1c, rm2[m1], q);
        q = fma(n2, rm2[z0], q);
        q = fma(n3, rm1[m2], q);
        q = fma(n4, rm1[m1], q);
        q = fma(n5, rm1[z0], q);
        q = fma(n7, o2, q);
        q = fma(n6, rm1[p1], q);
        q = fma(n8, o1, q);
        const double p = q * ninv;
        rg[ixr & (RW - 1)] = p;
        own[z0] = p;
        o2 = o1;
        o1 = p;
        __syncwarp();
    }
}

template <bool BWD>
__device__ __noinline__ void wf_stage_G_fast(const WfCtx *C, int j, int F,
                                             double *gring, int kind, int rlo,
                                             int nrows, double *ebuf) {
    using namespace wf;
    const int lane = threadIdx.x & 31;
    const bool edge = lane == 0 || lane == 31;
    const int ixr = j * CW + lane;
    const int eo = lane == 0 ? 1 : 0;
    const int n1 = C->P.n1;
    const int64_t N = C->N;
    double v[HR + 2][2];
    // row pointers of the two source fields
    const double *p0[2];
    int64_t rstep;
    if (kind == 0) {
        const int64_t L = (int64_t)(C->iy0 + rlo - 1) * n1 + ixr;
        for (int f = 0; f < 2; ++f) p0[f] = C->P.r + f * N + (BWD ? N - 1 - L : L);
        rstep = BWD ? -n1 : n1;
    } else {
        for (int f = 0; f < 2; ++f)
            p0[f] = C->P.ringu + (int64_t)C->b * C->psu + (int64_t)f * ROWS * RW +
                    (int64_t)(rlo - 1) * RW + (ixr & (RW - 1));
        rstep = RW;
    }
    const int ldx = (kind == 0 && BWD) ? 1 : -1;  // address step of col - 1
#pragma unroll
    for (int t = 0; t < HR + 2; ++t)
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const double *p = p0[f] + t * rstep;
            if (kind != 0 && rlo - 1 + t < 0)  // row -1: band b-1's lane REAL-1
                p = C->P.ringu + (int64_t)(C->b - 1) * C->psu +
                    (int64_t)f * ROWS * RW + (int64_t)(REAL - 1) * RW +
                    (ixr & (RW - 1));
            v[t][f] = __ldcg(p);
            if (edge) {
                double *slot = ebuf + 2 * (2 * t + f);
                if (kind == 0) {
                    wfd::cp_async8_ca(slot + eo, p + (lane == 0 ? ldx : -ldx));
                } else {  // ring: aligned pair holding the edge, slot wrap
                    const double *row = p - (ixr & (RW - 1));
                    wfd::cp_async16_cg(
                        slot, row + ((lane == 0 ? ixr - 2 : ixr + 1) & (RW - 1)));
                }
            }
        }
    wfd::cp_async_wait_all();
    __syncwarp();
    const double *w = C->sAW + kP1Classes * 28 + kMidClass * 28 + F * 14;
    double W0[7], W1[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) {
        W0[d] = w[BWD ? 6 - d : d];
        W1[d] = w[7 + (BWD ? 6 - d : d)];
    }
#pragma unroll
    for (int t = 1; t <= HR; ++t) {
        const int i = rlo - 1 + t;
        double g = 0.0;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const double *Wf = f ? W1 : W0;
            const double a = __shfl_up_sync(0xffffffffu, v[t - 1][f], 1);
            const double bq = __shfl_up_sync(0xffffffffu, v[t][f], 1);
            const double cq = __shfl_down_sync(0xffffffffu, v[t][f], 1);
            const double d = __shfl_down_sync(0xffffffffu, v[t + 1][f], 1);
            const double lp = lane == 0 ? ebuf[2 * (2 * (t - 1) + f) + eo] : a;
            const double lc = lane == 0 ? ebuf[2 * (2 * t + f) + eo] : bq;
            const double rc = lane == 31 ? ebuf[2 * (2 * t + f) + eo] : cq;
            const double rn = lane == 31 ? ebuf[2 * (2 * (t + 1) + f) + eo] : d;
            g = fma(Wf[0], lp, g);
            g = fma(Wf[1], v[t - 1][f], g);
            g = fma(Wf[2], lc, g);
            g = fma(Wf[3], v[t][f], g);
            g = fma(Wf[4], rc, g);
            g = fma(Wf[5], v[t + 1][f], g);
            g = fma(Wf[6], rn, g);
        }
        if (i < nrows) gring[i * WIN + (ixr & (WIN - 1))] = g;
    }
}

// rows rlo + o .. rlo + o + M - 1 of the apply stage (see below)
template <bool BWD, int M>
__device__ __forceinline__ void wf_apply_part(const WfCtx *C, int j, int FP, int which,
                                              int bkind, int okind, int rlo, int o,
                                              int nrows, double *ebuf) {
    using namespace wf;
    const int lane = threadIdx.x & 31;
    const bool edge = lane == 0 || lane == 31;
    const int ixr = j * CW + lane;
    const int eo = lane == 0 ? 1 : 0;
    const int n1 = C->P.n1;
    const int64_t N = C->N;
    double *pring = which == 0 ? C->P.ring1 : C->P.ring2;
    const int slot = ixr & (RW - 1);
    double pv[M + 2], bv[M][2], xv[M];
#pragma unroll
    for (int t = 0; t < M + 2; ++t) {
        const int i = rlo + o - 1 + t;
        const double *p =
            i < 0 ? pring + (int64_t)(C->b - 1) * C->ps1 + (int64_t)(REAL - 1) * RW + slot
                  : pring + (int64_t)C->b * C->ps1 + (int64_t)i * RW + slot;
        pv[t] = __ldcg(p);
        if (edge)
            wfd::cp_async16_cg(ebuf + 2 * t,
                               p - slot + ((lane == 0 ? ixr - 2 : ixr + 1) & (RW - 1)));
    }
    const int64_t L0 = (int64_t)(C->iy0 + rlo + o) * n1 + ixr;  // actual for FWD
    const int64_t lstep = BWD ? -n1 : n1;
    const int64_t lin0 = BWD ? N - 1 - L0 : L0;
#pragma unroll
    for (int t = 0; t < M; ++t) {
        const int64_t lin = lin0 + t * lstep;
#pragma unroll
        for (int f = 0; f < 2; ++f)
            bv[t][f] = bkind == 0
                           ? __ldcg(C->P.r + f * N + lin)
                           : __ldcg(C->P.ringu + (int64_t)C->b * C->psu +
                                    (int64_t)f * ROWS * RW +
                                    (int64_t)(rlo + o + t) * RW + slot);
        xv[t] = __ldcg(C->P.x + FP * N + lin);
    }
    wfd::cp_async_wait_all();
    __syncwarp();
    // stencil coefficients read from shared memory at each use (broadcast):
    // held in registers they pushed this stage over the 96-register cap of a
    // 19-warp CTA and it spilled
    const double *a = C->sAW + kMidClass * 28 + FP * 7;
    auto A0 = [&](int d) { return -a[BWD ? 6 - d : d]; };
    auto A1 = [&](int d) { return -a[14 + (BWD ? 6 - d : d)]; };
#pragma unroll
    for (int t = 1; t <= M; ++t) {
        const int i = rlo + o - 1 + t;
        const double su = __shfl_up_sync(0xffffffffu, pv[t - 1], 1);
        const double sc = __shfl_up_sync(0xffffffffu, pv[t], 1);
        const double dc = __shfl_down_sync(0xffffffffu, pv[t], 1);
        const double dn = __shfl_down_sync(0xffffffffu, pv[t + 1], 1);
        const double lp = lane == 0 ? ebuf[2 * (t - 1) + eo] : su;
        const double lc = lane == 0 ? ebuf[2 * t + eo] : sc;
        const double rc = lane == 31 ? ebuf[2 * t + eo] : dc;
        const double rn = lane == 31 ? ebuf[2 * (t + 1) + eo] : dn;
        if (i < nrows) {
            const int64_t lin = lin0 + (t - 1) * lstep;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                auto Af = [&](int d) { return f ? A1(d) : A0(d); };
                double w = bv[t - 1][f];
                w = fma(Af(0), lp, w);
                w = fma(Af(1), pv[t - 1], w);
                w = fma(Af(2), lc, w);
                w = fma(Af(3), pv[t], w);
                w = fma(Af(4), rc, w);
                w = fma(Af(5), pv[t + 1], w);
                w = fma(Af(6), rn, w);
                if (okind == 0)
                    C->P.ringu[(int64_t)C->b * C->psu + (int64_t)f * ROWS * RW +
                               (int64_t)i * RW + slot] = w;
                else
                    C->P.r[f * N + lin] = w;
            }
            if (i < C->nreal) C->P.x[FP * N + lin] = xv[t - 1] + pv[t];
        }
    }
    __syncwarp();  // ebuf is reused by the next part
}

// the apply stages on an interior tile, in two halves of HR/2 rows: the
// loads of all HR rows in flight at once spilled under the 96-register cap,
// and a spill of a loaded value waits for the load
template <bool BWD>
__device__ __noinline__ void wf_stage_apply_fast(const WfCtx *C, int j, int FP,
                                                 int which, int bkind,
                                                 int okind, int rlo, int nrows,
                                                 double *ebuf) {
    wf_apply_part<BWD, wf::HR / 2>(C, j, FP, which, bkind, okind, rlo, 0, nrows, ebuf);
    wf_apply_part<BWD, wf::HR / 2>(C, j, FP, which, bkind, okind, rlo, wf::HR / 2, nrows, ebuf);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <bool BWD>
__global__ void __launch_bounds__(wf::NTHREADS, 1)
k_wavefront(WfParams P) {
    using namespace wf;
    extern __shared__ double sm[];
    __shared__ WfCtx ctx;
    double *sAW = sm;                  // A then W
    double *sWF = sAW + SM_AW;
    double *win1 = sWF + SM_WF;
    double *win2 = win1 + SM_WIN;
    double *ext1 = win2 + SM_WIN;
    double *ext2 = ext1 + SM_EXT;
    double *g1 = ext2 + SM_EXT;
    double *g2 = g1 + SM_G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // fields: chain 1 works on F1, chain 2 on F2 (0 state, 1 adjoint)
    constexpr int F1 = BWD ? 1 : 0, F2 = 1 - F1;
    constexpr int NB1 = BWD ? 27 : 0;    // N coefficients of chain 1
    constexpr int NB2 = BWD ? 18 : 9;    // ... of chain 2
    constexpr int INV1 = 36 + F1, INV2 = 36 + F2;

    if (threadIdx.x == 0) {
        ctx.P = P;
        ctx.b = blockIdx.x;
        ctx.iy0 = blockIdx.x * REAL;
        ctx.nreal = min(REAL, P.n1 - ctx.iy0);
        ctx.N = (int64_t)P.n1 * P.n1;
        ctx.ps1 = (int64_t)ROWS * RW;
        ctx.psu = 2 * (int64_t)ROWS * RW;
        ctx.sAW = sAW;
        ctx.sWF = sWF;
    }
    for (int t = threadIdx.x; t < SM_AW; t += blockDim.x) sAW[t] = P.T[t];
    for (int t = threadIdx.x; t < SM_WF; t += blockDim.x) sWF[t] = P.WF[t];
    for (int t = threadIdx.x; t < 2 * SM_WIN + 2 * SM_EXT + 2 * SM_G;
         t += blockDim.x)
        win1[t] = 0.0;
    __syncthreads();
    const WfCtx *C = &ctx;

    const int hw = warp - 3;            // helper warp index 0..15
    const int stage = hw >= 0 ? hw / HPS : -1;
    const int rlo = hw >= 0 ? (hw % HPS) * HR : 0;
    double *ebuf = sm + SM_TOTAL - SM_EDGE + (hw >= 0 ? hw : 0) * EDGE_W +
                   (lane == 31 ? EDGE_W / 2 : 0);

#ifdef OCMG_WF_PROFILE
    auto gtimer = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        return t;
    };
#endif
    // iteration -1 is the prologue: G1 of chunk 0 and the scout for 0
    for (int c = -1; c < P.niter; ++c) {
#ifdef OCMG_WF_PROFILE
        const unsigned long long t_begin = gtimer();
#endif
        // interior tests are warp-uniform: band rows x chunk columns
        const bool band_int = wf_interior_rows(C, 0, ROWS - 1);
        const bool rows_int = hw >= 0 && wf_interior_rows(C, rlo, rlo + HR - 1);
        auto cols_int = [&](int j) {
            return wf_interior_cols(C, j * CW, j * CW + CW - 1);
        };
        if (warp == 0) {
            if (c >= 0 && c < P.nch + 2) {
                if (band_int && wf_interior_cols(C, c * CW - 2 * (ROWS - 1), c * CW + CW - 1))
                    wf_chain_fast<BWD>(C, c, NB1, INV1, win1, ext1, g1, P.ring1);
                else
                    wf_chain<BWD>(C, c, NB1, INV1, ROWS, win1, ext1, g1, P.ring1);
            }
        } else if (warp == 1) {
            const int jc = c - LAG_A;
            if (jc >= 0 && jc < P.nch + 2) {
                if (band_int && wf_interior_cols(C, jc * CW - 2 * (ROWS - 1), jc * CW + CW - 1))
                    wf_chain_fast<BWD>(C, jc, NB2, INV2, win2, ext2, g2, P.ring2);
                else
                    wf_chain<BWD>(C, jc, NB2, INV2, ROWS_C2, win2, ext2, g2, P.ring2);
            }
        } else if (warp == 2) {
            if (c + 1 < P.niter) wf_scout<BWD>(C, c + 1, ext1, ext2);
        } else if (stage == 0) {
            const int j = c + 1;
            if (j < P.nch) {
                if (rows_int && cols_int(j))
                    wf_stage_G_fast<BWD>(C, j, F1, g1, 0, rlo, ROWS, ebuf);
                else
                    wf_stage_G<BWD>(C, j, F1, g1, 0, rlo, ROWS, ebuf);
            }
        } else if (stage == 1) {
            const int j = c - LAG_U;
            if (j >= 0 && j < P.nch) {
                if (rows_int && cols_int(j))
                    wf_stage_apply_fast<BWD>(C, j, F1, 0, 0, 0, rlo, ROWS_U, ebuf);
                else
                    wf_stage_apply<BWD>(C, j, F1, 0, ROWS, 0, 0, rlo, ROWS_U, ebuf);
            }
        } else if (stage == 2) {
            const int j = c - LAG_G;
            if (j >= 0 && j < P.nch) {
                if (rows_int && cols_int(j))
                    wf_stage_G_fast<BWD>(C, j, F2, g2, 1, rlo, ROWS_G2, ebuf);
                else
                    wf_stage_G<BWD>(C, j, F2, g2, 1, rlo, ROWS_G2, ebuf);
            }
        } else {
            const int j = c - LAG_R;
            if (j >= 0 && j < P.nch) {
                if (rows_int && cols_int(j))
                    wf_stage_apply_fast<BWD>(C, j, F2, 1, 1, 1, rlo, ctx.nreal, ebuf);
                else
                    wf_stage_apply<BWD>(C, j, F2, 1, ROWS_C2, 1, 1, rlo, ctx.nreal,
                                        ebuf);
            }
        }
#ifdef OCMG_WF_PROFILE
        if (lane == 0 && P.prof && c >= 0) {
            unsigned long long *pp =
                P.prof + (((int64_t)blockIdx.x * P.niter + c) * NWARPS + warp) * 2;
            pp[0] = t_begin;
            pp[1] = gtimer();
        }
#endif
        __syncthreads();
        if (threadIdx.x == 0 && c >= 0)
            wfd::st_release(P.iter + blockIdx.x * FLAG_STRIDE, c + 1);
    }
}
// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct P1Wavefront {
    int k = 0, n1 = 0, nb = 0, nch = 0, niter = 0;
    const double *T = nullptr;
    const double *tab = nullptr;  // device WF tables
    DevBuf<double> ring1, ring2, ringu;
    DevBuf<int> iter;
    DevBuf<unsigned long long> prof;
    bool ok = false;

    void init(int k_, int n1_, const double *T_, const double *wf_tab) {
        k = k_;
        n1 = n1_;
        T = T_;
        tab = wf_tab;
        nb = (n1 + wf::REAL - 1) / wf::REAL;
        nch = (n1 + wf::CW - 1) / wf::CW;
        niter = nch + wf::LAG_R;
        int dev = 0, sms = 0, coop = 0;
        OCMG_CUDA(cudaGetDevice(&dev));
        OCMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        OCMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        OCMG_CUDA(cudaFuncSetAttribute(k_wavefront<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)wf::SM_BYTES));
        OCMG_CUDA(cudaFuncSetAttribute(k_wavefront<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)wf::SM_BYTES));
        int per_sm = 0;
        OCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_wavefront<false>, wf::NTHREADS, wf::SM_BYTES));
        if (!coop || per_sm < 1 || nb > sms * per_sm) return;  // level too big
        const size_t plane = (size_t)nb * wf::ROWS * wf::RW;
        ring1.alloc(plane);
        ring2.alloc(plane);
        ringu.alloc(2 * plane);
        iter.alloc((size_t)nb * wf::FLAG_STRIDE);
#ifdef OCMG_WF_PROFILE
        prof.alloc((size_t)nb * niter * wf::NWARPS * 2);
#endif
        ok = true;
    }
    bool ready() const { return ok; }

    void sweep(bool forward, double *x, double *r, cudaStream_t s) const {
        WfParams P;
        P.n1 = n1;
        P.nb = nb;
        P.nch = nch;
        P.niter = niter;
        P.T = T;
        P.WF = tab;
        P.x = x;
        P.r = r;
        P.ring1 = ring1.p;
        P.ring2 = ring2.p;
        P.ringu = ringu.p;
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
