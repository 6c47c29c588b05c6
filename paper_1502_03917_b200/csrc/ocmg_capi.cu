// C ABI of the ocmg_b200 library (declared in include/ocmg_b200.h).
//
// Owns the per-level device data (what SmootherState.__init__ precomputes,
// smoothers.py:189-216), the transfers (transfer.py), the coarse LU
// (multigrid.py:67-102) and the on-device cycle driver (multigrid.py:130-204),
// and dispatches to the kernels in ocmg_csr.cuh / ocmg_p1.cuh /
// ocmg_wavefront.cuh.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "ocmg_common.cuh"
#include "ocmg_csr.cuh"
#include "ocmg_p1.cuh"
#include "ocmg_p1_tiled.cuh"
#include "ocmg_p1_mc.cuh"
#include "ocmg_p1_mc2.cuh"
#include "ocmg_p1_mc_small.cuh"
#include "ocmg_p1_gsdiag.cuh"
#include "ocmg_p1_dense.cuh"
#include "ocmg_subcycle.cuh"
#include "ocmg_cgs.cuh"
#include "ocmg_cgs_mc.cuh"
#include "ocmg_wavefront.cuh"

using namespace ocmg;

namespace {
thread_local std::string g_last_error;

template <class F>
int guarded(F &&fn) {
    try {
        fn();
        return OCMG_OK;
    } catch (const Error &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return OCMG_E_STATE;
    }
}

enum LevelKind { kCsr = 0, kP1 = 1 };

struct Schedule {  // rows bucketed by dependency level (or colour)
    DevBuf<int32_t> rows;
    std::vector<int64_t> off;
    DevBuf<int64_t> doff;  // device copy of off (one-CTA sweep)
    std::vector<int32_t> hrows;  // host copy of rows
    // grouped SELL-32: each group's rows in slices of 32 (last one padded
    // with row -1), entries entry-major per slice (build_group_sell)
    bool has_gsell = false;
    std::vector<int64_t> gslice;  // [ngroups + 1] first slice of each group
    DevBuf<int32_t> gsrow, gslen, gscol;
    DevBuf<int64_t> gsbase;
    DevBuf<double> gsval, gsw;
};

}  // namespace

struct ocmg_level {
    int problem = OCMG_POISSON;
    int kind = kCsr;
    int64_t n = 0, nnz = 0;
    std::vector<int64_t> field_off;
    uint32_t pmask = 0;
    // generic CSR
    CsrDev A;
    DevBuf<double> W, L, ndiag;
    SellDev sell;  // A and W again in SELL-32 (residual, NE-Jacobi)
    Schedule sched[2];  // 0 forward, 1 backward
    Schedule colours;
    bool has_colours = false;
    // tiny levels (n <= kDenseN): dense sweep maps [mode: 0 exact, 1
    // multicolour][0 forward, 1 backward], each S^T then T^T (n*n each)
    DevBuf<double> dense[2][2];
    bool has_dense = false;
    // Vanka patches (ocmg_level_set_vanka)
    int64_t vk_np = 0;
    int vk_mmax = 0;
    DevBuf<int64_t> vk_off;
    DevBuf<int32_t> vk_dofs;
    DevBuf<double> vk_inv;
    Schedule vk_sched;  // patches by dependency level, forward order
    int64_t vk_ops = 0;  // touched entries per sweep (kernels.py:130)
    // structured P1
    int k = 0, n1 = 0;
    double alpha = 0.0;
    DevBuf<double> tables;
    P1Coef28 cA{}, cW{};  // class-(3,3) A and row_scaled rows (tiled kernels)
    double cL[2] = {0.0, 0.0};
    P1Wavefront wf;
    // k <= 5: the exact-order sweep as a dense map (ocmg_p1_dense.cuh), S
    // row-major per direction, and its scratch d = S r
    DevBuf<double> pmap[2], pmap_d;
    bool has_pmap = false;
    int mc_tier = 2;          // 0 one-CTA, 1 cooperative, 2 pipelined strips
    int mc_grid = 0;          // tier-1 CTAs
    DevBuf<unsigned> mc_bar;  // tier-1 grid barrier
    McsPlan mc;               // one-launch multicolour sweep geometry
    DevBuf<double> mc_r;      // its out-of-place residual
    DevBuf<double> mc_coef;   // [49][2][29] W row, A row, n_diag
    CgsmPlan cgsm;            // one-launch 3-colour CGS geometry
    double cgs_mk[49][4] = {};  // per class m, k, -m/alpha, det (CGS 2x2)
    double cgs_a24[28] = {};    // interior-class A rows
    double mc_ci[58] = {};    // its class-(3,3) rows
    double mc_cu[mcs::NU] = {};  // their distinct values (mcs::umap)
    // reduction scratch
    DevBuf<double> partial, scal;
};

struct ocmg_transfer {
    int kind = kCsr;
    int64_t nf = 0, nc = 0;
    CsrDev P, R;
    int kc = 0, nc1 = 0, n_fields = 0;
};

struct ocmg_coarse {
    int problem = OCMG_POISSON;
    int64_t n = 0, p_off = 0, mu_off = 0, n_p = 0;
    DevBuf<double> lu;
    DevBuf<int32_t> piv;
    DevBuf<double> inv;  // row-major A^-1 (n <= kCoarseInvMax): the cycle's solve
};

struct ocmg_hierarchy {
    std::vector<ocmg_level *> levels;  // index 0 = hierarchy index 1
    std::vector<ocmg_transfer *> transfers;
    ocmg_coarse *coarse = nullptr;
    ocmg_cycle_config cfg{};
    // per hierarchy index h (0 = coarse): residual r[h] and NE scratch for
    // h>=1, and for h < top: restricted rhs crhs[h], correction corr[h]
    std::vector<DevBuf<double>> r, scratch, crhs, corr;
    DevBuf<double> tmp, scal;
    // fused coarse end of the cycle (ocmg_subcycle.cuh): a visit of hierarchy
    // index sub_hi runs everything below it in one launch (0 = off)
    int sub_hi = 0;
    SubcycleParams sub{};
    size_t sub_smem = 0;
    // collapsed coarse end (setup_collapse): the coarse correction of
    // hierarchy index col_hi + 1, i.e. its rec visits of index col_hi from a
    // zero start, is the dense map col_map (row-major, leading dimension
    // col_ld) applied to the restricted residual (0 = off)
    int col_hi = 0, col_ld = 0;
    DevBuf<double> col_map;
    const double *col_p = nullptr;  // col_map (or, in a build clone, the owner's)
    int64_t col_max_n = 0;
    cudaGraphExec_t graph = nullptr;
    const double *graph_x = nullptr, *graph_f = nullptr;
    cudaStream_t graph_stream = nullptr;
    // legacy-default-stream callers: graphs run on this stream instead
    cudaStream_t own_stream = nullptr;
    cudaEvent_t own_event = nullptr;
    ~ocmg_hierarchy() {
        if (graph) cudaGraphExecDestroy(graph);
        if (own_event) cudaEventDestroy(own_event);
        if (own_stream) cudaStreamDestroy(own_stream);
    }
};

namespace {

// ---------------------------------------------------------------------------
// host-side setup helpers
// ---------------------------------------------------------------------------

// ASAP dependency levels of the sequential NE-GS sweep: unknown i touches
// (reads and writes) r_j for every j in column i = row i; it must follow
// every earlier unknown touching one of those j.
Schedule build_schedule(int64_t n, const int64_t *off, const int64_t *col,
                        bool forward) {
    std::vector<int32_t> lev(n), touch(n, -1);
    int32_t maxlev = -1;
    for (int64_t s = 0; s < n; ++s) {
        const int64_t i = forward ? s : n - 1 - s;
        int32_t m = -1;
        for (int64_t t = off[i]; t < off[i + 1]; ++t)
            m = std::max(m, touch[col[t]]);
        lev[i] = m + 1;
        for (int64_t t = off[i]; t < off[i + 1]; ++t) touch[col[t]] = m + 1;
        maxlev = std::max(maxlev, m + 1);
    }
    Schedule S;
    S.off.assign(maxlev + 2, 0);
    for (int64_t i = 0; i < n; ++i) S.off[lev[i] + 1]++;
    for (size_t l = 1; l < S.off.size(); ++l) S.off[l] += S.off[l - 1];
    std::vector<int32_t> rows(n);
    std::vector<int64_t> fill(S.off.begin(), S.off.end() - 1);
    for (int64_t s = 0; s < n; ++s) {
        const int64_t i = forward ? s : n - 1 - s;
        rows[fill[lev[i]]++] = (int32_t)i;
    }
    S.rows.upload(rows);
    S.doff.upload(S.off);
    S.hrows = std::move(rows);
    return S;
}

// Greedy distance-2 colouring in index order (smallest free colour).
Schedule build_colouring(int64_t n, const int64_t *off, const int64_t *col) {
    std::vector<int32_t> colour(n, -1), mark;
    int32_t ncol = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t t = off[i]; t < off[i + 1]; ++t) {
            const int64_t j = col[t];
            for (int64_t u = off[j]; u < off[j + 1]; ++u) {
                const int32_t c = colour[col[u]];
                if (c >= 0) {
                    if ((int32_t)mark.size() <= c) mark.resize(c + 1, -1);
                    mark[c] = (int32_t)i;
                }
            }
        }
        int32_t c = 0;
        while (c < (int32_t)mark.size() && mark[c] == (int32_t)i) ++c;
        colour[i] = c;
        ncol = std::max(ncol, c + 1);
    }
    Schedule S;
    S.off.assign(ncol + 1, 0);
    for (int64_t i = 0; i < n; ++i) S.off[colour[i] + 1]++;
    for (int c = 1; c <= ncol; ++c) S.off[c] += S.off[c - 1];
    std::vector<int32_t> rows(n);
    std::vector<int64_t> fill(S.off.begin(), S.off.end() - 1);
    for (int64_t i = 0; i < n; ++i) rows[fill[colour[i]]++] = (int32_t)i;
    S.rows.upload(rows);
    S.doff.upload(S.off);
    S.hrows = std::move(rows);
    return S;
}

// the grouped SELL-32 copy of a schedule (A, W of the level's CSR)
void build_group_sell(Schedule &S, int64_t n, const int64_t *row_off,
                      const CsrDev &A, const double *w) {
    const int64_t ng = (int64_t)S.off.size() - 1;
    S.gslice.assign(ng + 1, 0);
    for (int64_t g = 0; g < ng; ++g)
        S.gslice[g + 1] = S.gslice[g] + (S.off[g + 1] - S.off[g] + 31) / 32;
    const int64_t nsl = S.gslice[ng];
    std::vector<int32_t> srow(nsl * 32, -1);
    std::vector<int64_t> base(nsl + 1, 0);
    for (int64_t g = 0; g < ng; ++g)
        for (int64_t k = S.off[g]; k < S.off[g + 1]; ++k)
            srow[S.gslice[g] * 32 + (k - S.off[g])] = S.hrows[k];
    for (int64_t sl = 0; sl < nsl; ++sl) {
        int64_t wmax = 0;
        for (int l = 0; l < 32; ++l) {
            const int32_t i = srow[sl * 32 + l];
            if (i >= 0) wmax = std::max(wmax, row_off[i + 1] - row_off[i]);
        }
        base[sl + 1] = base[sl] + 32 * wmax;
    }
    const int64_t ent = base[nsl];
    S.gsrow.upload(srow);
    S.gsbase.upload(base);
    S.gslen.alloc(nsl * 32);
    S.gscol.alloc(ent);
    S.gsval.alloc(ent);
    S.gsw.alloc(ent);
    OCMG_CUDA(cudaMemset(S.gscol.p, 0, ent * sizeof(int32_t)));
    OCMG_LAUNCH(k_gsell_fill, grid_for(nsl * 32, 256), 256, 0, 0, nsl * 32, S.gsrow.p,
                S.gsbase.p, A.off.p, A.col.p, A.val.p, w, S.gslen.p, S.gscol.p,
                S.gsval.p, S.gsw.p);
    OCMG_LAUNCH_CHECK();
    S.has_gsell = true;
    (void)n;
}

void upload_csr(CsrDev &C, int64_t nrows, int64_t ncols, const int64_t *off,
                const int64_t *col, const double *val) {
    C.n = nrows;
    C.ncols = ncols;
    C.nnz = off[nrows];
    C.off.upload(off, nrows + 1);
    std::vector<int32_t> c32(C.nnz);
    for (int64_t t = 0; t < C.nnz; ++t) {
        OCMG_REQUIRE(col[t] >= 0 && col[t] < ncols, "column index out of range");
        c32[t] = (int32_t)col[t];
    }
    C.col.upload(c32);
    C.val.upload(val, C.nnz);
}

void csr_transpose(int64_t nrows, int64_t ncols, const int64_t *off,
                   const int64_t *col, const double *val,
                   std::vector<int64_t> &toff, std::vector<int64_t> &tcol,
                   std::vector<double> &tval) {
    const int64_t nnz = off[nrows];
    toff.assign(ncols + 1, 0);
    for (int64_t t = 0; t < nnz; ++t) toff[col[t] + 1]++;
    for (int64_t c = 0; c < ncols; ++c) toff[c + 1] += toff[c];
    tcol.resize(nnz);
    tval.resize(nnz);
    std::vector<int64_t> fill(toff.begin(), toff.end() - 1);
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t t = off[i]; t < off[i + 1]; ++t) {
            const int64_t p = fill[col[t]]++;
            tcol[p] = i;
            tval[p] = val[t];
        }
}

// ---------------------------------------------------------------------------
// level operations
// ---------------------------------------------------------------------------

constexpr int kBlk = 256;
// levels up to this side length (L9) take the one-row-per-thread residual
// and transfer kernels: latency, not bandwidth, sets their time
constexpr int kSmallN1 = 513;

dim3 p1_interior_grid(int n1) {
    const int m = n1 - 2 * kRing;
    return dim3((m + kTX - 1) / kTX, (m + kTY * kRPT - 1) / (kTY * kRPT));
}

// rows [ylo, yhi) of a structured level (a rank's strip); the whole level
// by default
void level_residual(const ocmg_level *lv, const double *x, const double *f,
                    double *r, cudaStream_t s, int ylo = 0, int yhi = -1) {
    if (lv->kind == kP1) {
        if (yhi < 0) yhi = lv->n1;
        if (lv->n1 <= kSmallN1 && ylo == 0 && yhi == lv->n1) {
            const int64_t N = (int64_t)lv->n1 * lv->n1;
            OCMG_LAUNCH_PDL(k_p1_residual_all, grid_for(N, kBlk), kBlk, 0, s, lv->n1,
                        lv->tables.p, x, f, r);
            OCMG_LAUNCH_CHECK();
            return;
        }
        const int rlo = std::max(kRing, ylo), rhi = std::min(lv->n1 - kRing, yhi);
        const int m = lv->n1 - 2 * kRing;
        if (rhi > rlo) {
            const dim3 g((m + kTX - 1) / kTX, (rhi - rlo + kTY * kRPT - 1) / (kTY * kRPT));
            OCMG_LAUNCH(k_p1_residual_int, g, dim3(kTX, kTY), 0, s, lv->n1, lv->cA, x, f,
                        r, ylo, yhi);
        }
        OCMG_LAUNCH(k_p1_residual_ring, grid_for(p1_ring_count(lv->n1, kRing), kBlk),
                    kBlk, 0, s, lv->n1, lv->tables.p, x, f, r, ylo, yhi);
    } else {
        const SellDev &S = lv->sell;
        OCMG_LAUNCH(k_sell_residual, grid_for(lv->n, kBlk), kBlk, 0, s, lv->n, S.base.p,
                    S.len.p, S.col.p, S.val.p, x, f, r);
    }
    OCMG_LAUNCH_CHECK();
}

// the two halves of an NE-Jacobi sweep on a structured level, for the rows
// [ylo, yhi) (a strip: p of rows ylo..yhi needs r of rows ylo-1..yhi, the
// apply half p of rows ylo-1..yhi)
void p1_ne_p_half(const ocmg_level *lv, double tau, const double *r, double *p,
                  cudaStream_t s, int ylo, int yhi) {
    const dim3 g = p1_interior_grid(lv->n1), b(kTX, kTY);
    P1JacCoef C;
    for (int t = 0; t < 28; ++t) C.w[t] = lv->cW.c[t];
    C.l[0] = lv->cL[0];
    C.l[1] = lv->cL[1];
    C.tau = tau;
    OCMG_LAUNCH(k_p1_ne_p_int, g, b, 0, s, lv->n1, C, r, p, ylo, yhi);
    OCMG_LAUNCH(k_p1_ne_p_ring, grid_for(p1_ring_count(lv->n1, kRing), kBlk), kBlk, 0, s,
                lv->n1, lv->tables.p, tau, r, p, ylo, yhi);
}
void p1_ne_apply_half(const ocmg_level *lv, const double *p, double *x, double *r,
                      cudaStream_t s, int ylo, int yhi) {
    const dim3 g = p1_interior_grid(lv->n1), b(kTX, kTY);
    const dim3 ga(g.x, (lv->n1 - 2 * kRing + kTY * (kRPT / 2) - 1) / (kTY * (kRPT / 2)));
    OCMG_LAUNCH(k_p1_ne_apply_int, ga, b, 0, s, lv->n1, lv->cA, p, x, r, ylo, yhi);
    OCMG_LAUNCH(k_p1_ne_apply_ring, grid_for(p1_ring_count(lv->n1, kRing), kBlk), kBlk, 0,
                s, lv->n1, lv->tables.p, p, x, r, ylo, yhi);
}

void level_ne_jacobi(const ocmg_level *lv, double tau, double *x, double *r,
                     double *scratch, cudaStream_t s) {
    if (lv->kind == kP1) {
        p1_ne_p_half(lv, tau, r, scratch, s, 0, lv->n1);
        p1_ne_apply_half(lv, scratch, x, r, s, 0, lv->n1);
    } else {
        const SellDev &S = lv->sell;
        OCMG_LAUNCH(k_sell_ne_p, grid_for(lv->n, kBlk), kBlk, 0, s, lv->n, S.base.p,
                    S.len.p, S.col.p, S.w.p, lv->L.p, tau, r, scratch);
        OCMG_LAUNCH(k_sell_ne_apply, grid_for(lv->n, kBlk), kBlk, 0, s, lv->n, S.base.p,
                    S.len.p, S.col.p, S.val.p, scratch, x, r);
    }
    OCMG_LAUNCH_CHECK();
}

void run_schedule(const ocmg_level *lv, const Schedule &S, bool reverse,
                  double *x, double *r, cudaStream_t s, bool warp_rows = false) {
    const int64_t nb = (int64_t)S.off.size() - 1;
    if (lv->n <= kCsrSmallN) {
        // small level: every group in one CTA, __syncthreads between groups;
        // staged in shared memory when it fits
        const size_t sm = csr_small_smem(lv->n, lv->A.nnz, nb);
        if (warp_rows && lv->n <= kCsrWarpN && sm <= kCsrSmallSmemMax) {
            OCMG_LAUNCH(k_csr_gs_warp_small, 1, 32, sm, s, (int)nb, S.doff.p, S.rows.p,
                        reverse ? 1 : 0, (int)lv->n, lv->A.off.p, lv->A.col.p, lv->A.val.p,
                        lv->W.p, lv->ndiag.p, x, r);
            OCMG_LAUNCH_CHECK();
            return;
        }
        if (sm <= kCsrSmallSmemMax) {
            const int nt = lv->n < 1024 ? (int)(32 * ((lv->n + 31) / 32)) : 1024;
            OCMG_LAUNCH(k_csr_gs_sched_smem, 1, nt, sm, s, (int)nb, S.doff.p, S.rows.p,
                        reverse ? 1 : 0, (int)lv->n, lv->A.off.p, lv->A.col.p, lv->A.val.p,
                        lv->W.p, lv->ndiag.p, x, r);
            OCMG_LAUNCH_CHECK();
            return;
        }
        OCMG_LAUNCH(k_csr_gs_sched_small, 1, 1024, 0, s, (int)nb, S.doff.p,
                    S.rows.p, reverse ? 1 : 0, lv->A.off.p, lv->A.col.p, lv->A.val.p,
                    lv->W.p, lv->ndiag.p, x, r);
        OCMG_LAUNCH_CHECK();
        return;
    }
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t l = reverse ? nb - 1 - b : b;
        const int64_t lo = S.off[l], cnt = S.off[l + 1] - lo;
        if (!cnt) continue;
        if (warp_rows) {
            const int64_t thr = cnt * 32;
            const int blk = thr < 256 ? (int)thr : 256;
            OCMG_LAUNCH_PDL(k_csr_gs_rows_warp, grid_for(thr, blk), blk, 0, s, (int)cnt,
                            (const int32_t *)(S.rows.p + lo), (const int64_t *)lv->A.off.p,
                            (const int32_t *)lv->A.col.p, (const double *)lv->A.val.p,
                            (const double *)lv->W.p, (const double *)lv->ndiag.p, x, r);
        } else if (S.has_gsell) {
            const int64_t s0 = S.gslice[l], slots = (S.gslice[l + 1] - s0) * 32;
            const int blk = slots < 128 ? (int)slots : 128;
            OCMG_LAUNCH(k_gsell_gs_rows, grid_for(slots, blk), blk, 0, s, slots, s0,
                        S.gsrow.p, S.gsbase.p, S.gslen.p, S.gscol.p, S.gsval.p, S.gsw.p,
                        lv->ndiag.p, x, r);
        } else {
            const int blk = cnt < 128 ? 32 * (int)((cnt + 31) / 32) : 128;
            OCMG_LAUNCH(k_csr_gs_rows, grid_for(cnt, blk), blk, 0, s, (int)cnt,
                        S.rows.p + lo, lv->A.off.p, lv->A.col.p, lv->A.val.p, lv->W.p,
                        lv->ndiag.p, x, r);
        }
    }
    OCMG_LAUNCH_CHECK();
}

// One dependency level of the Vanka sweep (kernels.py:99-131), a warp per
// patch (<= 32 dofs, lane a = local dof a): gather r on the patch, the local
// inverse times it (b in order, separate multiply and add), the damped
// update, x += s, then the downdates r_j -= A_jc s_c dof by dof (lanes over
// the entries of column c = row c; rows of one column are distinct), so
// every r_j receives its terms in the reference's order.  Patches of one
// level share no row.
__global__ void k_vanka_level(int cnt, const int32_t *__restrict__ ids,
                              const int64_t *__restrict__ poff,
                              const int32_t *__restrict__ dofs,
                              const double *__restrict__ inv, int mmax,
                              const int64_t *__restrict__ aoff,
                              const int32_t *__restrict__ acol,
                              const double *__restrict__ aval, double tau,
                              double *__restrict__ x, double *__restrict__ r) {
    pdl_trigger();  // launched with PDL in the per-level loops
    pdl_wait();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= cnt) return;
    const int p = ids[w];
    const int64_t lo = poff[p];
    const int m = (int)(poff[p + 1] - lo);
    const int c = lane < m ? dofs[lo + lane] : 0;
    const double lr = lane < m ? r[c] : 0.0;
    const double *ip = inv + ((int64_t)p * mmax + lane) * mmax;
    double acc = 0.0;
    for (int b = 0; b < m; ++b) {
        const double lb = __shfl_sync(0xffffffffu, lr, b);
        if (lane < m) acc = __dadd_rn(acc, __dmul_rn(ip[b], lb));
    }
    const double s = __dmul_rn(tau, acc);
    if (lane < m) x[c] = __dadd_rn(x[c], s);
    for (int a = 0; a < m; ++a) {
        const double sa = __shfl_sync(0xffffffffu, s, a);
        const int ca = __shfl_sync(0xffffffffu, c, a);
        for (int64_t t = aoff[ca] + lane; t < aoff[ca + 1]; t += 32) {
            const int j = acol[t];
            r[j] = __dsub_rn(r[j], __dmul_rn(aval[t], sa));
        }
        __syncwarp();
    }
}

void level_vanka(const ocmg_level *lv, double tau, bool forward, double *x, double *r,
                 cudaStream_t s) {
    OCMG_REQUIRE(lv->vk_np > 0, "no Vanka patches on this level (ocmg_level_set_vanka)");
    const Schedule &S = lv->vk_sched;
    const int64_t nb = (int64_t)S.off.size() - 1;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t l = forward ? b : nb - 1 - b;
        const int64_t lo = S.off[l], cnt = S.off[l + 1] - lo;
        if (!cnt) continue;
        const int64_t thr = cnt * 32;
        const int blk = thr < 128 ? (int)thr : 128;
        OCMG_LAUNCH_PDL(k_vanka_level, grid_for(thr, blk), blk, 0, s, (int)cnt, S.rows.p + lo,
                    lv->vk_off.p, lv->vk_dofs.p, lv->vk_inv.p, lv->vk_mmax, lv->A.off.p,
                    lv->A.col.p, lv->A.val.p, tau, x, r);
    }
    OCMG_LAUNCH_CHECK();
}

// one multicolour sweep.  Tiers 0/1 update r in place (returns false);
// tier 2 reads r and writes the new residual to rout (returns true).
bool p1_mc_sweep(const ocmg_level *lv, bool forward, double *x, double *r,
                 double *rout, cudaStream_t s) {
    if (lv->mc_tier == 0) {
        OCMG_LAUNCH_PDL(k_p1_mc_small, 1, 1024, mc_small_smem(lv->n1), s, lv->n1,
                    forward ? 1 : 0, lv->mc_coef.p, x, r);
        OCMG_LAUNCH_CHECK();
        return false;
    }
    if (lv->mc_tier == 1) {
        int n1 = lv->n1, fw = forward ? 1 : 0;
        const double *T = lv->tables.p;
        unsigned *bar = lv->mc_bar.p;
        void *args[] = {&n1, &fw, &T, &x, &r, &bar};
        launch_counter().fetch_add(1, std::memory_order_relaxed);
        OCMG_CUDA(cudaLaunchCooperativeKernel((const void *)k_p1_mc_grid,
                                              dim3(lv->mc_grid), dim3(256), args, 0, s));
        return false;
    }
    McsParams P{};
    P.n1 = lv->n1;
    P.nstrips = lv->mc.nstrips;
    P.base = lv->mc.base;
    P.rem = lv->mc.rem;
    P.forward = forward ? 1 : 0;
    P.y_begin = 0;
    P.y_end = lv->n1;
    P.fs_in = P.fs_out = P.fs_x = (int64_t)lv->n1 * lv->n1;
    std::copy(lv->mc_cu, lv->mc_cu + mcs::NU, P.cu);
    P.C = lv->mc_coef.p;
    P.rin = r;
    P.rout = rout;
    P.x = x;
    mc_launch(P, lv->mc.grid, s);
    OCMG_LAUNCH_CHECK();
    return true;
}

void level_ne_gs(const ocmg_level *lv, int mode, bool forward, double *x,
                 double *r, cudaStream_t s) {
    OCMG_REQUIRE(mode >= OCMG_GS_REFERENCE && mode <= OCMG_GS_MULTICOLOUR,
                 "unknown NE-GS mode");
    if (lv->kind == kP1) {
        const int n1 = lv->n1;
        if (mode == OCMG_GS_MULTICOLOUR) {
            if (p1_mc_sweep(lv, forward, x, r, lv->mc_r.p, s))
                OCMG_CUDA(cudaMemcpyAsync(r, lv->mc_r.p, sizeof(double) * lv->n,
                                          cudaMemcpyDeviceToDevice, s));
        } else if (mode == OCMG_GS_WAVEFRONT && lv->has_pmap) {
            // k <= 5: d = S r, then x += d, r -= A d
            const int n = (int)lv->n;
            OCMG_LAUNCH(k_dense_rows, (n + kDenseRowsWarps - 1) / kDenseRowsWarps,
                        32 * kDenseRowsWarps, 0, s, n, n, lv->pmap[forward ? 0 : 1].p, r,
                        lv->pmap_d.p);
            OCMG_LAUNCH(k_p1_dense_finish, grid_for(n / 2, 128), 128, 0, s, n1, lv->tables.p,
                        lv->pmap_d.p, x, r);
        } else if (n1 <= kGsSmallMaxN1 && ((uintptr_t)x % 16 | (uintptr_t)r % 16) == 0) {
            // both exact modes: one CTA, levels separated by barriers
            const int nt = 64 * ((n1 + 1) / 2 > 32 ? 2 : 1);
            if (mode == OCMG_GS_WAVEFRONT)
                OCMG_LAUNCH(k_p1_gs_small<true>, 1, nt, gs_small_smem(n1), s, n1, lv->tables.p,
                            forward ? 1 : 0, x, r, (int64_t)0);
            else
                OCMG_LAUNCH(k_p1_gs_small<false>, 1, nt, gs_small_smem(n1), s, n1, lv->tables.p,
                            forward ? 1 : 0, x, r, (int64_t)0);
        } else if (n1 >= gsd::kMinN1 && n1 <= gsd::kMaxN1 &&
                   !(mode == OCMG_GS_WAVEFRONT && lv->wf.ready())) {
            // (the wavefront mode takes the band kernel from L7 up: 5-9
            // bands run a sweep in ~0.1-0.2 ms against the one-CTA ring's
            // 0.23-0.57 ms; the reference mode keeps the bitwise ring)
            // both exact modes: one CTA, anti-diagonal ring of r
            const int nt = 2 * gsd::per_field(n1);
            const size_t sm = gsd::smem(n1);
            const bool fast = mode == OCMG_GS_WAVEFRONT;
            if (forward && fast)
                OCMG_LAUNCH((k_p1_gs_diag<320, gsd::kRing, false, true>), 1, nt, sm, s, n1, lv->tables.p, x, r);
            else if (forward)
                OCMG_LAUNCH((k_p1_gs_diag<320, gsd::kRing, false, false>), 1, nt, sm, s, n1, lv->tables.p, x, r);
            else if (fast)
                OCMG_LAUNCH((k_p1_gs_diag<320, gsd::kRing, true, true>), 1, nt, sm, s, n1, lv->tables.p, x, r);
            else
                OCMG_LAUNCH((k_p1_gs_diag<320, gsd::kRing, true, false>), 1, nt, sm, s, n1, lv->tables.p, x, r);
        } else if (mode == OCMG_GS_WAVEFRONT && lv->wf.ready()) {
            lv->wf.sweep(forward, x, r, s);
        } else {
            const int depth = 3 * (n1 - 1) + 8;
            const int blk = 2 * n1 < 256 ? 32 * ((2 * n1 + 31) / 32) : 256;
            for (int t = 0; t < depth; ++t)
                OCMG_LAUNCH_PDL(k_p1_gs_level, grid_for(2 * n1, blk), blk, 0, s, 
                    n1, lv->tables.p, t, forward ? 1 : 0, x, r);
        }
        OCMG_LAUNCH_CHECK();
        return;
    }
    if (mode != OCMG_GS_REFERENCE && lv->has_dense &&
        (mode == OCMG_GS_WAVEFRONT || lv->has_colours)) {
        // tiny level: the sweep as its dense map (k_dense_sweep)
        const DevBuf<double> &D = lv->dense[mode == OCMG_GS_MULTICOLOUR][forward ? 0 : 1];
        const int n = (int)lv->n;
        OCMG_LAUNCH(k_dense_sweep, 1, n < 256 ? (int)(32 * ((n + 31) / 32)) : 256, 0, s, n,
                    D.p, D.p + (int64_t)n * n, x, r);
        OCMG_LAUNCH_CHECK();
        return;
    }
    if (mode == OCMG_GS_MULTICOLOUR) {
        OCMG_REQUIRE(lv->has_colours,
                     "multicolour NE-GS needs a level created with colouring");
        run_schedule(lv, lv->colours, !forward, x, r, s);
    } else {
        // wavefront mode: reference order, warp per row (FMA; 1e-12);
        // reference mode: thread per row, the reference's arithmetic
        run_schedule(lv, lv->sched[forward ? 0 : 1], false, x, r, s,
                     mode == OCMG_GS_WAVEFRONT);
    }
}

// debug: force the six-launch 3-colour CGS form (ocmg__debug_cgs_six_launch)
bool g_cgs_six_launch = false;

// one CGS sweep (kernels.py:70-96): mode OCMG_GS_MULTICOLOUR = 3 colours,
// otherwise the reference order (anti-diagonal levels); scratch: n doubles
void level_cgs(const ocmg_level *lv, int mode, double *x, double *r, double *scratch,
               cudaStream_t s) {
    OCMG_REQUIRE(lv->problem == OCMG_POISSON,
                 "collective sweep needs a scalar control system");
    OCMG_REQUIRE(lv->alpha > 0.0, "level has no control weight (ocmg_level_set_alpha)");
    if (lv->kind != kP1) {
        OCMG_LAUNCH(k_csr_cgs_seq, 1, 32, 0, s, lv->n / 2, lv->A.off.p, lv->A.col.p,
                    lv->A.val.p, lv->alpha, x, r);
        OCMG_LAUNCH_CHECK();
        return;
    }
    const int n1 = lv->n1;
    const int64_t N = (int64_t)n1 * n1;
    if (mode == OCMG_GS_MULTICOLOUR && lv->mc_tier == 2 && !g_cgs_six_launch) {
        // one launch, residual out of place through the level's mc_r
        CgsmParams P{};
        P.n1 = n1;
        P.nstrips = lv->cgsm.nstrips;
        P.base = lv->cgsm.base;
        P.rem = lv->cgsm.rem;
        P.alpha = lv->alpha;
        std::copy(&lv->cgs_mk[0][0], &lv->cgs_mk[0][0] + 49 * 4, &P.mk[0][0]);
        std::copy(lv->cgs_a24, lv->cgs_a24 + 28, P.a24);
        P.T = lv->tables.p;
        P.rin = r;
        P.rout = lv->mc_r.p;
        P.x = x;
        OCMG_LAUNCH(k_p1_cgs_mc_sweep, lv->cgsm.grid, cgsm::NT, cgsm::SMEM, s, P);
        OCMG_CUDA(cudaMemcpyAsync(r, lv->mc_r.p, sizeof(double) * lv->n,
                                  cudaMemcpyDeviceToDevice, s));
    } else if (mode == OCMG_GS_MULTICOLOUR) {
        const int64_t per = (int64_t)((n1 + 2) / 3) * n1;
        for (int c = 0; c < 3; ++c) {
            OCMG_LAUNCH(k_p1_cgs_solve, grid_for(per, kBlk), kBlk, 0, s, n1, lv->tables.p,
                        lv->alpha, 3, c, x, r, scratch);
            OCMG_LAUNCH(k_p1_cgs_apply, grid_for(N, kBlk), kBlk, 0, s, n1, lv->tables.p,
                        3, c, scratch, r);
        }
    } else {
        const int blk = n1 < 256 ? 32 * ((n1 + 31) / 32) : 256;
        for (int l = 0; l <= 2 * (n1 - 1); ++l) {
            OCMG_LAUNCH_PDL(k_p1_cgs_solve, grid_for(n1, blk), blk, 0, s, n1, lv->tables.p,
                            lv->alpha, 0, l, x, r, scratch);
            OCMG_LAUNCH_PDL(k_p1_cgs_apply, grid_for(5 * (int64_t)n1, kBlk), kBlk, 0, s, n1,
                            lv->tables.p, 0, l, scratch, r);
        }
    }
    OCMG_LAUNCH_CHECK();
}

void level_mean_project(const ocmg_level *lv, double *x, cudaStream_t s) {
    if (lv->problem != OCMG_STOKES) return;
    const int nf = (int)lv->field_off.size() - 1;
    for (int f = 0; f < nf; ++f) {
        if (!((lv->pmask >> f) & 1u)) continue;
        const int64_t lo = lv->field_off[f], hi = lv->field_off[f + 1];
        OCMG_LAUNCH(k_sum_partial, kRedGrid, kRedBlock, 0, s, lo, hi, x, lv->partial.p);
        OCMG_LAUNCH(k_finish_sum, 1, kRedBlock, 0, s, kRedGrid, lv->partial.p,
                                             (double)(hi - lo), lv->scal.p + f);
        OCMG_LAUNCH(k_sub_scalar, grid_for(hi - lo, kBlk), kBlk, 0, s, lo, hi, x,
                                                              lv->scal.p + f);
    }
    OCMG_LAUNCH_CHECK();
}

void sumsq(int64_t n, const double *x, const double *w, double *partial,
           double *out, cudaStream_t s) {
    OCMG_LAUNCH(k_sumsq_partial, kRedGrid, kRedBlock, 0, s, n, x, w, partial);
    OCMG_LAUNCH(k_finish_sum, 1, kRedBlock, 0, s, kRedGrid, partial, 1.0, out);
    OCMG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// coarse solve: pivoted LU substitution in one CTA
// ---------------------------------------------------------------------------
__global__ void k_coarse_solve(int n, const double *__restrict__ lu,
                               const int32_t *__restrict__ piv, int stokes,
                               int p_off, int mu_off, int n_p,
                               const double *__restrict__ rhs,
                               double *__restrict__ xout) {
    extern __shared__ double b[];
    __shared__ double sh[32];
    __shared__ double mean[2];
    for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = rhs[i];
    __syncthreads();
    const int offs[2] = {p_off, mu_off};
    if (stokes) {  // project the rhs, pin (multigrid.py:95-99)
        for (int f = 0; f < 2; ++f) {
            double acc = 0.0;
            for (int i = threadIdx.x; i < n_p; i += blockDim.x)
                acc += b[offs[f] + i];
            acc = block_sum(acc, sh);
            if (threadIdx.x == 0) mean[f] = acc / (double)n_p;
            __syncthreads();
            for (int i = threadIdx.x; i < n_p; i += blockDim.x)
                b[offs[f] + i] -= mean[f];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            b[p_off] = 0.0;
            b[mu_off] = 0.0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)  // row interchanges (getrs / laswp)
        for (int i = 0; i < n; ++i) {
            const int p = piv[i];
            if (p != i) {
                const double t = b[i];
                b[i] = b[p];
                b[p] = t;
            }
        }
    __syncthreads();
    for (int j = 0; j < n; ++j) {  // unit lower solve, column oriented
        const double bj = b[j];
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
            b[i] -= lu[i + (int64_t)j * n] * bj;
        __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {  // upper solve
        if (threadIdx.x == 0) b[j] /= lu[j + (int64_t)j * n];
        __syncthreads();
        const double bj = b[j];
        for (int i = threadIdx.x; i < j; i += blockDim.x)
            b[i] -= lu[i + (int64_t)j * n] * bj;
        __syncthreads();
    }
    if (stokes) {  // re-centre (pressure_mean_projection)
        for (int f = 0; f < 2; ++f) {
            double acc = 0.0;
            for (int i = threadIdx.x; i < n_p; i += blockDim.x)
                acc += b[offs[f] + i];
            acc = block_sum(acc, sh);
            if (threadIdx.x == 0) mean[f] = acc / (double)n_p;
            __syncthreads();
            for (int i = threadIdx.x; i < n_p; i += blockDim.x)
                b[offs[f] + i] -= mean[f];
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = b[i];
}

// Coarse solve as x = A^-1 b (A^-1 formed once on the host from the same LU):
// one warp per row, the whole (projected) rhs in shared memory.  Used by the
// cycle driver, where the coarsest level is visited once per coarse-grid
// correction (2^(levels-1) times per W-cycle); replacing the triangular solves
// by an explicit inverse changes cycle iterates by <= 2e-16 (Poisson) /
// 6.2e-15 (Stokes) with identical cycle counts (SURVEY.md §8(a) CoarseSolver).
constexpr int64_t kCoarseInvMax = 1024;

__global__ void __launch_bounds__(256)
    k_coarse_inv(int n, const double *__restrict__ inv, int stokes, int p_off,
                 int mu_off, int n_p, const double *__restrict__ rhs,
                 double *__restrict__ xout) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    extern __shared__ double b[];
    __shared__ double sh[32];
    __shared__ double mean[2];
    for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = rhs[i];
    __syncthreads();
    if (stokes) {  // project the rhs, pin (multigrid.py:95-99)
        const int offs[2] = {p_off, mu_off};
        for (int f = 0; f < 2; ++f) {
            double acc = 0.0;
            for (int i = threadIdx.x; i < n_p; i += blockDim.x) acc += b[offs[f] + i];
            acc = block_sum(acc, sh);
            if (threadIdx.x == 0) mean[f] = acc / (double)n_p;
            __syncthreads();
            for (int i = threadIdx.x; i < n_p; i += blockDim.x) b[offs[f] + i] -= mean[f];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            b[p_off] = 0.0;
            b[mu_off] = 0.0;
        }
        __syncthreads();
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + warp;
    if (row >= n) return;
    const double *a = inv + (int64_t)row * n;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc = fma(__ldg(a + j), b[j], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) xout[row] = acc;
}

// Stokes: re-centre the pressure fields of the solution (one CTA)
__global__ void k_coarse_recentre(int p_off, int mu_off, int n_p,
                                  double *__restrict__ x) {
    __shared__ double sh[32];
    __shared__ double mean;
    const int offs[2] = {p_off, mu_off};
    for (int f = 0; f < 2; ++f) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < n_p; i += blockDim.x) acc += x[offs[f] + i];
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) mean = acc / (double)n_p;
        __syncthreads();
        for (int i = threadIdx.x; i < n_p; i += blockDim.x) x[offs[f] + i] -= mean;
        __syncthreads();
    }
}

void coarse_solve_inv(const ocmg_coarse *c, const double *rhs, double *x,
                      cudaStream_t s) {
    const int n = (int)c->n;
    const size_t smem = (size_t)n * sizeof(double);
    const bool stokes = c->problem == OCMG_STOKES;
    OCMG_LAUNCH_PDL(k_coarse_inv, (n + 7) / 8, 256, smem, s, n, c->inv.p, stokes ? 1 : 0,
                (int)c->p_off, (int)c->mu_off, (int)c->n_p, rhs, x);
    if (stokes)
        OCMG_LAUNCH(k_coarse_recentre, 1, 256, 0, s, (int)c->p_off, (int)c->mu_off,
                    (int)c->n_p, x);
    OCMG_LAUNCH_CHECK();
}

void coarse_solve(const ocmg_coarse *c, const double *rhs, double *x,
                  cudaStream_t s) {
    const size_t smem = (size_t)c->n * sizeof(double);
    OCMG_LAUNCH(k_coarse_solve, 1, 256, smem, s, 
        (int)c->n, c->lu.p, c->piv.p, c->problem == OCMG_STOKES ? 1 : 0,
        (int)c->p_off, (int)c->mu_off, (int)c->n_p, rhs, x);
    OCMG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// transfers
// ---------------------------------------------------------------------------
void do_restrict(const ocmg_transfer *t, const double *rf, double *rc,
                 cudaStream_t s, int cylo = 0, int cyhi = -1) {
    if (t->kind == kP1) {
        if (cyhi < 0) cyhi = t->nc1;
        const int m = t->nc1, rows = cyhi - cylo;
        if (rows <= 0) return;
        if (m <= kSmallN1) {  // small level: a coarse row per thread
            const dim3 g((m + kTX - 1) / kTX, (rows + kTY - 1) / kTY);
            OCMG_LAUNCH_PDL(k_p1_restrict_tiled<1>, g, dim3(kTX, kTY), 0, s, t->nc1,
                        t->n_fields, rf, rc, cylo, cyhi);
        } else {
            const dim3 g((m + kTX - 1) / kTX, (rows + kTY * kRPT - 1) / (kTY * kRPT));
            OCMG_LAUNCH_PDL(k_p1_restrict_tiled<kRPT>, g, dim3(kTX, kTY), 0, s, t->nc1,
                        t->n_fields, rf, rc, cylo, cyhi);
        }
    } else {
        OCMG_LAUNCH(k_csr_spmv, grid_for(t->nc, kBlk), kBlk, 0, s, 
            t->nc, t->R.off.p, t->R.col.p, t->R.val.p, rf, rc);
    }
    OCMG_LAUNCH_CHECK();
}

void do_prolong_add(const ocmg_transfer *t, const double *c, double *xf,
                    cudaStream_t s, int fylo = 0, int fyhi = -1) {
    if (t->kind == kP1) {
        const int nf1 = 2 * t->nc1 - 1;
        if (fyhi < 0) fyhi = nf1;
        const int crows = std::min(t->nc1, (fyhi + 1) >> 1) - (fylo >> 1);
        if (crows <= 0) return;
        const bool all = fylo == 0 && fyhi == nf1;
        if (nf1 <= kSmallN1 && all) {  // small level: a coarse row per thread
            const dim3 g((nf1 + kTX - 1) / kTX, (crows + kTY - 1) / kTY);
            OCMG_LAUNCH_PDL((k_p1_prolong_add_tiled<true, 1>), g, dim3(kTX, kTY), 0, s, t->nc1,
                        t->n_fields, c, xf, fylo, fyhi);
        } else {
            const dim3 g((nf1 + kTX - 1) / kTX, (crows + kTY * kPRPT - 1) / (kTY * kPRPT));
            if (all)
                OCMG_LAUNCH_PDL((k_p1_prolong_add_tiled<true, kPRPT>), g, dim3(kTX, kTY), 0, s,
                            t->nc1, t->n_fields, c, xf, fylo, fyhi);
            else
                OCMG_LAUNCH_PDL((k_p1_prolong_add_tiled<false, kPRPT>), g, dim3(kTX, kTY), 0, s,
                            t->nc1, t->n_fields, c, xf, fylo, fyhi);
        }
    } else {
        OCMG_LAUNCH(k_csr_spmv_add, grid_for(t->nf, kBlk), kBlk, 0, s, 
            t->nf, t->P.off.p, t->P.col.p, t->P.val.p, c, xf);
    }
    OCMG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// cycle driver (multigrid.py:130-159)
// ---------------------------------------------------------------------------
void smooth(ocmg_hierarchy *h, int hi, double *x, double *r, cudaStream_t s,
            bool post = false) {
    ocmg_level *lv = h->levels[hi - 1];
    const ocmg_cycle_config &c = h->cfg;
    switch (c.smoother) {
    case OCMG_SMOOTHER_VANKA:  // smoothers.py:240-244: backward when post
        level_vanka(lv, c.tau, !post, x, r, s);
        break;
    case OCMG_SMOOTHER_NORMAL:
        level_ne_jacobi(lv, c.tau, x, r, h->scratch[hi].p, s);
        break;
    case OCMG_SMOOTHER_LSGS:
        level_ne_gs(lv, c.gs_mode, true, x, r, s);
        break;
    case OCMG_SMOOTHER_CGS:
        level_cgs(lv, c.gs_mode, x, r, h->scratch[hi].p, s);
        break;
    default:
        level_ne_gs(lv, c.gs_mode, true, x, r, s);
        level_ne_gs(lv, c.gs_mode, false, x, r, s);
    }
}

// nu smoothing steps; multicolour sweeps on structured levels ping-pong the
// residual between r and the level scratch instead of copying it back
void smooth_n(ocmg_hierarchy *h, int hi, int nu, double *x, double *r,
              cudaStream_t s, bool post = false) {
    ocmg_level *lv = h->levels[hi - 1];
    const ocmg_cycle_config &c = h->cfg;
    if (!(lv->kind == kP1 && c.gs_mode == OCMG_GS_MULTICOLOUR &&
          (c.smoother == OCMG_SMOOTHER_LSGS || c.smoother == OCMG_SMOOTHER_SLSGS))) {
        for (int i = 0; i < nu; ++i) smooth(h, hi, x, r, s, post);
        return;
    }
    double *buf[2] = {r, h->scratch[hi].p};
    int cur = 0;
    for (int i = 0; i < nu; ++i) {
        const int nsw = c.smoother == OCMG_SMOOTHER_LSGS ? 1 : 2;
        for (int k = 0; k < nsw; ++k)
            if (p1_mc_sweep(lv, k == 0, x, buf[cur], buf[1 - cur], s)) cur = 1 - cur;
    }
    if (cur)
        OCMG_CUDA(cudaMemcpyAsync(r, buf[1], sizeof(double) * lv->n,
                                  cudaMemcpyDeviceToDevice, s));
}

void cycle_rec(ocmg_hierarchy *h, int hi, double *x, const double *rhs,
               cudaStream_t s);

// corr = the coarse correction of hierarchy index hi for the restricted
// residual crhs: rec visits of index hi - 1 from zero (multigrid.py:150-152),
// or, collapsed (setup_collapse), G crhs in one launch
void coarse_correction(ocmg_hierarchy *h, int hi, const double *crhs, double *corr,
                       cudaStream_t s) {
    const int64_t nc = h->corr[hi - 1].n;
    if (h->col_hi > 0 && hi - 1 == h->col_hi) {
        OCMG_LAUNCH(k_dense_rows, (unsigned)((nc + kDenseRowsWarps - 1) / kDenseRowsWarps),
                    32 * kDenseRowsWarps, 0, s, (int)nc, h->col_ld, h->col_p, crhs, corr);
        OCMG_LAUNCH_CHECK();
        return;
    }
    OCMG_CUDA(cudaMemsetAsync(corr, 0, nc * sizeof(double), s));
    // the exact coarse solve ignores its start vector, so the W-cycle's
    // second visit of level 0 would recompute the same vector: elided
    const int rec = (h->cfg.cycle_w && hi - 1 > 0) ? 2 : 1;
    for (int k = 0; k < rec; ++k) cycle_rec(h, hi - 1, corr, crhs, s);
}

void cycle_rec(ocmg_hierarchy *h, int hi, double *x, const double *rhs,
               cudaStream_t s) {
    if (h->sub_hi > 0 && hi == h->sub_hi) {
        SubcycleParams P = h->sub;
        P.x = x;
        P.rhs = rhs;
        OCMG_LAUNCH_PDL(k_p1_subcycle, 1, kSubThreads, h->sub_smem, s, P);
        OCMG_LAUNCH_CHECK();
        return;
    }
    if (hi == 0) {
        if (h->coarse->inv.p)
            coarse_solve_inv(h->coarse, rhs, x, s);
        else
            coarse_solve(h->coarse, rhs, x, s);
        return;
    }
    ocmg_level *lv = h->levels[hi - 1];
    ocmg_transfer *tr = h->transfers[hi - 1];
    double *r = h->r[hi].p;
    level_residual(lv, x, rhs, r, s);
    smooth_n(h, hi, h->cfg.nu_pre, x, r, s);
    double *crhs = h->crhs[hi - 1].p, *corr = h->corr[hi - 1].p;
    do_restrict(tr, r, crhs, s);
    coarse_correction(h, hi, crhs, corr, s);
    do_prolong_add(tr, corr, x, s);
    level_mean_project(lv, x, s);
    level_residual(lv, x, rhs, r, s);
    smooth_n(h, hi, h->cfg.nu_post, x, r, s, true);
}

// Collapse the coarse end of the cycle into one dense map.  Every smoother,
// transfer and the coarse solve are linear, so the coarse correction of
// hierarchy index c + 1 -- rec visits of index c from a zero start on the
// restricted residual b (multigrid.py:150-152) -- is corr = G_c b for a fixed
// matrix G_c.  Its columns are built by running exactly that device code on
// the unit vectors e_j, bottom up (G_c's own coarse correction uses G_{c-1}),
// and the deepest index with at most max_n unknowns below the finest level is
// kept.  In a W-cycle from L12 this replaces the 2^(12-k) visits of every
// level k <= 5 (~17K launches) by 64 map applications of 38 MB, L2-resident.
// Not in the reference mode (its contract is bit-identity with the
// reference's arithmetic); the other modes keep their 1e-12 contract.
constexpr int64_t kCollapseMaxN = 8450;  // Poisson L6 (571 MB map; L7 would
                                         // stream 8.9 GB per application)
constexpr int kCollapseClones = 32;      // concurrent columns (parallel build)

// X[j * ld + i] = (coarse correction of index c + 1 applied to e_j)_i
void collapse_columns(ocmg_hierarchy *h, int c, double *X, int ld) {
    const int64_t n = h->levels[c - 1]->n;
    const int rec = (h->cfg.cycle_w && c > 0) ? 2 : 1;
    const ocmg_level *lc = h->levels[c - 1];
    // concurrent columns need the visit of level c to touch no level-owned
    // scratch (the one-CTA sweeps of k = 6 and the hierarchy's own vectors;
    // the levels below are already collapsed into the owner's map)
    const bool par = c - 1 == h->col_hi && lc->kind == kP1 && lc->problem == OCMG_POISSON &&
                     !lc->has_pmap && lc->mc_tier == 0 && lc->n1 <= kGsSmallMaxN1 &&
                     n > 4 * kCollapseClones;
    if (!par) {
        cudaStream_t s = nullptr;
        double *crhs = h->crhs[c].p, *corr = h->corr[c].p;
        for (int64_t j = 0; j < n; ++j) {
            OCMG_LAUNCH(k_unit_vector, grid_for(n, kBlk), kBlk, 0, s, n, j, crhs);
            OCMG_CUDA(cudaMemsetAsync(corr, 0, n * sizeof(double), s));
            for (int k = 0; k < rec; ++k) cycle_rec(h, c, corr, crhs, s);
            OCMG_CUDA(cudaMemcpyAsync(X + j * ld, corr, n * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
        }
        OCMG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // K clones of the hierarchy's bottom (shared levels, own vectors), each
    // with a captured graph for "column idx[k]; idx[k] += K", replayed on its
    // own stream
    const int K = kCollapseClones;
    std::vector<int64_t> first(K);
    for (int k = 0; k < K; ++k) first[k] = k;
    DevBuf<int64_t> idx;
    idx.upload(first);
    std::vector<std::unique_ptr<ocmg_hierarchy>> cl(K);
    std::vector<cudaStream_t> st(K, nullptr);
    std::vector<cudaGraphExec_t> ge(K, nullptr);
    auto cleanup = [&]() {
        for (int k = 0; k < K; ++k) {
            if (ge[k]) cudaGraphExecDestroy(ge[k]);
            if (st[k]) cudaStreamDestroy(st[k]);
        }
    };
    try {
        OCMG_CUDA(cudaDeviceSynchronize());
        for (int k = 0; k < K; ++k) {
            auto q = std::make_unique<ocmg_hierarchy>();
            q->levels.assign(h->levels.begin(), h->levels.begin() + c);
            q->transfers.assign(h->transfers.begin(), h->transfers.begin() + c);
            q->coarse = h->coarse;
            q->cfg = h->cfg;
            q->r.resize(c + 1);
            q->scratch.resize(c + 1);
            q->crhs.resize(c + 1);
            q->corr.resize(c + 1);
            for (int i = 0; i <= c; ++i) {
                const int64_t ni = h->corr[i].n;
                q->crhs[i].alloc(ni);
                q->corr[i].alloc(ni);
                if (i >= 1) {
                    q->r[i].alloc(ni);
                    if (h->scratch[i].n) q->scratch[i].alloc(ni);
                }
            }
            q->col_hi = h->col_hi;
            q->col_ld = h->col_ld;
            q->col_p = h->col_p;
            OCMG_CUDA(cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking));
            cudaGraph_t g;
            OCMG_CUDA(cudaStreamBeginCapture(st[k], cudaStreamCaptureModeThreadLocal));
            try {
                OCMG_LAUNCH(k_unit_vector_at, grid_for(n, kBlk), kBlk, 0, st[k], n, idx.p + k,
                            q->crhs[c].p);
                OCMG_CUDA(cudaMemsetAsync(q->corr[c].p, 0, n * sizeof(double), st[k]));
                for (int r = 0; r < rec; ++r) cycle_rec(q.get(), c, q->corr[c].p, q->crhs[c].p, st[k]);
                OCMG_LAUNCH(k_store_column, grid_for(n, kBlk), kBlk, 0, st[k], n, ld, idx.p + k,
                            q->corr[c].p, X);
                OCMG_LAUNCH(k_index_advance, 1, 1, 0, st[k], idx.p + k, (int64_t)K);
            } catch (...) {
                cudaStreamEndCapture(st[k], &g);
                throw;
            }
            OCMG_CUDA(cudaStreamEndCapture(st[k], &g));
            OCMG_CUDA(cudaGraphInstantiate(&ge[k], g, 0));
            cudaGraphDestroy(g);
            cl[k] = std::move(q);
        }
        for (int64_t rep = 0; rep < (n + K - 1) / K; ++rep)
            for (int k = 0; k < K; ++k) OCMG_CUDA(cudaGraphLaunch(ge[k], st[k]));
        OCMG_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

void setup_collapse(ocmg_hierarchy *h, int64_t max_n) {
    h->col_hi = 0;
    h->col_map = DevBuf<double>();
    h->col_p = nullptr;
    h->col_max_n = max_n;
    h->graph_x = nullptr;  // recapture
    h->graph_f = nullptr;
    if (max_n <= 0 || h->cfg.gs_mode == OCMG_GS_REFERENCE) return;
    const int nl = (int)h->levels.size();
    int m = 0;
    for (int c = 1; c < nl; ++c) {  // c < nl: the finest level is never collapsed
        if (h->levels[c - 1]->n > max_n) break;
        m = c;
    }
    if (m < 1) return;
    const int saved_sub = h->sub_hi;
    h->sub_hi = 0;  // per-level path during the build (the fused block's
                    // single launch is slower than the smaller maps)
    try {
        for (int c = 1; c <= m; ++c) {
            const int64_t n = h->levels[c - 1]->n;
            const int ld = (int)(n + (n & 1));
            DevBuf<double> X, G;
            X.alloc(n * ld);
            G.alloc(n * ld);
            collapse_columns(h, c, X.p, ld);
            OCMG_LAUNCH(k_dense_transpose,
                        dim3((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32)), dim3(32, 8), 0,
                        nullptr, (int)n, ld, X.p, G.p);
            OCMG_LAUNCH_CHECK();
            OCMG_CUDA(cudaDeviceSynchronize());
            h->col_map = std::move(G);
            h->col_p = h->col_map.p;
            h->col_ld = ld;
            h->col_hi = c;
        }
    } catch (...) {
        h->sub_hi = saved_sub;
        throw;
    }
    h->sub_hi = saved_sub;
}

// Enable the fused coarse block when the bottom of the hierarchy is
// structured Poisson with multicolour NE-GS and an explicit coarse inverse.
void setup_subcycle(ocmg_hierarchy *h) {
    h->sub_hi = 0;
    const ocmg_cycle_config &c = h->cfg;
    if (c.gs_mode != OCMG_GS_MULTICOLOUR ||
        !(c.smoother == OCMG_SMOOTHER_LSGS || c.smoother == OCMG_SMOOTHER_SLSGS))
        return;
    if (!h->coarse->inv.p || h->coarse->problem != OCMG_POISSON) return;
    const ocmg_level *l0 = h->levels[0];
    // a generic bottom level: Poisson L2 (n1 = 5, too small for the 49
    // class tables) over the reference's default coarsest level L1
    auto csr_l2 = [](const ocmg_level *lv) {
        return lv->kind != kP1 && lv->problem == OCMG_POISSON && lv->n == 50 &&
               lv->has_colours && lv->A.nnz <= kSubCsrNnz &&
               (int64_t)lv->colours.off.size() <= kSubCsrRows && lv->n < kSubCsrRows;
    };
    if (l0->kind != kP1 && !csr_l2(l0)) return;
    const int nc1 = l0->kind == kP1 ? (1 << (l0->k - 1)) + 1 : 3;
    if (h->coarse->n != 2 * (int64_t)nc1 * nc1) return;
    int top = 0;  // last hierarchy index with a level k <= kSubMaxK
    for (int hi = 1; hi <= (int)h->levels.size(); ++hi) {
        const ocmg_level *lv = h->levels[hi - 1];
        const ocmg_transfer *t = h->transfers[hi - 1];
        const bool ok = lv->kind == kP1 ? lv->k <= kSubMaxK : (hi == 1 && csr_l2(lv));
        if (!ok || t->kind != kP1) break;
        top = hi;
    }
    if (top < 1 || top + 1 > kSubMaxK) return;
    SubcycleParams P{};
    P.nlev = top + 1;
    std::vector<unsigned short> ops;
    sub_ops(top, c.cycle_w, c.nu_pre, c.nu_post, c.smoother == OCMG_SMOOTHER_SLSGS, ops);
    if ((int)ops.size() > kSubMaxOps) return;
    P.nops = (int)ops.size();
    std::copy(ops.begin(), ops.end(), P.ops);
    P.lv[0].n1 = nc1;
    int n1s[kSubMaxK] = {nc1};
    for (int j = 1; j <= top; ++j) {
        const ocmg_level *lv = h->levels[j - 1];
        SubLevel &sl = P.lv[j];
        if (lv->kind == kP1) {
            sl.n1 = lv->n1;
            sl.T = lv->tables.p;
            sl.C = lv->mc_coef.p;
        } else {
            sl.n1 = 5;
            sl.csr = 1;
            sl.ngroups = (int)lv->colours.off.size() - 1;
            sl.off = lv->A.off.p;
            sl.col = lv->A.col.p;
            sl.val = lv->A.val.p;
            sl.w = lv->W.p;
            sl.nd = lv->ndiag.p;
            sl.goff = lv->colours.doff.p;
            sl.rows = lv->colours.rows.p;
            if (lv->has_dense) {  // the same dense maps as level_ne_gs
                sl.dense[0] = lv->dense[1][0].p;
                sl.dense[1] = lv->dense[1][1].p;
            }
        }
        n1s[j] = sl.n1;
    }
    P.inv = h->coarse->inv.p;
    const SubLayout L = sub_layout(P.nlev, n1s);
    const size_t smem = (size_t)L.total * sizeof(double);
    if (smem > 200 * 1024) return;
    // per call: the attribute is per device, and cheap to set
    OCMG_CUDA(cudaFuncSetAttribute(k_p1_subcycle, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    h->sub = P;
    h->sub_smem = smem;
    h->sub_hi = top;
}

// one cycle + projection + ||f - A x||^2 into h->scal[0]
void cycle_and_measure(ocmg_hierarchy *h, double *x, const double *f,
                       cudaStream_t s) {
    const int top = (int)h->levels.size();
    cycle_rec(h, top, x, f, s);
    ocmg_level *fine = h->levels.back();
    level_mean_project(fine, x, s);
    level_residual(fine, x, f, h->tmp.p, s);
    sumsq(fine->n, h->tmp.p, nullptr, fine->partial.p, h->scal.p, s);
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char *ocmg_last_error(void) { return g_last_error.c_str(); }
int ocmg_abi_version(void) { return 1; }

int ocmg_device_sm_count(int *out) {
    return guarded([&] {
        int dev = 0;
        OCMG_CUDA(cudaGetDevice(&dev));
        OCMG_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
    });
}

int ocmg_launch_count(int64_t *out) {
    return guarded([&] {
        OCMG_REQUIRE(out, "null argument");
        *out = launch_counter().load();
    });
}

int ocmg_level_create_csr(int problem, int64_t n, const int64_t *row_off,
                          const int64_t *col, const double *val,
                          const double *norm_diag, int n_fields,
                          const int64_t *field_off, uint32_t pressure_mask,
                          int want_colouring, ocmg_level **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && row_off && col && val && norm_diag,
                     "null argument");
        OCMG_REQUIRE(n > 0 && n < (int64_t)1 << 31, "bad level size");
        OCMG_REQUIRE(n_fields >= 1 && field_off && field_off[0] == 0 &&
                         field_off[n_fields] == n,
                     "field offsets do not cover the level");
        for (int64_t i = 0; i < n; ++i)
            OCMG_REQUIRE(norm_diag[i] > 0.0, "norm_diag must be positive");
        // symmetric (bitwise) operator: column i == row i
        {
            std::vector<int64_t> toff, tcol;
            std::vector<double> tval;
            csr_transpose(n, n, row_off, col, val, toff, tcol, tval);
            for (int64_t i = 0; i <= n; ++i)
                OCMG_REQUIRE(toff[i] == row_off[i], "operator is not symmetric");
            for (int64_t t = 0; t < row_off[n]; ++t)
                OCMG_REQUIRE(tcol[t] == col[t] && tval[t] == val[t],
                             "operator is not symmetric");
        }
        auto lv = std::make_unique<ocmg_level>();
        lv->problem = problem;
        lv->kind = kCsr;
        lv->n = n;
        lv->field_off.assign(field_off, field_off + n_fields + 1);
        lv->pmask = pressure_mask;
        upload_csr(lv->A, n, n, row_off, col, val);
        lv->nnz = lv->A.nnz;
        lv->L.upload(norm_diag, n);
        lv->W.alloc(lv->nnz);
        lv->ndiag.alloc(n);
        OCMG_LAUNCH(k_csr_row_scaled, grid_for(lv->nnz, kBlk), kBlk, 0, 0, 
            lv->nnz, lv->A.col.p, lv->A.val.p, lv->L.p, lv->W.p);
        OCMG_LAUNCH(k_csr_ndiag, grid_for(n, kBlk), kBlk, 0, 0, n, lv->A.off.p,
                    lv->A.val.p, lv->W.p, lv->ndiag.p);
        OCMG_LAUNCH_CHECK();
        // per call: the attribute is per device, and cheap to set
        OCMG_CUDA(cudaFuncSetAttribute(k_csr_gs_sched_smem,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kCsrSmallSmemMax));
        OCMG_CUDA(cudaFuncSetAttribute(k_csr_gs_warp_small,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kCsrSmallSmemMax));
        {   // SELL-32 copy of A and W
            SellDev &S = lv->sell;
            S.nslices = (n + 31) / 32;
            std::vector<int64_t> base(S.nslices + 1, 0);
            for (int64_t sl = 0; sl < S.nslices; ++sl) {
                int64_t wmax = 0;
                for (int64_t i = 32 * sl; i < std::min(n, 32 * sl + 32); ++i)
                    wmax = std::max(wmax, row_off[i + 1] - row_off[i]);
                base[sl + 1] = base[sl] + 32 * wmax;
            }
            const int64_t ent = base[S.nslices];
            S.base.upload(base);
            S.len.alloc(n);
            S.col.alloc(ent);
            S.val.alloc(ent);
            S.w.alloc(ent);
            OCMG_CUDA(cudaMemset(S.col.p, 0, ent * sizeof(int32_t)));
            OCMG_LAUNCH(k_sell_fill, grid_for(n, kBlk), kBlk, 0, 0, n, lv->A.off.p,
                        lv->A.col.p, lv->A.val.p, lv->W.p, S.base.p, S.len.p, S.col.p,
                        S.val.p, S.w.p);
            OCMG_LAUNCH_CHECK();
        }
        lv->sched[0] = build_schedule(n, row_off, col, true);
        lv->sched[1] = build_schedule(n, row_off, col, false);
        if (want_colouring) {
            lv->colours = build_colouring(n, row_off, col);
            lv->has_colours = true;
        }
        if (n > kCsrSmallN) {  // grouped SELL for the per-group launches
            build_group_sell(lv->sched[0], n, row_off, lv->A, lv->W.p);
            build_group_sell(lv->sched[1], n, row_off, lv->A, lv->W.p);
            if (want_colouring) build_group_sell(lv->colours, n, row_off, lv->A, lv->W.p);
        }
        if (n <= kDenseN) {
            // dense sweep maps (k_dense_sweep): columns from the sequential
            // sweep of each unit residual, exact order and colour order
            const size_t sm = csr_small_smem(n, lv->A.nnz, n + 1);
            if (sm <= kCsrSmallSmemMax) {
                OCMG_CUDA(cudaFuncSetAttribute(k_csr_gs_sched_smem,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kCsrSmallSmemMax));
                const int nt = (int)(32 * ((n + 31) / 32));
                for (int md = 0; md < 2; ++md) {
                    if (md == 1 && !want_colouring) continue;
                    for (int dir = 0; dir < 2; ++dir) {
                        const Schedule &S = md == 0 ? lv->sched[dir] : lv->colours;
                        const int reverse = md == 1 && dir == 1;
                        DevBuf<double> &D = lv->dense[md][dir];
                        D.alloc(2 * n * n);
                        OCMG_LAUNCH(k_dense_unit, grid_for(n * n, kBlk), kBlk, 0, 0, (int)n,
                                    D.p, D.p + n * n);
                        OCMG_LAUNCH(k_csr_gs_sched_smem, (unsigned)n, nt, sm, 0,
                                    (int)S.off.size() - 1, S.doff.p, S.rows.p, reverse,
                                    (int)n, lv->A.off.p, lv->A.col.p, lv->A.val.p, lv->W.p,
                                    lv->ndiag.p, D.p, D.p + n * n, n);
                        OCMG_LAUNCH_CHECK();
                    }
                }
                OCMG_CUDA(cudaDeviceSynchronize());
                lv->has_dense = true;
            }
        }
        lv->partial.alloc(kRedGrid);
        lv->scal.alloc(8);
        // n_diag > 0 check (smoothers.py:213-215)
        std::vector<double> nd(n);
        OCMG_CUDA(cudaMemcpy(nd.data(), lv->ndiag.p, n * sizeof(double),
                             cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i)
            OCMG_REQUIRE(nd[i] > 0.0, "operator has an empty row; the "
                                      "normal-equation diagonal degenerates");
        *out = lv.release();
    });
}

int ocmg_level_create_p1(int k, double alpha, const double *tables,
                         int64_t n_tables, ocmg_level **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && tables, "null argument");
        OCMG_REQUIRE(k >= 3 && k <= 14, "structured P1 levels need 3 <= k <= 14");
        OCMG_REQUIRE(n_tables == kP1TableDoubles + kWfTableDoubles,
                     "P1 table size mismatch");
        OCMG_REQUIRE(alpha > 0.0, "alpha must be positive");
        auto lv = std::make_unique<ocmg_level>();
        lv->problem = OCMG_POISSON;
        lv->kind = kP1;
        lv->k = k;
        lv->n1 = (1 << k) + 1;
        lv->alpha = alpha;
        const int64_t N = (int64_t)lv->n1 * lv->n1;
        lv->n = 2 * N;
        const int64_t pairs = 7 * N - 8 * (int64_t)lv->n1 + 2;
        lv->nnz = 4 * pairs;
        lv->field_off = {0, N, 2 * N};
        lv->tables.upload(tables, n_tables);
        for (int t = 0; t < 28; ++t) {
            lv->cA.c[t] = tables[kP1OffA + 24 * 28 + t];
            lv->cW.c[t] = tables[kP1OffW + 24 * 28 + t];
        }
        lv->cL[0] = tables[kP1OffL + 24 * 2];
        lv->cL[1] = tables[kP1OffL + 24 * 2 + 1];
        lv->wf.init(lv->k, lv->n1, lv->tables.p, lv->tables.p + kP1TableDoubles);
        {
            // per call: the attribute is per device, and cheap to set
            mcs_set_smem();
            mc2_set_smem();
            int dev = 0, sms = 148;
            OCMG_CUDA(cudaGetDevice(&dev));
            OCMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            lv->mc = mc_plan(lv->n1, sms);
            // per call: the attribute is per device, and cheap to set
            OCMG_CUDA(cudaFuncSetAttribute(k_p1_mc_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           mc_small_smem(kMcSmallMaxN1)));
            OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)gs_small_smem(kGsSmallMaxN1)));
            OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)gs_small_smem(kGsSmallMaxN1)));
            {
                const int gsm = (int)gsd::smem(gsd::kMaxN1);
                OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_diag<320, gsd::kRing, false, false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
                OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_diag<320, gsd::kRing, true, false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
                OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_diag<320, gsd::kRing, false, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
                OCMG_CUDA(cudaFuncSetAttribute(k_p1_gs_diag<320, gsd::kRing, true, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
            }
            if (lv->n1 <= kP1DenseMaxN1) {
                // dense exact-order maps: column j = the reference-order
                // sweep of unit residual j from x = 0 (one CTA per column)
                const int n = (int)lv->n;
                DevBuf<double> X, R;
                X.alloc((int64_t)n * n);
                R.alloc((int64_t)n * n);
                const int nt = 64 * ((lv->n1 + 1) / 2 > 32 ? 2 : 1);
                for (int dir = 0; dir < 2; ++dir) {
                    OCMG_LAUNCH(k_p1_dense_unit, grid_for((int64_t)n * n, kBlk), kBlk, 0, 0, n,
                                X.p, R.p);
                    OCMG_LAUNCH(k_p1_gs_small<false>, (unsigned)n, nt, gs_small_smem(lv->n1), 0,
                                lv->n1, lv->tables.p, dir == 0 ? 1 : 0, X.p, R.p, (int64_t)n);
                    lv->pmap[dir].alloc((int64_t)n * n);
                    OCMG_LAUNCH(k_dense_transpose, dim3((n + 31) / 32, (n + 31) / 32), dim3(32, 8),
                                0, 0, n, n, X.p, lv->pmap[dir].p);
                    OCMG_LAUNCH_CHECK();
                }
                OCMG_CUDA(cudaDeviceSynchronize());
                lv->pmap_d.alloc(n);
                lv->has_pmap = true;
            }
            lv->mc_tier = lv->n1 <= kMcSmallMaxN1 ? 0 : lv->n1 <= kMcGridMaxN1 ? 1 : 2;
            if (lv->mc_tier == 1) {
                int occ = 0;
                OCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p1_mc_grid,
                                                                        256, 0));
                const int64_t work = (int64_t)((lv->n1 + 6) / 7) * lv->n1;
                lv->mc_grid = (int)std::min<int64_t>((work + 255) / 256,
                                                     (int64_t)std::max(1, occ) * sms);
                lv->mc_bar.alloc(2);
                OCMG_CUDA(cudaMemset(lv->mc_bar.p, 0, 2 * sizeof(unsigned)));
            }
            if (lv->mc_tier == 2) lv->mc_r.alloc(lv->n);
            lv->cgsm = cgsm_plan(lv->n1, sms);
            for (int c = 0; c < 49; ++c) {  // kernels.py:85-88 operation order
                const double m = tables[kP1OffA + c * 28 + 3];
                const double k = tables[kP1OffA + c * 28 + 7 + 3];
                volatile double mm = -m * m;  // no contraction across these
                volatile double q = mm / alpha;
                volatile double kk = k * k;
                lv->cgs_mk[c][0] = m;
                lv->cgs_mk[c][1] = k;
                lv->cgs_mk[c][2] = -m / alpha;
                lv->cgs_mk[c][3] = q - kk;
            }
            std::copy(tables + kP1OffA + 24 * 28, tables + kP1OffA + 25 * 28, lv->cgs_a24);
            // per call: the attribute is per device, and cheap to set
            OCMG_CUDA(cudaFuncSetAttribute(k_p1_cgs_mc_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           cgsm::SMEM));
            std::vector<double> C(49 * 2 * 29);
            for (int c = 0; c < 49; ++c)
                for (int f = 0; f < 2; ++f) {
                    double *o = C.data() + (c * 2 + f) * 29;
                    for (int e = 0; e < 14; ++e) {
                        o[e] = tables[kP1OffW + c * 28 + f * 14 + e];
                        o[14 + e] = tables[kP1OffA + c * 28 + f * 14 + e];
                    }
                    o[28] = 1.0 / tables[kP1OffND + c * 2 + f];
                }
            lv->mc_coef.upload(C.data(), (int64_t)C.size());
            std::copy(C.data() + 24 * 58, C.data() + 25 * 58, lv->mc_ci);
            OCMG_REQUIRE(mcs_fill_cu(lv->mc_cu, lv->mc_ci),
                         "interior stencil row lacks the P1 mesh symmetry");
        }
        lv->partial.alloc(kRedGrid);
        lv->scal.alloc(8);
        *out = lv.release();
    });
}

int ocmg_level_set_alpha(ocmg_level *lv, double alpha) {
    return guarded([&] {
        OCMG_REQUIRE(lv, "null level");
        OCMG_REQUIRE(alpha > 0.0, "alpha must be positive");
        lv->alpha = alpha;
    });
}

int ocmg_level_set_vanka(ocmg_level *lv, int64_t n_patches, int mmax,
                         const int64_t *offsets, const int64_t *dofs,
                         const double *inverses) {
    return guarded([&] {
        OCMG_REQUIRE(lv && offsets && dofs && inverses, "null argument");
        OCMG_REQUIRE(lv->kind == kCsr, "Vanka patches need a generic (CSR) level");
        OCMG_REQUIRE(n_patches > 0 && mmax > 0 && mmax <= 32, "bad patch sizes");
        const int64_t nd = offsets[n_patches];
        std::vector<int32_t> d32(nd);
        for (int64_t i = 0; i < nd; ++i) {
            OCMG_REQUIRE(dofs[i] >= 0 && dofs[i] < lv->n, "patch dof out of range");
            d32[i] = (int32_t)dofs[i];
        }
        for (int64_t p = 0; p < n_patches; ++p)
            OCMG_REQUIRE(offsets[p + 1] - offsets[p] >= 1 &&
                             offsets[p + 1] - offsets[p] <= mmax,
                         "patch larger than mmax");
        // the operator's pattern (A symmetric: column c = row c)
        std::vector<int64_t> aoff(lv->n + 1);
        std::vector<int32_t> acol(lv->A.nnz);
        OCMG_CUDA(cudaMemcpy(aoff.data(), lv->A.off.p, aoff.size() * 8, cudaMemcpyDeviceToHost));
        OCMG_CUDA(cudaMemcpy(acol.data(), lv->A.col.p, acol.size() * 4, cudaMemcpyDeviceToHost));
        // ASAP levels in patch order: a patch touches its dofs (x, and the
        // r it gathers) and the rows of their columns (r downdates)
        std::vector<int32_t> last(lv->n, -1), lev(n_patches);
        int32_t maxlev = -1;
        for (int64_t p = 0; p < n_patches; ++p) {
            int32_t m = -1;
            for (int64_t i = offsets[p]; i < offsets[p + 1]; ++i) {
                const int32_t c = d32[i];
                m = std::max(m, last[c]);
                for (int64_t t = aoff[c]; t < aoff[c + 1]; ++t) m = std::max(m, last[acol[t]]);
            }
            lev[p] = m + 1;
            for (int64_t i = offsets[p]; i < offsets[p + 1]; ++i) {
                const int32_t c = d32[i];
                last[c] = m + 1;
                for (int64_t t = aoff[c]; t < aoff[c + 1]; ++t) last[acol[t]] = m + 1;
            }
            maxlev = std::max(maxlev, m + 1);
        }
        Schedule &S = lv->vk_sched;
        S.off.assign(maxlev + 2, 0);
        for (int64_t p = 0; p < n_patches; ++p) S.off[lev[p] + 1]++;
        for (size_t l = 1; l < S.off.size(); ++l) S.off[l] += S.off[l - 1];
        std::vector<int32_t> rows(n_patches);
        std::vector<int64_t> fill(S.off.begin(), S.off.end() - 1);
        for (int64_t p = 0; p < n_patches; ++p) rows[fill[lev[p]]++] = (int32_t)p;
        S.rows.upload(rows);
        S.doff.upload(S.off);
        lv->vk_off.upload(offsets, n_patches + 1);
        lv->vk_dofs.upload(d32);
        lv->vk_inv.upload(inverses, n_patches * (int64_t)mmax * mmax);
        lv->vk_np = n_patches;
        lv->vk_mmax = mmax;
        lv->vk_ops = 0;
        for (int64_t i = 0; i < nd; ++i) lv->vk_ops += aoff[d32[i] + 1] - aoff[d32[i]];
    });
}

int ocmg_vanka_sweep(const ocmg_level *lv, double tau, int forward, double *x,
                     double *r, void *stream, int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r, "null argument");
        OCMG_REQUIRE(tau > 0.0 && tau < 2.0, "damping parameter must lie in (0, 2)");
        level_vanka(lv, tau, forward != 0, x, r, as_stream(stream));
        if (ops) *ops = lv->vk_ops;
    });
}

int ocmg_level_destroy(ocmg_level *lv) {
    return guarded([&] { delete lv; });
}

int64_t ocmg_level_n(const ocmg_level *lv) { return lv ? lv->n : -1; }
int64_t ocmg_level_nnz(const ocmg_level *lv) { return lv ? lv->nnz : -1; }

int ocmg_residual(const ocmg_level *lv, const double *x, const double *f,
                  double *r, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r, "null argument");
        level_residual(lv, x, f, r, as_stream(stream));
    });
}

int ocmg_ne_jacobi_sweep(const ocmg_level *lv, double tau, double *x,
                         double *r, double *scratch, void *stream,
                         int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r && scratch, "null argument");
        OCMG_REQUIRE(tau > 0.0 && tau < 2.0, "damping parameter must lie in (0, 2)");
        level_ne_jacobi(lv, tau, x, r, scratch, as_stream(stream));
        if (ops) *ops = 2 * lv->nnz;
    });
}

int ocmg_ne_gs_sweep(const ocmg_level *lv, int mode, int forward, double *x,
                     double *r, void *stream, int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r, "null argument");
        level_ne_gs(lv, mode, forward != 0, x, r, as_stream(stream));
        if (ops) *ops = 2 * lv->nnz;
    });
}

int ocmg_ne_gs_sweep_into(const ocmg_level *lv, int mode, int forward, double *x,
                          double *r_in, double *r_out, void *stream, int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r_in && r_out, "null argument");
        OCMG_REQUIRE(r_in != r_out, "r_in and r_out must differ");
        cudaStream_t s = as_stream(stream);
        if (!(lv->kind == kP1 && mode == OCMG_GS_MULTICOLOUR &&
              p1_mc_sweep(lv, forward != 0, x, r_in, r_out, s))) {
            // in-place forms: sweep r_in, then hand it over
            if (!(lv->kind == kP1 && mode == OCMG_GS_MULTICOLOUR))
                level_ne_gs(lv, mode, forward != 0, x, r_in, s);
            OCMG_CUDA(cudaMemcpyAsync(r_out, r_in, sizeof(double) * lv->n,
                                      cudaMemcpyDeviceToDevice, s));
        }
        if (ops) *ops = 2 * lv->nnz;
    });
}

int ocmg_ne_gs_sweep_strip(const ocmg_level *lv, int forward, int y_begin,
                           int y_end, int slab_begin, int slab_end, double *x,
                           const double *r_in, double *r_out, void *stream,
                           int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r_in && r_out, "null argument");
        OCMG_REQUIRE(lv->kind == kP1, "strip sweeps need a structured P1 level");
        const int n1 = lv->n1;
        OCMG_REQUIRE(0 <= y_begin && y_begin < y_end && y_end <= n1,
                     "strip rows out of range");
        OCMG_REQUIRE(slab_begin <= std::max(0, y_begin - (mcs::H + 1)) &&
                         slab_end >= std::min(n1, y_end + mcs::H + 1) && slab_begin >= 0 &&
                         slab_end <= n1,
                     "slab must hold 15 ghost rows on each side of the strip");
        OCMG_REQUIRE(r_in != r_out, "r_in and r_out must differ");
        int dev = 0, sms = 148;
        OCMG_CUDA(cudaGetDevice(&dev));
        OCMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const McsPlan pl = mc_plan(n1, sms, y_end - y_begin);
        McsParams P{};
        P.n1 = n1;
        P.nstrips = pl.nstrips;
        P.base = pl.base;
        P.rem = pl.rem;
        P.forward = forward ? 1 : 0;
            P.y_begin = y_begin;
        P.y_end = y_end;
        P.fs_in = P.fs_out = P.fs_x = (int64_t)(slab_end - slab_begin) * n1;
        std::copy(lv->mc_cu, lv->mc_cu + mcs::NU, P.cu);
        P.C = lv->mc_coef.p;
        P.rin = r_in - (int64_t)slab_begin * n1;
        P.rout = r_out - (int64_t)slab_begin * n1;
        P.x = x - (int64_t)slab_begin * n1;
        mc_launch(P, pl.grid, as_stream(stream));
        OCMG_LAUNCH_CHECK();
        if (ops) *ops = 2 * lv->nnz * (int64_t)(y_end - y_begin) / n1;
    });
}

int ocmg_residual_rows(const ocmg_level *lv, const double *x, const double *f,
                       double *r, int y_begin, int y_end, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r, "null argument");
        OCMG_REQUIRE(lv->kind == kP1, "row ranges need a structured P1 level");
        OCMG_REQUIRE(0 <= y_begin && y_begin <= y_end && y_end <= lv->n1, "bad rows");
        level_residual(lv, x, f, r, as_stream(stream), y_begin, y_end);
    });
}

int ocmg_ne_jacobi_p_rows(const ocmg_level *lv, double tau, const double *r, double *p,
                          int y_begin, int y_end, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && r && p, "null argument");
        OCMG_REQUIRE(lv->kind == kP1, "row ranges need a structured P1 level");
        OCMG_REQUIRE(tau > 0.0 && tau < 2.0, "damping parameter must lie in (0, 2)");
        OCMG_REQUIRE(0 <= y_begin && y_begin <= y_end && y_end <= lv->n1, "bad rows");
        p1_ne_p_half(lv, tau, r, p, as_stream(stream), y_begin, y_end);
        OCMG_LAUNCH_CHECK();
    });
}

int ocmg_ne_jacobi_apply_rows(const ocmg_level *lv, const double *p, double *x, double *r,
                              int y_begin, int y_end, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && p && x && r, "null argument");
        OCMG_REQUIRE(lv->kind == kP1, "row ranges need a structured P1 level");
        OCMG_REQUIRE(0 <= y_begin && y_begin <= y_end && y_end <= lv->n1, "bad rows");
        p1_ne_apply_half(lv, p, x, r, as_stream(stream), y_begin, y_end);
        OCMG_LAUNCH_CHECK();
    });
}

int ocmg_restrict_rows(const ocmg_transfer *t, const double *rf, double *rc,
                       int cy_begin, int cy_end, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(t && rf && rc, "null argument");
        OCMG_REQUIRE(t->kind == kP1, "row ranges need a structured P1 transfer");
        OCMG_REQUIRE(0 <= cy_begin && cy_begin <= cy_end && cy_end <= t->nc1, "bad rows");
        do_restrict(t, rf, rc, as_stream(stream), cy_begin, cy_end);
    });
}

int ocmg_prolong_add_rows(const ocmg_transfer *t, const double *c, double *xf,
                          int fy_begin, int fy_end, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(t && c && xf, "null argument");
        OCMG_REQUIRE(t->kind == kP1, "row ranges need a structured P1 transfer");
        OCMG_REQUIRE(0 <= fy_begin && fy_begin <= fy_end && fy_end <= 2 * t->nc1 - 1,
                     "bad rows");
        do_prolong_add(t, c, xf, as_stream(stream), fy_begin, fy_end);
    });
}

int ocmg_cgs_sweep(const ocmg_level *lv, int mode, double *x, double *r,
                   double *scratch, void *stream, int64_t *ops) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && r && scratch, "null argument");
        OCMG_REQUIRE(mode >= OCMG_GS_REFERENCE && mode <= OCMG_GS_MULTICOLOUR,
                     "unknown sweep mode");
        level_cgs(lv, mode, x, r, scratch, as_stream(stream));
        if (ops) *ops = lv->nnz;
    });
}

int ocmg_mean_project(const ocmg_level *lv, double *x, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x, "null argument");
        level_mean_project(lv, x, as_stream(stream));
    });
}

int ocmg_norm2(const ocmg_level *lv, const double *x, int weighted,
               double *out_dev, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && x && out_dev, "null argument");
        cudaStream_t s = as_stream(stream);
        if (weighted && lv->kind == kP1) {
            OCMG_LAUNCH(k_p1_wsumsq_partial, kRedGrid, kRedBlock, 0, s, 
                lv->n1, lv->tables.p, x, lv->partial.p);
            OCMG_LAUNCH(k_finish_sum, 1, kRedBlock, 0, s, kRedGrid, lv->partial.p, 1.0,
                                                 out_dev);
            OCMG_LAUNCH_CHECK();
            return;
        }
        sumsq(lv->n, x, weighted ? lv->L.p : nullptr, lv->partial.p, out_dev,
              s);
    });
}

int ocmg_transfer_create_csr(int64_t nf, int64_t nc, const int64_t *row_off,
                             const int64_t *col, const double *val,
                             ocmg_transfer **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && row_off && col && val, "null argument");
        auto t = std::make_unique<ocmg_transfer>();
        t->kind = kCsr;
        t->nf = nf;
        t->nc = nc;
        upload_csr(t->P, nf, nc, row_off, col, val);
        std::vector<int64_t> toff, tcol;
        std::vector<double> tval;
        csr_transpose(nf, nc, row_off, col, val, toff, tcol, tval);
        upload_csr(t->R, nc, nf, toff.data(), tcol.data(), tval.data());
        *out = t.release();
    });
}

int ocmg_transfer_create_p1(int kc, int n_fields, ocmg_transfer **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && kc >= 0 && kc < 14 && n_fields >= 1,
                     "bad P1 transfer arguments");
        auto t = std::make_unique<ocmg_transfer>();
        t->kind = kP1;
        t->kc = kc;
        t->nc1 = (1 << kc) + 1;
        t->n_fields = n_fields;
        const int64_t nf1 = 2 * (int64_t)t->nc1 - 1;
        t->nc = (int64_t)n_fields * t->nc1 * t->nc1;
        t->nf = (int64_t)n_fields * nf1 * nf1;
        *out = t.release();
    });
}

int ocmg_transfer_destroy(ocmg_transfer *t) {
    return guarded([&] { delete t; });
}

int ocmg_restrict(const ocmg_transfer *t, const double *rf, double *rc,
                  void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(t && rf && rc, "null argument");
        do_restrict(t, rf, rc, as_stream(stream));
    });
}

int ocmg_prolong_add(const ocmg_transfer *t, const double *c, double *xf,
                     void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(t && c && xf, "null argument");
        do_prolong_add(t, c, xf, as_stream(stream));
    });
}

int ocmg_coarse_create(int problem, int64_t n, const double *lu,
                       const int64_t *piv, int64_t p_off, int64_t mu_off,
                       int64_t n_p, ocmg_coarse **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && lu && piv, "null argument");
        OCMG_REQUIRE(n > 0 && n <= 5000,
                     "coarsest system too large; raise coarsest_level");
        for (int64_t i = 0; i < n; ++i)
            if (lu[i + i * n] == 0.0)
                throw Error(OCMG_E_SINGULAR,
                            "exactly singular pivot in LU factorization");
        auto c = std::make_unique<ocmg_coarse>();
        c->problem = problem;
        c->n = n;
        c->p_off = p_off;
        c->mu_off = mu_off;
        c->n_p = n_p;
        c->lu.upload(lu, (size_t)(n * n));
        std::vector<int32_t> p32(n);
        for (int64_t i = 0; i < n; ++i) p32[i] = (int32_t)piv[i];
        c->piv.upload(p32);
        if (n <= kCoarseInvMax) {
            // A^-1 column by column with the same getrs steps as k_coarse_solve
            std::vector<double> inv((size_t)(n * n)), b((size_t)n);
            for (int64_t col = 0; col < n; ++col) {
                std::fill(b.begin(), b.end(), 0.0);
                b[col] = 1.0;
                for (int64_t i = 0; i < n; ++i)
                    if (piv[i] != i) std::swap(b[i], b[piv[i]]);
                for (int64_t j = 0; j < n; ++j)
                    for (int64_t i = j + 1; i < n; ++i) b[i] -= lu[i + j * n] * b[j];
                for (int64_t j = n - 1; j >= 0; --j) {
                    b[j] /= lu[j + j * n];
                    for (int64_t i = 0; i < j; ++i) b[i] -= lu[i + j * n] * b[j];
                }
                for (int64_t i = 0; i < n; ++i) inv[i * n + col] = b[i];  // row-major
            }
            c->inv.upload(inv);
        }
        *out = c.release();
    });
}

int ocmg_coarse_destroy(ocmg_coarse *c) {
    return guarded([&] { delete c; });
}

int ocmg_coarse_solve(const ocmg_coarse *c, const double *rhs, double *x,
                      void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(c && rhs && x, "null argument");
        coarse_solve(c, rhs, x, as_stream(stream));
    });
}

int ocmg_hierarchy_create(int n_levels, ocmg_level *const *levels,
                          ocmg_transfer *const *transfers, ocmg_coarse *coarse,
                          const ocmg_cycle_config *cfg, ocmg_hierarchy **out) {
    return guarded([&] {
        OCMG_REQUIRE(out && levels && transfers && coarse && cfg,
                     "null argument");
        OCMG_REQUIRE(n_levels >= 1, "need at least one smoothed level");
        OCMG_REQUIRE(cfg->smoother >= OCMG_SMOOTHER_NORMAL &&
                         cfg->smoother <= OCMG_SMOOTHER_VANKA,
                     "unknown smoother kind");
        if (cfg->smoother == OCMG_SMOOTHER_VANKA)
            for (int i = 0; i < n_levels; ++i)
                OCMG_REQUIRE(levels[i]->vk_np > 0 && cfg->tau > 0.0 && cfg->tau < 2.0,
                             "the patch smoother needs Vanka patches on every level "
                             "(ocmg_level_set_vanka) and a damping in (0, 2)");
        OCMG_REQUIRE(cfg->smoother != OCMG_SMOOTHER_CGS ||
                         levels[n_levels - 1]->problem == OCMG_POISSON,
                     "collective sweep needs a scalar control system");
        OCMG_REQUIRE(cfg->nu_pre + cfg->nu_post >= 1,
                     "need at least one smoothing step per cycle");
        auto h = std::make_unique<ocmg_hierarchy>();
        h->levels.assign(levels, levels + n_levels);
        h->transfers.assign(transfers, transfers + n_levels);
        h->coarse = coarse;
        h->cfg = *cfg;
        h->r.resize(n_levels + 1);
        h->scratch.resize(n_levels + 1);
        h->crhs.resize(n_levels);
        h->corr.resize(n_levels);
        std::vector<int64_t> sizes(n_levels + 1);
        sizes[0] = coarse->n;
        for (int i = 0; i < n_levels; ++i) sizes[i + 1] = levels[i]->n;
        for (int i = 0; i < n_levels; ++i) {
            OCMG_REQUIRE(transfers[i]->nc == sizes[i] &&
                             transfers[i]->nf == sizes[i + 1],
                         "transfer sizes do not match the levels");
        }
        for (int hi = 1; hi <= n_levels; ++hi) {
            h->r[hi].alloc(sizes[hi]);
            // NE-Jacobi update vector / multicolour ping-pong residual
            if (cfg->smoother == OCMG_SMOOTHER_NORMAL || cfg->smoother == OCMG_SMOOTHER_CGS ||
                cfg->gs_mode == OCMG_GS_MULTICOLOUR)
                h->scratch[hi].alloc(sizes[hi]);
        }
        for (int hi = 0; hi < n_levels; ++hi) {
            h->crhs[hi].alloc(sizes[hi]);
            h->corr[hi].alloc(sizes[hi]);
        }
        h->tmp.alloc(sizes[n_levels]);
        h->scal.alloc(8);
        setup_subcycle(h.get());
        setup_collapse(h.get(), kCollapseMaxN);
        *out = h.release();
    });
}

int ocmg_hierarchy_destroy(ocmg_hierarchy *h) {
    return guarded([&] { delete h; });
}

int ocmg_hierarchy_collapsed_level(const ocmg_hierarchy *h, int *level_index) {
    return guarded([&] {
        OCMG_REQUIRE(h && level_index, "null argument");
        *level_index = h->col_hi;
    });
}

int ocmg_coarse_correction(ocmg_hierarchy *h, int level_index, const double *crhs,
                           double *corr, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(h && crhs && corr, "null argument");
        OCMG_REQUIRE(level_index >= 1 && level_index <= (int)h->levels.size(),
                     "level index out of range");
        coarse_correction(h, level_index, crhs, corr, as_stream(stream));
    });
}

int ocmg_cycle(ocmg_hierarchy *h, double *x, const double *f, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(h && x && f, "null argument");
        cycle_rec(h, (int)h->levels.size(), x, f, as_stream(stream));
    });
}

int ocmg_solve(ocmg_hierarchy *h, double *x, const double *f, double tol,
               int max_cycles, int use_graph, double *hist, int *n_done,
               void *stream) {
    int diverged = 0;
    return ocmg_solve_ex(h, x, f, tol, max_cycles, use_graph, 1e6, hist,
                         n_done, &diverged, stream);
}

int ocmg_solve_ex(ocmg_hierarchy *h, double *x, const double *f, double tol,
                  int max_cycles, int use_graph, double divergence_factor,
                  double *hist, int *n_done, int *diverged, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(h && x && f && hist && n_done && diverged,
                     "null argument");
        *diverged = 0;
        cudaStream_t s = as_stream(stream);
        if (use_graph && s == nullptr) {
            // the legacy default stream cannot be captured: run the solve on
            // a private non-blocking stream ordered after the caller's work
            if (!h->own_stream) {
                OCMG_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
                OCMG_CUDA(cudaEventCreateWithFlags(&h->own_event, cudaEventDisableTiming));
            }
            OCMG_CUDA(cudaEventRecord(h->own_event, nullptr));
            OCMG_CUDA(cudaStreamWaitEvent(h->own_stream, h->own_event, 0));
            s = h->own_stream;
        }
        ocmg_level *fine = h->levels.back();
        // ||f||^2
        sumsq(fine->n, f, nullptr, fine->partial.p, h->scal.p + 1, s);
        double fn2 = 0.0;
        OCMG_CUDA(cudaMemcpyAsync(&fn2, h->scal.p + 1, sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
        OCMG_CUDA(cudaStreamSynchronize(s));
        const double fn = std::sqrt(fn2);
        OCMG_REQUIRE(fn > 0.0, "right-hand side is zero");
        // relative residual of the entering iterate: the divergence test's
        // norm0 (multigrid.py:26,198-200 abort once the norm exceeds
        // DIVERGENCE_FACTOR * norm0)
        level_residual(fine, x, f, h->tmp.p, s);
        sumsq(fine->n, h->tmp.p, nullptr, fine->partial.p, h->scal.p + 2, s);
        double r02 = 0.0;
        OCMG_CUDA(cudaMemcpyAsync(&r02, h->scal.p + 2, sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
        OCMG_CUDA(cudaStreamSynchronize(s));
        const double rel0 = std::sqrt(r02) / fn;
        const bool graphs = use_graph && s != nullptr;
        if (graphs && (h->graph_x != x || h->graph_f != f ||
                       h->graph_stream != s)) {
            if (h->graph) cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
            cudaGraph_t g;
            OCMG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                cycle_and_measure(h, x, f, s);
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                throw;
            }
            OCMG_CUDA(cudaStreamEndCapture(s, &g));
            OCMG_CUDA(cudaGraphInstantiate(&h->graph, g, 0));
            cudaGraphDestroy(g);
            h->graph_x = x;
            h->graph_f = f;
            h->graph_stream = s;
        }
        int done = 0;
        for (int c = 0; c < max_cycles; ++c) {
            if (graphs)
                OCMG_CUDA(cudaGraphLaunch(h->graph, s));
            else
                cycle_and_measure(h, x, f, s);
            double r2 = 0.0;
            OCMG_CUDA(cudaMemcpyAsync(&r2, h->scal.p, sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
            OCMG_CUDA(cudaStreamSynchronize(s));
            const double rel = std::sqrt(r2) / fn;
            hist[c] = rel;
            done = c + 1;
            if (rel <= tol) break;
            if (!std::isfinite(rel) ||
                (divergence_factor > 0.0 && rel > divergence_factor * rel0)) {
                *diverged = 1;
                break;
            }
        }
        *n_done = done;
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// internal debug hooks (not part of the ABI in include/ocmg_b200.h)
// ---------------------------------------------------------------------------

// internal: per-warp iteration timestamps of the last wavefront sweep
// (only when built with -DOCMG_WF_PROFILE); returns nb, niter, nwarps
extern "C" int ocmg__debug_wf_prof(const ocmg_level *lv, unsigned long long *out,
                                   int64_t *dims) {
    return guarded([&] {
        OCMG_REQUIRE(lv && lv->kind == kP1 && lv->wf.ready(), "no wavefront");
        dims[0] = lv->wf.nb;
        dims[1] = lv->wf.niter();
        dims[2] = wf::NWARPS;
        dims[3] = (int64_t)lv->wf.prof.n;
        if (out && lv->wf.prof.n)
            OCMG_CUDA(cudaMemcpy(out, lv->wf.prof.p,
                                 lv->wf.prof.n * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost));
    });
}

// internal: the multicolour sweep as 7 colour passes (one launch per
// colour, in place) -- the reference form the one-launch kernel must match
extern "C" int ocmg__debug_mc_passes(const ocmg_level *lv, int forward, double *x,
                                     double *r, void *stream) {
    return guarded([&] {
        OCMG_REQUIRE(lv && lv->kind == kP1 && x && r, "structured P1 level only");
        const int n1 = lv->n1;
        const int64_t work = (int64_t)((n1 + 6) / 7) * n1;
        cudaStream_t s = as_stream(stream);
        for (int b = 0; b < kMcColours; ++b) {
            const int c = forward ? b : kMcColours - 1 - b;
            OCMG_LAUNCH(k_p1_gs_colour, grid_for(work, kBlk), kBlk, 0, s, n1,
                        lv->tables.p, c, forward ? 1 : 0, x, r);
        }
        OCMG_LAUNCH_CHECK();
    });
}

#ifdef MC2_PROF
extern "C" int ocmg__debug_mc2_prof(unsigned long long *out, int n) {
    return guarded([&] {
        OCMG_CUDA(cudaMemcpyFromSymbol(out, mc2_prof, sizeof(unsigned long long) * n));
    });
}
#endif

// internal: switch the fused coarse block of a hierarchy off (0) or back on
// (1), so tests can compare the fused and per-level cycles
extern "C" int ocmg__debug_hierarchy_fuse(ocmg_hierarchy *h, int on) {
    return guarded([&] {
        OCMG_REQUIRE(h, "null hierarchy");
        if (on)
            setup_subcycle(h);
        else
            h->sub_hi = 0;
        h->graph_x = nullptr;  // recapture
        h->graph_f = nullptr;
    });
}

// internal: collapse the coarse end of a hierarchy's cycle for levels of at
// most max_n unknowns (0: off), so tests can compare both cycles
extern "C" int ocmg__debug_hierarchy_collapse(ocmg_hierarchy *h, int64_t max_n, int *col_hi) {
    return guarded([&] {
        OCMG_REQUIRE(h, "null hierarchy");
        setup_collapse(h, max_n < 0 ? kCollapseMaxN : max_n);
        if (col_hi) *col_hi = h->col_hi;
    });
}

// internal: one launch of a hierarchy's fused coarse block on (x, rhs), with
// per-op timestamps into prof (device, nops + 1 entries); returns nops
extern "C" int ocmg__debug_subcycle_prof(ocmg_hierarchy *h, double *x, const double *rhs,
                                         unsigned long long *prof, int *nops) {
    return guarded([&] {
        OCMG_REQUIRE(h && h->sub_hi > 0, "no fused block");
        SubcycleParams P = h->sub;
        P.x = x;
        P.rhs = rhs;
        P.prof = prof;
        *nops = P.nops;
        OCMG_LAUNCH(k_p1_subcycle, 1, kSubThreads, h->sub_smem, nullptr, P);
        OCMG_LAUNCH_CHECK();
        OCMG_CUDA(cudaDeviceSynchronize());
    });
}

// internal: 1 = multicolour CGS sweeps use the six-launch form on every level
// (the reference the one-launch kernel must match), 0 = normal dispatch
extern "C" int ocmg__debug_cgs_six_launch(int on) {
    return guarded([&] { g_cgs_six_launch = on != 0; });
}
