// The coarse end of a multigrid cycle in ONE launch (structured Poisson,
// multicolour NE-GS; below the structured levels possibly the generic CSR
// level L2 over the coarsest L1): a visit of level kt (<= 5) runs the whole recursion
// below it -- residual, pre-smoothing, restriction, the coarser visits
// (twice for W), the coarse solve, prolongation, residual, post-smoothing --
// in one CTA with every vector in shared memory.
//
// Why: a W-cycle visits level l 2^(L-l) times, so the coarse levels are
// thousands of tiny launches per cycle (launch-latency bound; at L12 they were
// ~75 of ~85 ms per W-cycle).  Here a visit of level 5 costs one launch.
//
// Every operation repeats the arithmetic of the per-level kernels it replaces
// (k_p1_residual_int/ring, k_p1_mc_small, k_p1_restrict_tiled,
// k_p1_prolong_add_tiled, k_coarse_inv), so a cycle with the fused block is
// bit-identical to one without it (tests/test_gpu_parity.py).
#pragma once

#include "ocmg_p1_mc.cuh"

namespace ocmg {

constexpr int kSubMaxK = 5;        // top level of the fused block
constexpr int kSubThreads = 256;

struct SubLevel {
    int n1;
    const double *T;  // class tables (ocmg_p1.cuh layout)
    const double *C;  // multicolour table [49][2][29]
    // generic (CSR) Poisson level below the structured ones (L2 when the
    // coarsest level is the reference default L1): its operator, row_scaled,
    // n_diag and multicolour groups, the arithmetic of k_csr_residual and
    // k_csr_gs_sched_small
    int csr, ngroups;
    const int64_t *off, *goff;
    const int32_t *col, *rows;
    const double *val, *w, *nd;
    const double *dense[2];  // multicolour sweep as dense maps S^T, T^T
                             // (forward, backward; k_dense_sweep), or null
};

// The block's work as a flat op list (built on the host by unrolling the
// V/W recursion), executed by one loop with each operation's code present
// once: a template-unrolled recursion inlined every operation per level and
// visit, and the kernel ran out of instruction cache.
enum SubOp : int { kOpResid = 0, kOpSweepF, kOpSweepB, kOpRestrict, kOpCoarse, kOpProlong };
constexpr int kSubMaxOps = 256;

struct SubcycleParams {
    int nlev;          // levels kc .. kt: index 0 = coarse (kc), nlev-1 = kt
    int nops;
    unsigned short ops[kSubMaxOps];  // (op << 4) | level j
    SubLevel lv[kSubMaxK];
    const double *inv;  // coarse A^-1, row-major, n = 2 (2^kc+1)^2
    double *x;          // level kt iterate (global), updated
    const double *rhs;  // level kt right-hand side (global)
    unsigned long long *prof;  // debug: %globaltimer at each op (or null)
};

// shared-memory layout: per level j, X_j and B_j (2N doubles each); per
// smoothed level j >= 1, the residual R_j as a zero-guarded (n1+2)^2 grid of
// (state, adjoint) pairs
// the generic level's CSR data staged in shared memory (from global memory
// every access was an L2 round trip: the coarse inverse evicts L1)
constexpr int kSubCsrNnz = 1024, kSubCsrRows = 64;
constexpr int kSubCsrDoubles =
    2 * kSubCsrNnz + 2 * kSubCsrRows + (2 * kSubCsrNnz + 3 * kSubCsrRows) / 2;

struct SubLayout {
    int off_x[kSubMaxK], off_b[kSubMaxK], off_r[kSubMaxK];
    int off_a[kSubMaxK], off_c[kSubMaxK];  // A rows [49][28], mc table [49][2][29]
    int off_csr;  // kSubCsrDoubles: val, w, n_diag, then ints col, grid col, off, goff, rows
    int total;  // doubles
};

__host__ __device__ inline SubLayout sub_layout(int nlev, const int *n1s) {
    SubLayout L{};
    int o = 0;
    for (int j = 0; j < nlev; ++j) {
        const int n1 = n1s[j], N = n1 * n1;
        if (j >= 1) {  // 16-byte aligned pairs first
            o = (o + 1) & ~1;
            L.off_r[j] = o;
            o += 2 * (n1 + 2) * (n1 + 2);
        }
        L.off_x[j] = o;
        o += 2 * N;
        L.off_b[j] = o;
        o += 2 * N;
        if (j >= 1 && n1 >= 7) {  // the level's coefficients: shared memory, not
                                  // L1 (the coarse inverse streams through L1
                                  // every visit); CSR levels (n1 < 7) read theirs
            L.off_a[j] = o;
            o += 49 * 28;
            L.off_c[j] = o;
            o += 49 * 2 * 29;
        }
    }
    L.off_csr = o;
    o += kSubCsrDoubles;
    L.total = o;
    return L;
}

// shared-memory view of the generic level's CSR data
struct SubCsr {
    double *val, *w, *nd, *rt;
    int *col, *gcol, *off, *goff, *rows;
    __device__ SubCsr(double *base) {
        val = base;
        w = val + kSubCsrNnz;
        nd = w + kSubCsrNnz;
        rt = nd + kSubCsrRows;  // the entering residual of a dense-map sweep
        col = reinterpret_cast<int *>(rt + kSubCsrRows);
        gcol = col + kSubCsrNnz;
        off = gcol + kSubCsrNnz;
        goff = off + kSubCsrRows;
        rows = goff + kSubCsrRows;
    }
};

namespace sub {

__device__ __forceinline__ void residual(int n1, const double *At, const double *X,
                                         const double *B, double2 *R) {
    const int N = n1 * n1, P = n1 + 2;
    for (int v = threadIdx.x; v < N; v += blockDim.x) {
        const int iy = v / n1, ix = v - iy * n1;
        const P1Node q = p1_node(ix, iy, n1);
        const double *A = At + q.c * 28;
        double s[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {  // p1_row_dot order
            double acc = 0.0;
#pragma unroll
            for (int d = 0; d < 7; ++d)
                if (q.ex[d]) acc = __dadd_rn(acc, __dmul_rn(A[14 * b + d], X[q.nb[d]]));
#pragma unroll
            for (int d = 0; d < 7; ++d)
                if (q.ex[d]) acc = __dadd_rn(acc, __dmul_rn(A[14 * b + 7 + d], X[N + q.nb[d]]));
            s[b] = -acc;
        }
        R[(iy + 1) * P + ix + 1] =
            make_double2(__dadd_rn(s[0], B[v]), __dadd_rn(s[1], B[N + v]));
    }
    __syncthreads();
}

__device__ __forceinline__ void sweep(int n1, const double *Ct, double *X, double2 *R,
                                      bool forward) {
    const int N = n1 * n1, P = n1 + 2;
    const int per_row = (n1 + 6) / 7, count = per_row * n1;
    const int f0 = forward ? 0 : 1;
    for (int b = 0; b < kMcColours; ++b) {
        const int cm = forward ? b : kMcColours - 1 - b;
        for (int k = threadIdx.x; k < count; k += blockDim.x) {
            const int iy = k / per_row, jj = k - iy * per_row;
            const int ix = ((cm - 2 * iy) % 7 + 7) % 7 + 7 * jj;
            if (ix >= n1) continue;
            const int c = (iy + 1) * P + ix + 1;
            const int off[7] = {-P - 1, -P, -1, 0, 1, P, P + 1};
            double2 v[7];
#pragma unroll
            for (int d = 0; d < 7; ++d) v[d] = R[c + off[d]];
            const int cls = 7 * p1_axis_class(iy, n1) + p1_axis_class(ix, n1);
            double p[2];
            p[f0] = mcs::node_update(v, Ct + (cls * 2 + f0) * 29);
            p[1 - f0] = mcs::node_update(v, Ct + (cls * 2 + 1 - f0) * 29);
#pragma unroll
            for (int d = 0; d < 7; ++d) R[c + off[d]] = v[d];
            const int xi = iy * n1 + ix;
            X[xi] = __dadd_rn(X[xi], p[0]);
            X[N + xi] = __dadd_rn(X[N + xi], p[1]);
        }
        __syncthreads();
    }
}

// generic level: r = -(A x) + b in CSR column order (k_csr_residual), into
// the same guarded (state, adjoint) grid the structured ops use; gcol holds
// each column's (grid pair, field) position in that grid
__device__ __forceinline__ int grid_pos(int n1, int i) {
    const int N = n1 * n1, f = i >= N, v = i - f * N, iy = v / n1, ix = v - iy * n1;
    return 2 * ((iy + 1) * (n1 + 2) + ix + 1) + f;
}
__device__ __forceinline__ void residual_csr(const SubLevel &l, const SubCsr &c, const double *X,
                                             const double *B, double2 *R) {
    const int n = 2 * l.n1 * l.n1;
    double *Rd = reinterpret_cast<double *>(R);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
        for (int t = c.off[i]; t < c.off[i + 1]; ++t)
            s = __dadd_rn(s, __dmul_rn(c.val[t], X[c.col[t]]));
        Rd[grid_pos(l.n1, i)] = __dadd_rn(-s, B[i]);
    }
    __syncthreads();
}
// generic level, multicolour NE-GS as its dense map (k_dense_sweep's
// arithmetic: x += S r, r <- T r, sums over j in order)
__device__ __forceinline__ void sweep_dense(const SubLevel &l, const SubCsr &c, double *X,
                                            double2 *R, bool forward) {
    double *Rd = reinterpret_cast<double *>(R);
    const int n = 2 * l.n1 * l.n1;
    for (int j = threadIdx.x; j < n; j += blockDim.x) c.rt[j] = Rd[grid_pos(l.n1, j)];
    __syncthreads();
    const double *ST = l.dense[forward ? 0 : 1], *TT = ST + (int64_t)n * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double ds = 0.0, rt = 0.0;
        for (int j = 0; j < n; ++j) {
            const double rj = c.rt[j];
            ds = fma(__ldg(ST + (int64_t)j * n + i), rj, ds);
            rt = fma(__ldg(TT + (int64_t)j * n + i), rj, rt);
        }
        X[i] += ds;
        Rd[grid_pos(l.n1, i)] = rt;
    }
    __syncthreads();
}
// generic level, multicolour NE-GS: the colour groups in order (backward:
// reversed), a group's rows in parallel, csr_gs_row's arithmetic (used when
// the level has no dense maps)
__device__ __forceinline__ void sweep_csr(const SubLevel &l, const SubCsr &c, double *X,
                                          double2 *R, bool forward) {
    double *Rd = reinterpret_cast<double *>(R);
    for (int g = 0; g < l.ngroups; ++g) {
        const int gg = forward ? g : l.ngroups - 1 - g;
        const int lo = c.goff[gg], hi = c.goff[gg + 1];
        for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
            const int i = c.rows[k];
            const int b = c.off[i], e = c.off[i + 1];
            double q = 0.0;
            for (int t = b; t < e; ++t) q = __dadd_rn(q, __dmul_rn(c.w[t], Rd[c.gcol[t]]));
            const double p = __ddiv_rn(q, c.nd[i]);
            X[i] = __dadd_rn(X[i], p);
            constexpr int kB = 8;  // distinct columns: loads batched before stores
            for (int t0 = b; t0 < e; t0 += kB) {
                double rv[kB];
                int gv[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (t0 + u < e) {
                        gv[u] = c.gcol[t0 + u];
                        rv[u] = Rd[gv[u]];
                    }
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (t0 + u < e) Rd[gv[u]] = __dsub_rn(rv[u], __dmul_rn(c.val[t0 + u], p));
            }
        }
        __syncthreads();
    }
}

// coarse (nc1) <- R fine residual (2 nc1 - 1), k_p1_restrict arithmetic
__device__ __forceinline__ void restrict_to(int nc1, const double2 *R, double *Bc) {
    const int nf1 = 2 * nc1 - 1, P = nf1 + 2, Nc = nc1 * nc1;
    for (int v = threadIdx.x; v < Nc; v += blockDim.x) {
        const int cy = v / nc1, cx = v - cy * nc1;
        const bool l = cx > 0, rr = cx < nc1 - 1, dn = cy > 0, up = cy < nc1 - 1;
        const int c = (2 * cy + 1) * P + 2 * cx + 1;
        double s[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            auto f = [&](int i) { return b ? R[i].y : R[i].x; };
            double a = 0.0;
            if (l && dn) a = __dadd_rn(a, __dmul_rn(0.5, f(c - P - 1)));
            if (dn) a = __dadd_rn(a, __dmul_rn(0.5, f(c - P)));
            if (l) a = __dadd_rn(a, __dmul_rn(0.5, f(c - 1)));
            a = __dadd_rn(a, f(c));
            if (rr) a = __dadd_rn(a, __dmul_rn(0.5, f(c + 1)));
            if (up) a = __dadd_rn(a, __dmul_rn(0.5, f(c + P)));
            if (rr && up) a = __dadd_rn(a, __dmul_rn(0.5, f(c + P + 1)));
            s[b] = a;
        }
        Bc[v] = s[0];
        Bc[Nc + v] = s[1];
    }
    __syncthreads();
}

// fine X += P coarse X (k_p1_prolong_add arithmetic)
__device__ __forceinline__ void prolong_add(int nc1, const double *Xc, double *Xf) {
    const int nf1 = 2 * nc1 - 1, Nf = nf1 * nf1, Nc = nc1 * nc1;
    for (int v = threadIdx.x; v < Nf; v += blockDim.x) {
        const int fy = v / nf1, fx = v - fy * nf1;
        const int ox = fx & 1, oy = fy & 1;
        const int a = (fy >> 1) * nc1 + (fx >> 1);
        const int b2 = ((fy >> 1) + oy) * nc1 + (fx >> 1) + ox;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const double *cc = Xc + b * Nc;
            const double s = (ox | oy) ? __dadd_rn(__dmul_rn(0.5, cc[a]), __dmul_rn(0.5, cc[b2]))
                                       : __dmul_rn(1.0, cc[a]);
            Xf[b * Nf + v] = __dadd_rn(Xf[b * Nf + v], s);
        }
    }
    __syncthreads();
}

// X = A^-1 B, warp per row (k_coarse_inv arithmetic), four rows per warp in
// flight: a row's loads are one L2 round trip, and the rows of a warp used to
// queue behind each other
__device__ __forceinline__ void coarse(int n, const double *__restrict__ inv, const double *B, double *X) {
    constexpr int RW = 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int row0 = warp; row0 < n; row0 += RW * nw) {
        double acc[RW];
#pragma unroll
        for (int k = 0; k < RW; ++k) acc[k] = 0.0;
        for (int j = lane; j < n; j += 32) {
            const double bj = B[j];
#pragma unroll
            for (int k = 0; k < RW; ++k) {
                const int row = row0 + k * nw;
                if (row < n) acc[k] = fma(__ldg(inv + (int64_t)row * n + j), bj, acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < RW; ++k) {
#pragma unroll
            for (int o = 16; o; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
            const int row = row0 + k * nw;
            if (lane == 0 && row < n) X[row] = acc[k];
        }
    }
    __syncthreads();
}

}  // namespace sub

__global__ void __launch_bounds__(kSubThreads, 1)
    k_p1_subcycle(const __grid_constant__ SubcycleParams P) {
    pdl_trigger();  // launched with PDL (short dependent launches of a cycle)
    pdl_wait();
    extern __shared__ double sm[];
    int n1s[kSubMaxK];
    for (int j = 0; j < P.nlev; ++j) n1s[j] = P.lv[j].n1;
    const SubLayout L = sub_layout(P.nlev, n1s);
    for (int i = threadIdx.x; i < L.total; i += blockDim.x) sm[i] = 0.0;  // guards
    __syncthreads();
    const SubCsr csr(sm + L.off_csr);
    for (int j = 1; j < P.nlev; ++j) {
        if (P.lv[j].csr) {
            const SubLevel &l = P.lv[j];
            const int n = 2 * l.n1 * l.n1, nnz = (int)l.off[n];
            for (int t = threadIdx.x; t < nnz; t += blockDim.x) {
                csr.val[t] = l.val[t];
                csr.w[t] = l.w[t];
                csr.col[t] = l.col[t];
                csr.gcol[t] = sub::grid_pos(l.n1, l.col[t]);
            }
            for (int i = threadIdx.x; i <= n; i += blockDim.x) {
                csr.off[i] = (int)l.off[i];
                if (i < n) {
                    csr.nd[i] = l.nd[i];
                    csr.rows[i] = l.rows[i];
                }
            }
            for (int g = threadIdx.x; g <= l.ngroups; g += blockDim.x) csr.goff[g] = (int)l.goff[g];
            continue;
        }
        for (int i = threadIdx.x; i < 49 * 28; i += blockDim.x)
            sm[L.off_a[j] + i] = P.lv[j].T[kP1OffA + i];
        for (int i = threadIdx.x; i < 49 * 58; i += blockDim.x)
            sm[L.off_c[j] + i] = P.lv[j].C[i];
    }
    const int top = P.nlev - 1, N = P.lv[top].n1 * P.lv[top].n1;
    double *X = sm + L.off_x[top], *B = sm + L.off_b[top];
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
        X[i] = P.x[i];
        B[i] = P.rhs[i];
    }
    __syncthreads();
    for (int t = 0; t < P.nops; ++t) {
        const int op = P.ops[t] >> 4, j = P.ops[t] & 15;
        if (P.prof && threadIdx.x == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            P.prof[t] = g;
        }
        double *Xj = sm + L.off_x[j], *Bj = sm + L.off_b[j];
        double2 *Rj = reinterpret_cast<double2 *>(sm + L.off_r[j]);
        switch (op) {
        case kOpResid:
            if (P.lv[j].csr)
                sub::residual_csr(P.lv[j], csr, Xj, Bj, Rj);
            else
                sub::residual(P.lv[j].n1, sm + L.off_a[j], Xj, Bj, Rj);
            break;
        case kOpSweepF:
        case kOpSweepB:
            if (P.lv[j].csr && P.lv[j].dense[0])
                sub::sweep_dense(P.lv[j], csr, Xj, Rj, op == kOpSweepF);
            else if (P.lv[j].csr)
                sub::sweep_csr(P.lv[j], csr, Xj, Rj, op == kOpSweepF);
            else
                sub::sweep(P.lv[j].n1, sm + L.off_c[j], Xj, Rj, op == kOpSweepF);
            break;
        case kOpRestrict: {  // B_{j-1} = R R_j, X_{j-1} = 0
            const int nc1 = P.lv[j - 1].n1;
            double *Xc = sm + L.off_x[j - 1];
            for (int i = threadIdx.x; i < 2 * nc1 * nc1; i += blockDim.x) Xc[i] = 0.0;
            sub::restrict_to(nc1, Rj, sm + L.off_b[j - 1]);
            break;
        }
        case kOpCoarse: sub::coarse(2 * P.lv[0].n1 * P.lv[0].n1, P.inv, Bj, Xj); break;
        default: sub::prolong_add(P.lv[j - 1].n1, sm + L.off_x[j - 1], Xj); break;
        }
    }
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) P.x[i] = X[i];
}

// host: the op list of one visit of level j (mirrors cycle_rec)
inline void sub_ops(int j, int cycle_w, int nu_pre, int nu_post, bool slsgs,
                    std::vector<unsigned short> &ops) {
    auto push = [&](int op, int lev) { ops.push_back((unsigned short)((op << 4) | lev)); };
    if (j == 0) {
        push(kOpCoarse, 0);
        return;
    }
    auto smooth = [&](int nu) {
        for (int i = 0; i < nu; ++i) {
            push(kOpSweepF, j);
            if (slsgs) push(kOpSweepB, j);
        }
    };
    push(kOpResid, j);
    smooth(nu_pre);
    push(kOpRestrict, j);
    const int rec = (cycle_w && j - 1 > 0) ? 2 : 1;
    for (int k = 0; k < rec; ++k) sub_ops(j - 1, cycle_w, nu_pre, nu_post, slsgs, ops);
    push(kOpProlong, j);
    push(kOpResid, j);
    smooth(nu_post);
}

}  // namespace ocmg
