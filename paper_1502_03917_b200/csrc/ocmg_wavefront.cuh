// Fused wavefront NE-GS for structured P1 levels (reference sweep order).
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
// N = A^T L^-1 A is the normal-equation operator; the
// delta form p_i = (G_i - sum_k N_ik p_k) / N_ii with G = A^T L^-1 r_entry is
// algebraically the reference's lsgs_sweep (kernels.py:57-64) in the same
// order, with the residual folded in once per sweep instead of per update.
#pragma once

#include "ocmg_common.cuh"

namespace ocmg {

constexpr int kWfStride = 38;
constexpr int kWfTableDoubles = 49 * kWfStride;

struct P1Wavefront {
    int k = 0, n1 = 0;
    const double *tab = nullptr;  // device, kWfTableDoubles
    void init(int k_, int n1_, const double *t) {
        k = k_;
        n1 = n1_;
        tab = t;
    }
    bool ready() const { return false; }
    void sweep(bool, double *, double *, cudaStream_t) const {}
};

}  // namespace ocmg
