"""Pin the CPU oracle against fixtures produced by the reference itself.

The fixtures (tests/golden/*.npz) come from tests/golden/gen_golden.py, which
imports the reference package ``ocmg`` in the build container.  Poisson
operators are assembled in the reference's own element order and must match
bitwise; Stokes element matrices are integrated exactly here while the
reference uses a degree-4 rule, so Stokes values agree to round-off (the
reference also stores ~1e-15 quadrature-noise entries that are exact zeros
here).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O


def _csr(d, p):
    return sp.csr_matrix((d[p + "_data"], d[p + "_indices"],
                          d[p + "_indptr"]), shape=tuple(d[p + "_shape"]))


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_poisson_operators_bitwise(golden):
    d = golden("ops_poisson_k3.npz")
    s, c = O.poisson_system(3, 1e-6), O.poisson_system(2, 1e-6)
    A = _csr(d, "A")
    assert np.array_equal(A.indptr, s.A.indptr)
    assert np.array_equal(A.indices, s.A.indices)
    assert np.array_equal(A.data, s.A.data)
    assert np.array_equal(d["L"], s.L)
    st = O.OracleSmoother(s)
    assert np.array_equal(d["n_diag"], st.n_diag)
    assert np.array_equal(d["row_scaled"], st.row_scaled)
    t = O.system_transfer(c, s)
    assert (_csr(d, "P") != t.P).nnz == 0
    assert (_csr(d, "R") != t.R).nnz == 0


def test_stokes_operators_roundoff(golden):
    d = golden("ops_stokes_k2.npz")
    s, c = O.stokes_system(2, 1e-4), O.stokes_system(1, 1e-4)
    A = _csr(d, "A")
    assert abs(s.A - A).max() <= 1e-15 * abs(A).max()
    assert _rel(s.L, d["L"]) < 1e-15
    assert _rel(O.OracleSmoother(s).n_diag, d["n_diag"]) < 1e-15
    t = O.system_transfer(c, s)
    assert (_csr(d, "P") != t.P).nnz == 0   # P2/P1 weights are dyadic
    assert (_csr(d, "R") != t.R).nnz == 0


@pytest.mark.parametrize("prob,k,alpha", [("poisson", 4, 1e-6),
                                          ("stokes", 3, 1e-4)])
def test_sweeps(golden, prob, k, alpha):
    d = golden(f"sweep_{prob}_k{k}.npz")
    s = (O.poisson_system if prob == "poisson" else O.stokes_system)(k, alpha)
    tol = 0.0 if prob == "poisson" else 1e-14
    r0 = s.residual(d["x0"], d["f"])
    assert _rel(r0, d["r0"]) <= tol
    for name in ("normal", "lsgs", "slsgs"):
        st = O.OracleSmoother(s, name)
        x, r = d["x0"].copy(), d["r0"].copy()
        st.sweep(x, r)
        assert _rel(x, d[name + "_x"]) <= tol, name
        assert _rel(r, d[name + "_r"]) <= tol, name
        if prob == "poisson":
            assert st.op_count == int(d[name + "_ops"])
    st = O.OracleSmoother(s, "lsgs")
    x, r = d["x0"].copy(), d["r0"].copy()
    st.lsgs(x, r, forward=False)
    assert _rel(x, d["lsgs_bwd_x"]) <= tol
    assert _rel(r, d["lsgs_bwd_r"]) <= tol


def test_cgs_sweep_bitwise(golden):
    """CGS (kernels.py:70-96) restated in C: bitwise against the reference,
    one and two sweeps, touched-entry count."""
    d = golden("sweep_poisson_k4_cgs.npz")
    s = O.poisson_system(4, 1e-6)
    st = O.OracleSmoother(s, "cgs")
    x, r = d["x0"].copy(), d["r0"].copy()
    st.sweep(x, r)
    assert np.array_equal(x, d["cgs_x"]) and np.array_equal(r, d["cgs_r"])
    assert st.op_count == int(d["cgs_ops"])
    st.sweep(x, r)
    assert np.array_equal(x, d["cgs2_x"]) and np.array_equal(r, d["cgs2_r"])


@pytest.mark.parametrize("prob", ["poisson", "stokes"])
def test_coarse(golden, prob):
    d = golden(f"coarse_{prob}.npz")
    s = (O.poisson_system if prob == "poisson" else O.stokes_system)(
        1, 1e-6 if prob == "poisson" else 1e-4)
    x = O.OracleCoarse(s).solve(d["rhs"])
    assert _rel(x, d["x"]) < 1e-12


CASES = [
    # tag, problem, k, alpha, smoother, cycle, coarsest, seed, sine
    ("c1_lsgs", "poisson", 6, 1e-6, "lsgs", "v", 1, 0, False),
    ("c1_normal", "poisson", 6, 1e-6, "normal", "v", 1, 0, False),
    ("c1_slsgs", "poisson", 6, 1e-6, "slsgs", "v", 1, 0, False),
    ("c4_lsgs", "stokes", 5, 1e-4, "lsgs", "v", 1, 1, False),
    ("c4_normal", "stokes", 5, 1e-4, "normal", "v", 1, 1, False),
    # the CGS collective smoother
    ("c1_cgs", "poisson", 6, 1e-6, "cgs", "v", 1, 0, False),
    ("p6_a1e-4_c2_cgs", "poisson", 6, 1e-4, "cgs", "v", 2, 0, False),
    ("p5w_sine_cgs", "poisson", 5, 1e-6, "cgs", "w", 1, 0, True),
    ("p5w_sine", "poisson", 5, 1e-6, "lsgs", "w", 1, 0, True),
    ("p6_a1e-4_c2", "poisson", 6, 1e-4, "lsgs", "v", 2, 0, False),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_baseline_protocol(golden, case):
    tag, prob, k, alpha, sm, cyc, co, seed, sine = case
    d = golden(f"baseline_{tag}.npz")
    nu = 1 if sm == "slsgs" else 2
    mg = O.build_oracle(prob, k, alpha, coarsest=co, smoother=sm, cycle=cyc,
                        nu_pre=nu, nu_post=nu)
    f = O.baseline_rhs(mg.finest, seed, add_sine=sine)
    assert np.abs(f - d["f"]).max() <= 1e-15 * np.abs(d["f"]).max()
    x, hist, its = O.baseline_solve(mg, f, keep_iterates=len(d["iterates"]))
    assert len(hist) == len(d["hist"])           # identical cycle counts
    tol = 0.0 if prob == "poisson" else 1e-13
    for a, b in zip(its, d["iterates"]):
        assert _rel(a, b) <= tol
    assert _rel(x, d["x_final"]) <= tol


def test_reference_protocol(golden):
    d = golden("refproto_p4_lsgs.npz")
    mg = O.build_oracle("poisson", 4, 1.0, smoother="lsgs", cycle="w")
    hist = O.reference_solve(mg)
    assert len(hist) - 1 == int(d["iterations"])
    assert np.array_equal(np.array(hist), d["hist"])
    d = golden("refproto_s3_normal.npz")
    mg = O.build_oracle("stokes", 3, 1e-6, smoother="normal", cycle="w")
    hist = O.reference_solve(mg)
    assert len(hist) - 1 == int(d["iterations"])
    assert _rel(np.array(hist), d["hist"]) < 1e-12


def test_published_checkpoints():
    """Checkpoints from SURVEY.md §8(c) (measured on the reference)."""
    mg = O.build_oracle("poisson", 6, 1e-6, smoother="lsgs", cycle="v")
    f = O.baseline_rhs(mg.finest, 0)
    assert abs(np.linalg.norm(f) - 4.750547e-03) < 1e-9
    x, hist, _ = O.baseline_solve(mg, f)
    assert len(hist) == 28
    assert abs(hist[0] - 3.706431e+01) < 1e-5
    assert abs(x.sum() - (-2.886130646613e+01)) < 1e-9
