"""Vanka patch smoother on the device against the
oracle's restatement of kernels.vanka_sweep and the reference's own outputs
(tests/golden/*vanka*)."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1502_03917_b200 as P  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("k,alpha", [(2, 1e-4), (3, 1e-4), (4, 1e-6)])
def test_vanka_sweeps_bitwise_vs_oracle(k, alpha):
    """Same operator, same patches: the level-scheduled device sweep equals
    the oracle's sequential loop bit for bit, forward and backward."""
    dsys = P.build_stokes_system(k, alpha)
    st = P.make_smoother(dsys, "vanka")
    pt = st.patches
    A = dsys.to_scipy()
    rng = np.random.default_rng(30 + k)
    x0 = rng.uniform(-1, 1, dsys.n)
    f = rng.uniform(-1, 1, dsys.n)
    r0 = f - A @ x0
    xd = torch.from_numpy(x0.copy()).cuda()
    rd = torch.from_numpy(r0.copy()).cuda()
    xo, ro = x0.copy(), r0.copy()
    st.sweep(xd, rd)
    ops = O.ocmg_oracle.vanka_sweep(pt.offsets, pt.dofs, pt.inverses, pt.sizes,
                                    A, 0.4, xo, ro, True)
    assert np.array_equal(xd.cpu().numpy(), xo)
    assert np.array_equal(rd.cpu().numpy(), ro)
    assert st.op_count == ops
    st.sweep(xd, rd, post=True)
    O.ocmg_oracle.vanka_sweep(pt.offsets, pt.dofs, pt.inverses, pt.sizes, A, 0.4,
                              xo, ro, False)
    assert np.array_equal(xd.cpu().numpy(), xo)
    assert np.array_equal(rd.cpu().numpy(), ro)


def test_vanka_sweep_vs_reference_golden():
    g = np.load(os.path.join(GOLD, "sweep_stokes_k3_vanka.npz"))
    dsys = P.build_stokes_system(3, 1e-4)
    st = P.make_smoother(dsys, "vanka")
    assert np.array_equal(st.patches.dofs, g["dofs"])
    xd = torch.from_numpy(g["x0"].copy()).cuda()
    rd = torch.from_numpy(g["r0"].copy()).cuda()
    st.sweep(xd, rd)
    assert rel(xd.cpu().numpy(), g["fwd_x"]) < 1e-14
    assert rel(rd.cpu().numpy(), g["fwd_r"]) < 1e-14
    st.sweep(xd, rd, post=True)
    assert rel(xd.cpu().numpy(), g["fwdbwd_x"]) < 1e-14


@pytest.mark.parametrize("k,tag", [(4, "s4_vanka"), (5, "c4_vanka")])
def test_vanka_baseline_solve_vs_reference(k, tag):
    """BASELINE protocol (config-4 shape, V(2,2), Vanka pre forward / post
    backward): the reference's cycle count, history within 1e-10."""
    g = np.load(os.path.join(GOLD, f"baseline_{tag}.npz"))
    cfg = P.CycleConfig(smoother=P.SmootherKind("vanka"), cycle="v",
                        coarsest_level=1)
    mg = P.build_solver("stokes", k, 1e-4, cfg)
    f = P.baseline_rhs(mg.finest, 1)
    assert rel(f.cpu().numpy(), g["f"]) < 1e-14
    x, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=100)
    assert len(hist) == len(g["hist"])
    assert rel(np.array(hist), g["hist"]) < 1e-8
    assert rel(x.cpu().numpy(), g["x_final"]) < 1e-9
