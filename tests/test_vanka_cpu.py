"""Vanka patch smoother, CPU side: the oracle's
restatement of kernels.vanka_sweep and the package's patch builder against
the reference's own outputs (tests/golden/sweep_stokes_k3_vanka.npz, made by
tests/golden/gen_golden.py vanka)."""
import os
import types

import numpy as np

import oracle as O
from paper_1502_03917_b200.assembly import FieldLayout
from paper_1502_03917_b200.mesh import StructuredMesh
from paper_1502_03917_b200.vanka import build_vanka_patches

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    return np.load(os.path.join(GOLD, "sweep_stokes_k3_vanka.npz"))


def _ref_A(g):
    import scipy.sparse as sp
    return sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]),
                         shape=tuple(g["A_shape"]))


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_oracle_vanka_sweep_matches_reference():
    """On the reference's own operator and patches: bit-identical forward
    and forward+backward sweeps."""
    g = _golden()
    A = _ref_A(g)
    x, r = g["x0"].copy(), g["r0"].copy()
    O.ocmg_oracle.vanka_sweep(g["offsets"], g["dofs"], g["inverses"], g["sizes"],
                              A, 0.4, x, r, True)
    assert np.array_equal(x, g["fwd_x"]) and np.array_equal(r, g["fwd_r"])
    O.ocmg_oracle.vanka_sweep(g["offsets"], g["dofs"], g["inverses"], g["sizes"],
                              A, 0.4, x, r, False)
    assert np.array_equal(x, g["fwdbwd_x"]) and np.array_equal(r, g["fwdbwd_r"])


def test_oracle_vanka_on_exact_assembly():
    """On the exactly assembled operator (the package's and the oracle's:
    exact zeros where the reference's quadrature leaves ~1e-17): within
    1e-15 of the reference."""
    g = _golden()
    A = O.stokes_system(3, 1e-4).A
    x, r = g["x0"].copy(), g["r0"].copy()
    O.ocmg_oracle.vanka_sweep(g["offsets"], g["dofs"], g["inverses"], g["sizes"],
                              A, 0.4, x, r, True)
    assert rel(x, g["fwd_x"]) < 1e-15 and rel(r, g["fwd_r"]) < 1e-15


def test_patch_builder_matches_reference():
    """build_vanka_patches on the oracle's operator (the package's Stokes
    assembly is bit-identical to it): same patches, bit-identical inverses."""
    g = _golden()
    osys = O.stokes_system(3, 1e-4)
    mesh = StructuredMesh(3)
    counts = [c for _, c in osys.fields]
    layout = FieldLayout(("velocity", "pressure", "adjoint_velocity",
                          "adjoint_pressure"), tuple(counts),
                         ("p2", "p1", "p2", "p1"))
    system = types.SimpleNamespace(problem="stokes", mesh=mesh, layout=layout,
                                   n_velocity_scalar=counts[0] // 2,
                                   to_scipy=lambda: osys.A)
    pt = build_vanka_patches(system)
    for name in ("offsets", "dofs", "sizes", "vertex_ids"):
        assert np.array_equal(getattr(pt, name), g[name]), name
    # bit-identical on the reference's operator, 1e-12 on the exact one
    assert rel(pt.inverses, g["inverses"]) < 1e-12
    system.to_scipy = lambda: _ref_A(g)
    assert np.array_equal(build_vanka_patches(system).inverses, g["inverses"])
