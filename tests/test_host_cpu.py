"""CPU-only checks of the product's host side and the C ABI surface.

No kernel is launched here: these tests check that the host setup (mesh
numbering, assembly, stencil class tables, transfers) is bit-identical to
the oracle, and that libocmg_b200.so exports exactly what
include/ocmg_b200.h declares.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_1502_03917_b200 import _lib
from paper_1502_03917_b200 import assembly as As
from paper_1502_03917_b200 import mesh as Me
from paper_1502_03917_b200 import transfer as Tr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OFF7 = [(-1, -1), (0, -1), (-1, 0), (0, 0), (1, 0), (0, 1), (1, 1)]
LOW9 = [(-2, -2), (-1, -2), (0, -2), (-2, -1), (-1, -1), (0, -1), (1, -1),
        (-2, 0), (-1, 0)]


def _cls(i, n1):
    return i if i < 3 else (6 - (n1 - 1 - i) if i > n1 - 4 else 3)


def _split(t):
    A = t[:1372].reshape(49, 2, 14)
    W = t[1372:2744].reshape(49, 2, 14)
    L = t[2744:2842].reshape(49, 2)
    ND = t[2842:2940].reshape(49, 2)
    WF = t[2940:].reshape(49, 38)
    return A, W, L, ND, WF


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_poisson_csr_matches_oracle(k):
    a, L, _ = As._poisson_csr(Me.StructuredMesh(k), 1e-6)
    o = O.poisson_system(k, 1e-6)
    assert (a != o.A).nnz == 0 and np.array_equal(L, o.L)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_taylor_hood_matches_oracle(k):
    ms, ks, d = As.assemble_taylor_hood(Me.StructuredMesh(k))
    oms, oks, od = O.assemble_p2(O.StructuredLevel(k))
    assert (ms != oms).nnz == 0 and (ks != oks).nnz == 0 and (d != od).nnz == 0


@pytest.mark.parametrize("kc", [0, 1, 2, 3])
def test_prolongations_match_oracle(kc):
    c, f = Me.StructuredMesh(kc), Me.StructuredMesh(kc + 1)
    assert (Tr.p1_prolongation(c, f) != O.p1_prolongation(kc)).nnz == 0
    if kc >= 1:
        assert (Tr.p2_prolongation(c, f) != O.p2_prolongation(kc)).nnz == 0


@pytest.mark.parametrize("k,alpha", [(3, 1e-6), (4, 1.0), (5, 1e-4),
                                     (6, 1e-8), (5, 1e-12)])
def test_class_tables_bitwise(k, alpha):
    """Stencil tables reproduce A, row_scaled, L and n_diag of the
    assembled CSR bit for bit at every vertex."""
    A, W, L, ND, _ = _split(As.p1_class_tables(k, alpha))
    o = O.poisson_system(k, alpha)
    st = O.OracleSmoother(o)
    n1 = 2 ** k + 1
    N = n1 * n1
    for iy in range(n1):
        for ix in range(n1):
            c = 7 * _cls(iy, n1) + _cls(ix, n1)
            v = iy * n1 + ix
            for b in range(2):
                i = b * N + v
                lo, hi = o.A.indptr[i], o.A.indptr[i + 1]
                got = {}
                for d, (dx, dy) in enumerate(OFF7):
                    if 0 <= ix + dx < n1 and 0 <= iy + dy < n1:
                        u = (iy + dy) * n1 + ix + dx
                        got[u] = (A[c, b, d], W[c, b, d])
                        got[N + u] = (A[c, b, 7 + d], W[c, b, 7 + d])
                want = {j: (a, w) for j, a, w in zip(
                    o.A.indices[lo:hi], o.A.data[lo:hi],
                    st.row_scaled[lo:hi])}
                assert got == want
                assert L[c, b] == o.L[i] and ND[c, b] == st.n_diag[i]


@pytest.mark.parametrize("k,alpha", [(4, 1e-6), (5, 1.0)])
def test_normal_equation_tables(k, alpha):
    """Delta-form coefficients equal the dense N = A^T L^-1 A."""
    *_, WF = _split(As.p1_class_tables(k, alpha))
    o = O.poisson_system(k, alpha)
    A = o.A.toarray()
    Nm = A.T @ np.diag(1.0 / o.L) @ A
    n1 = 2 ** k + 1
    NN = n1 * n1
    for iy in range(n1):
        for ix in range(n1):
            c = 7 * _cls(iy, n1) + _cls(ix, n1)
            v = iy * n1 + ix
            for j, (dx, dy) in enumerate(LOW9):
                for sgn, base in ((1, 0), (-1, 18)):
                    ux, uy = ix + sgn * dx, iy + sgn * dy
                    ok = 0 <= ux < n1 and 0 <= uy < n1
                    u = uy * n1 + ux
                    ey = Nm[v, u] if ok else 0.0
                    el = Nm[NN + v, NN + u] if ok else 0.0
                    assert abs(WF[c, base + j] - ey) <= 1e-15 * Nm[v, v]
                    assert abs(WF[c, base + 9 + j] - el) <= \
                        1e-15 * Nm[NN + v, NN + v]
            assert abs(WF[c, 36] * Nm[v, v] - 1) < 1e-15
            assert abs(WF[c, 37] * Nm[NN + v, NN + v] - 1) < 1e-15


def test_norm_diag_vector():
    o = O.poisson_system(5, 1e-4)
    assert np.array_equal(As.p1_norm_diag(5, 1e-4), o.L)


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ocmg_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return set(re.findall(r"\b(ocmg_[a-z0-9_]+)\s*\(", hdr))


def test_library_exports_header_symbols():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ocmg_[a-z0-9_]+)$", out, flags=re.M))
    declared = _declared_symbols()
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    assert declared == set(_lib.SIGNATURES), \
        declared.symmetric_difference(set(_lib.SIGNATURES))
    lib = _lib.load()           # loads without a GPU
    assert lib.ocmg_abi_version() == 1


def test_device_path_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1502_03917_b200 as P
    with pytest.raises(RuntimeError):
        P.build_poisson_system(4, 1e-6)


def test_package_does_not_import_oracle():
    """The oracle is test infrastructure: the product never loads it."""
    import subprocess
    import sys
    code = ("import sys, paper_1502_03917_b200; "
            "assert not any(m == 'oracle' or m.startswith('oracle.') "
            "for m in sys.modules), 'oracle imported'")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)


def test_config_validation():
    import paper_1502_03917_b200 as P
    with pytest.raises(ValueError):
        P.SmootherKind("bogus")
    with pytest.raises(ValueError):
        P.SmootherKind("normal", tau=2.5)
    with pytest.raises(ValueError):
        P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="x")
    with pytest.raises(ValueError):
        P.CycleConfig(smoother=P.SmootherKind("lsgs"), nu_pre=0, nu_post=0)
    with pytest.raises(ValueError):
        P.CycleConfig(smoother=P.SmootherKind("lsgs"), gs_mode="fast")


def test_table_request_and_renderers():
    """The table runner's request normalisation and its three formats
    (no GPU: cells filled by hand)."""
    from paper_1502_03917_b200 import tables as T
    with pytest.raises(ValueError):
        T.TableRequest(problem="heat").resolved()
    with pytest.raises(ValueError):
        T.TableRequest(problem="poisson", levels=(1, 2)).resolved()
    req = T.TableRequest(problem="poisson", smoothers=("lsgs",), levels=(3, 4),
                         alphas=(1.0,)).resolved()
    assert req.steps("slsgs") == (1, 1) and req.steps("lsgs") == (2, 2)
    tab = T.IterationTable(req)
    tab.add(T.TableCell("lsgs", 1.0, 3, 11, True))
    tab.add(T.TableCell("lsgs", 1.0, 4, None, False, "boom"))
    md = tab.render("markdown")
    assert "| level | lsgs a=1 |" in md and "| 3 | 11 |" in md and "| 4 | div |" in md
    csv_ = tab.render("csv").splitlines()
    assert csv_[0] == "problem,smoother,alpha,level,iterations,converged"
    assert csv_[2] == "poisson,lsgs,1,4,,false"
    import json
    js = json.loads(tab.render("json"))
    assert js["cells"][0]["iterations"] == 11 and js["cells"][1]["converged"] is False


def test_rolling_window_schedule_emulation():
    """The schedule of the experimental rolling-window multicolour kernel
    (ocmg_p1_mc2.cuh: own masks, window inheritance, ring slots, duties,
    tile decomposition), emulated on the CPU line by line
    (scripts/mc2_emulate.py), reproduces a plain colour-by-colour sweep
    exactly, forward and backward, on tiles with halos on every side."""
    import os
    import re
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for args in (("47", "27", "5", "1"), ("47", "27", "5", "0"), ("40", "171", "3", "1")):
        out = subprocess.run([sys.executable, os.path.join(root, "scripts", "mc2_emulate.py"), *args],
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        m = re.search(r"max\|dr\| (\S+) nan (\d+) max\|dx\| (\S+)", out.stdout)
        assert m, out.stdout
        assert float(m.group(1)) == 0.0 and int(m.group(2)) == 0 and float(m.group(3)) == 0.0, out.stdout
