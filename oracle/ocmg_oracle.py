"""CPU restatement of the ocmg hot path -- TEST INFRASTRUCTURE ONLY.

See ``oracle/__init__.py`` for who may import this.  Everything here is a
restatement (numpy/scipy + the sequential C kernels in ``oracle_kernels.c``)
of the reference package ``ocmg``; each function cites the reference
``file:line`` it follows (paths relative to ``/root/reference/pkg/src/ocmg``).

Scope: structured mesh numbering, P1 / Taylor-Hood assembly, the two
saddle-point systems with their diagonal weights, P1/P2 transfers, the
normal-equation smoothers (NE-Jacobi = reference ``normal``, NE-GS =
reference ``lsgs``, sLSGS), the dense coarse solve, the V/W cycle, the
reference solve protocol and the BASELINE.json protocol (f = (M y_D, 0),
x0 = 0, stop at ||f - A x||_2 <= 1e-8 ||f||_2).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import scipy.linalg
import scipy.sparse as sp

__all__ = [
    "StructuredLevel", "p1_element", "p2_elements", "assemble_p1",
    "assemble_p2", "OracleSystem", "poisson_system", "stokes_system",
    "p1_prolongation", "p2_prolongation", "OracleTransfer",
    "system_transfer", "OracleSmoother", "OracleCoarse", "OracleMultigrid",
    "build_oracle", "baseline_rhs", "baseline_solve", "reference_solve",
    "csr_residual", "lib",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    """Load (building on first use) the sequential C oracle kernels."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle_kernels.c")
        if (not os.path.exists(path)
                or os.path.getmtime(path) < os.path.getmtime(src)):
            subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"],
                           check=True)
        L = ctypes.CDLL(path)
        i64, dbl, p = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        L.orc_csr_matvec.argtypes = [i64, p, p, p, p, p]
        L.orc_csr_matvec.restype = None
        L.orc_residual.argtypes = [i64, p, p, p, p, p, p]
        L.orc_residual.restype = None
        L.orc_normal_sweep.argtypes = [i64, p, p, p, p, p, p, p, dbl,
                                       p, p, p]
        L.orc_normal_sweep.restype = i64
        L.orc_lsgs_sweep.argtypes = [i64, p, p, p, p, p, p, p, p, p,
                                     ctypes.c_int]
        L.orc_lsgs_sweep.restype = i64
        L.orc_collective_sweep.argtypes = [i64, p, p, p, p, p, dbl, p, p]
        L.orc_collective_sweep.restype = i64
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _canon(m):
    """Canonical CSR as the reference finalizes it (sparse.py:81-88)."""
    c = m.tocsr().copy()
    c.sum_duplicates()
    c.sort_indices()
    c.eliminate_zeros()
    c.indptr = c.indptr.astype(np.int64)
    c.indices = c.indices.astype(np.int64)
    return c


# ---------------------------------------------------------------------------
# structured mesh (mesh.py:139-180, 183-231, 266-286)
# ---------------------------------------------------------------------------

@dataclass
class StructuredLevel:
    """Level-k triangulation of the unit square, SW-NE diagonals.

    Vertex (ix, iy) has index iy*(2^k+1)+ix (x fastest, mesh.py:146-147).
    Cells are visited x fastest and each contributes its lower-right
    triangle (v00, v10, v11) then its upper-left (v00, v11, v01)
    (mesh.py:149-157).  Edges are the sorted vertex pairs in lexicographic
    order (mesh.py:159-166): for each lower vertex the horizontal, vertical,
    then diagonal edge.
    """

    k: int
    n1: int = field(init=False)
    nv: int = field(init=False)

    def __post_init__(self):
        self.n1 = 2 ** self.k + 1
        self.nv = self.n1 * self.n1

    @property
    def m(self):
        return 2 ** self.k

    def coords(self):
        xs = np.linspace(0.0, 1.0, self.n1)
        return np.tile(xs, self.n1), np.repeat(xs, self.n1)

    def triangles(self):
        m, n1 = self.m, self.n1
        cy, cx = np.divmod(np.arange(m * m), m)
        v00 = cy * n1 + cx
        tri = np.empty((2 * m * m, 3), dtype=np.int64)
        tri[0::2] = np.column_stack([v00, v00 + 1, v00 + n1 + 1])
        tri[1::2] = np.column_stack([v00, v00 + n1 + 1, v00 + n1])
        return tri

    def edge_ids(self):
        """Per-vertex ids of its horizontal/vertical/diagonal edge (-1 if
        absent) and the (ne, 2) edge array in lexicographic order."""
        n1, m = self.n1, self.m
        iy, ix = np.divmod(np.arange(self.nv), n1)
        has = np.stack([ix < m, iy < m, (ix < m) & (iy < m)], axis=1)
        flat = has.ravel()
        ids = np.full(flat.shape, -1, dtype=np.int64)
        ids[flat] = np.arange(int(flat.sum()))
        ids = ids.reshape(-1, 3)
        v = np.arange(self.nv)
        hi = np.stack([v + 1, v + n1, v + n1 + 1], axis=1)
        edges = np.column_stack([np.repeat(v, 3).reshape(-1, 3)[has],
                                 hi[has]])
        return ids, edges

    def triangle_edges(self):
        ids, _ = self.edge_ids()
        tri = self.triangles()
        te = np.empty_like(tri)
        lr, ul = tri[0::2], tri[1::2]
        # lower-right (v00,v10,v11): edges (v00,v10) h, (v10,v11) v, (v11,v00) d
        te[0::2] = np.column_stack([ids[lr[:, 0], 0], ids[lr[:, 1], 1],
                                    ids[lr[:, 0], 2]])
        # upper-left (v00,v11,v01): edges (v00,v11) d, (v11,v01) h, (v01,v00) v
        te[1::2] = np.column_stack([ids[ul[:, 0], 2], ids[ul[:, 2], 0],
                                    ids[ul[:, 0], 1]])
        return te

    def boundary(self):
        n1, m = self.n1, self.m
        iy, ix = np.divmod(np.arange(self.nv), n1)
        bv = (ix == 0) | (ix == m) | (iy == 0) | (iy == m)
        ids, edges = self.edge_ids()
        be = np.zeros(edges.shape[0], dtype=bool)
        hmask = ids[:, 0] >= 0
        be[ids[hmask, 0]] = (iy[hmask] == 0) | (iy[hmask] == m)
        vmask = ids[:, 1] >= 0
        be[ids[vmask, 1]] = (ix[vmask] == 0) | (ix[vmask] == m)
        return bv, be

    def p2_interior(self):
        """P2 dofs (vertices, then edges) that are not Dirichlet, and the
        dof -> interior position map (mesh.py:95-109, 273-281)."""
        bv, be = self.boundary()
        bnd = np.concatenate([bv, be])
        interior = np.where(~bnd)[0]
        idx = np.full(bnd.shape, -1, dtype=np.int64)
        idx[interior] = np.arange(interior.size)
        return interior, idx

    def p2_points(self):
        x, y = self.coords()
        _, edges = self.edge_ids()
        ex = 0.5 * (x[edges[:, 0]] + x[edges[:, 1]])
        ey = 0.5 * (y[edges[:, 0]] + y[edges[:, 1]])
        return np.concatenate([x, ex]), np.concatenate([y, ey])


# ---------------------------------------------------------------------------
# element matrices (assembly.py:22-36, 39-66, 69-80, 97-118, 134-183)
# ---------------------------------------------------------------------------

def _tri_shapes(h):
    """Vertex coordinates of the two congruent triangle types."""
    lr = np.array([[0.0, 0.0], [h, 0.0], [h, h]])
    ul = np.array([[0.0, 0.0], [h, h], [0.0, h]])
    return lr, ul


def p1_element(p):
    """Exact P1 mass and pure-Laplace stiffness of one triangle
    (assembly.py:69-80, 97-118)."""
    x, y = p[:, 0], p[:, 1]
    b = np.array([y[1] - y[2], y[2] - y[0], y[0] - y[1]])
    c = np.array([x[2] - x[1], x[0] - x[2], x[1] - x[0]])
    det = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0])
    area = 0.5 * det
    mass = (np.ones((3, 3)) + np.eye(3)) * (area / 12.0)
    lap = (np.outer(b, b) + np.outer(c, c)) / (4.0 * area)
    return mass, lap


def _poly_mul(a, b):
    out = {}
    for ea, ca in a.items():
        for eb, cb in b.items():
            e = (ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2])
            out[e] = out.get(e, 0) + ca * cb
    return out


def _poly_int(poly, area):
    """Exact integral over a triangle of a polynomial in the barycentric
    coordinates: int l0^a l1^b l2^c = 2 area a! b! c! / (a+b+c+2)!."""
    from math import factorial
    tot = Fraction(0)
    for (a, b, c), coef in poly.items():
        tot += coef * Fraction(2 * factorial(a) * factorial(b) * factorial(c),
                               factorial(a + b + c + 2))
    return tot * area


def _p2_polys():
    """P2 shape functions as barycentric polynomials and their partial
    derivatives d/dlambda_i; dof order: 3 vertices, then midpoints of the
    local edges (0,1), (1,2), (2,0) (assembly.py:39-66)."""
    def mono(i, j=None, c=1):
        e = [0, 0, 0]
        e[i] += 1
        if j is not None:
            e[j] += 1
        return {tuple(e): Fraction(c)}
    shapes = []
    for i in range(3):           # l_i (2 l_i - 1) = 2 l_i^2 - l_i
        p = {k: 2 * v for k, v in mono(i, i).items()}
        for k, v in mono(i).items():
            p[k] = p.get(k, 0) - v
        shapes.append(p)
    for i, j in ((0, 1), (1, 2), (2, 0)):
        shapes.append(mono(i, j, 4))

    def deriv(p, i):
        out = {}
        for e, c in p.items():
            if e[i]:
                f = list(e)
                f[i] -= 1
                out[tuple(f)] = out.get(tuple(f), 0) + c * e[i]
        return out
    return shapes, [[deriv(p, i) for i in range(3)] for p in shapes]


def p2_elements(p):
    """P2 mass, P2 Laplace and the P1 x P2 negative-divergence blocks of one
    triangle, integrated exactly and rounded once (the reference integrates
    the same polynomials with a degree-4 rule, assembly.py:134-183)."""
    pts = [(Fraction(float(x)), Fraction(float(y))) for x, y in p]
    (x0, y0), (x1, y1), (x2, y2) = pts
    det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    area = det / 2
    # gradient of lambda_i = (b_i, c_i) / det
    grad = [((y1 - y2) / det, (x2 - x1) / det),
            ((y2 - y0) / det, (x0 - x2) / det),
            ((y0 - y1) / det, (x1 - x0) / det)]
    shapes, dshapes = _p2_polys()

    def phys(a, comp):           # d phi_a / d x_comp as a polynomial
        out = {}
        for i in range(3):
            for e, c in dshapes[a][i].items():
                out[e] = out.get(e, 0) + c * grad[i][comp]
        return out
    mass = np.zeros((6, 6))
    lap = np.zeros((6, 6))
    dx = np.zeros((3, 6))
    dy = np.zeros((3, 6))
    g = [[phys(a, c) for c in range(2)] for a in range(6)]
    for a in range(6):
        for b in range(6):
            mass[a, b] = float(_poly_int(_poly_mul(shapes[a], shapes[b]),
                                         area))
            lap[a, b] = float(sum(_poly_int(_poly_mul(g[a][c], g[b][c]),
                                            area) for c in range(2)))
    for q in range(3):
        lam = {tuple(1 if t == q else 0 for t in range(3)): Fraction(1)}
        for a in range(6):
            dx[q, a] = float(-_poly_int(_poly_mul(lam, g[a][0]), area))
            dy[q, a] = float(-_poly_int(_poly_mul(lam, g[a][1]), area))
    return mass, lap, dx, dy


def _scatter(rows_l2g, cols_l2g, local, shape):
    """Triangle-by-triangle, local row-major COO scatter -> CSR
    (assembly.py:92-94)."""
    nt, a = rows_l2g.shape
    b = cols_l2g.shape[1]
    rows = np.repeat(rows_l2g, b, axis=1).ravel()
    cols = np.tile(cols_l2g, (1, a)).ravel()
    vals = np.broadcast_to(local.reshape(-1, a * b),
                           (nt, a * b)).ravel() if local.ndim == 3 \
        else local.ravel()
    return sp.coo_matrix((vals, (rows, cols)), shape=shape).tocsr()


def _per_type(local_lr, local_ul, nt):
    out = np.empty((nt,) + local_lr.shape)
    out[0::2] = local_lr
    out[1::2] = local_ul
    return out


def assemble_p1(level: StructuredLevel):
    """P1 mass M and K = Laplace + mass (Neumann, nothing eliminated)
    (assembly.py:97-131)."""
    tri = level.triangles()
    nt = tri.shape[0]
    lr, ul = _tri_shapes(1.0 / level.m)
    m_lr, l_lr = p1_element(lr)
    m_ul, l_ul = p1_element(ul)
    shape = (level.nv, level.nv)
    mass = _scatter(tri, tri, _per_type(m_lr, m_ul, nt), shape)
    lap = _scatter(tri, tri, _per_type(l_lr, l_ul, nt), shape)
    return _canon(mass), _canon(lap + mass)


def assemble_p2(level: StructuredLevel):
    """Taylor-Hood blocks with Dirichlet velocity dofs eliminated: scalar P2
    mass, P2 Laplace and D = [Dx | Dy] (n_p x 2 n_int) (assembly.py:134-201).
    """
    tri = level.triangles()
    te = level.triangle_edges()
    nt = tri.shape[0]
    nv = level.nv
    l2g2 = np.hstack([tri, nv + te])
    n2 = nv + te.max() + 1
    lr, ul = _tri_shapes(1.0 / level.m)
    e_lr = p2_elements(lr)
    e_ul = p2_elements(ul)
    mass_f = _scatter(l2g2, l2g2, _per_type(e_lr[0], e_ul[0], nt), (n2, n2))
    lap_f = _scatter(l2g2, l2g2, _per_type(e_lr[1], e_ul[1], nt), (n2, n2))
    dx_f = _scatter(tri, l2g2, _per_type(e_lr[2], e_ul[2], nt), (nv, n2))
    dy_f = _scatter(tri, l2g2, _per_type(e_lr[3], e_ul[3], nt), (nv, n2))
    interior, _ = level.p2_interior()
    mass = _canon(mass_f[interior][:, interior])
    lap = _canon(lap_f[interior][:, interior])
    div = _canon(sp.hstack([dx_f[:, interior], dy_f[:, interior]]))
    return mass, lap, div


# ---------------------------------------------------------------------------
# block systems (assembly.py:205-341, 381-388)
# ---------------------------------------------------------------------------

@dataclass
class OracleSystem:
    problem: str
    k: int
    alpha: float
    A: sp.csr_matrix
    L: np.ndarray                 # norm_diag (assembly.py:278-286, 318-334)
    fields: tuple                 # ((name, count), ...) in layout order
    mass: sp.csr_matrix           # state-state block used for f = M y_D

    @property
    def n(self):
        return self.A.shape[0]

    def slice_of(self, name):
        off = 0
        for nm, cnt in self.fields:
            if nm == name:
                return slice(off, off + cnt)
            off += cnt
        raise KeyError(name)

    def residual(self, x, rhs=None):
        """r = -(A x) + rhs in the reference rounding (assembly.py:259-263)."""
        return csr_residual(self.A, x, rhs)

    def norm(self, x):
        """sqrt(sum L_i x_i^2) (assembly.py:265-267)."""
        return float(np.sqrt(np.dot(self.L * x, x)))

    def mean_project(self, x):
        """Zero the means of both pressure fields (assembly.py:381-388)."""
        if self.problem == "stokes":
            for name in ("pressure", "adjoint_pressure"):
                s = self.slice_of(name)
                x[s] -= x[s].mean()
        return x


def poisson_system(k, alpha):
    """[[M, K], [K, -M/alpha]], L = [diag(M+sqrt(a)K), diag(..)/alpha]
    (assembly.py:270-290).  Scalar division of a scipy matrix multiplies by
    the reciprocal, which the reference inherits; restated here."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    lvl = StructuredLevel(k)
    m, kk = assemble_p1(lvl)
    a = sp.bmat([[m, kk], [kk, -m / alpha]], format="csr")
    w = m + np.sqrt(alpha) * kk
    wd = w.diagonal()
    n = lvl.nv
    return OracleSystem("poisson", k, float(alpha), _canon(a),
                        np.concatenate([wd, wd / alpha]),
                        (("state", n), ("adjoint", n)), m)


def stokes_system(k, alpha):
    """4x4 Taylor-Hood velocity-tracking system (assembly.py:293-341)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if k < 1:
        raise ValueError("velocity tracking needs mesh level >= 1")
    lvl = StructuredLevel(k)
    ms, ks, d = assemble_p2(lvl)
    mv = sp.block_diag([ms, ms], format="csr")
    kv = sp.block_diag([ks, ks], format="csr")
    dt = d.T.tocsr()
    a = sp.bmat([[mv, None, kv, dt], [None, None, d, None],
                 [kv, dt, -mv / alpha, None], [d, None, None, None]],
                format="csr")
    ws = ms + np.sqrt(alpha) * ks
    w_hat = np.concatenate([ws.diagonal(), ws.diagonal()])
    winv = 1.0 / w_hat
    contrib = d.data ** 2 * winv[d.indices]
    rows = np.repeat(np.arange(d.shape[0]), np.diff(d.indptr))
    tri = np.zeros(d.shape[0])
    np.add.at(tri, rows, contrib)            # sparse.py:239-255
    p_hat = alpha * tri
    n_int, n_p = ms.shape[0], lvl.nv
    fields = (("velocity", 2 * n_int), ("pressure", n_p),
              ("adjoint_velocity", 2 * n_int), ("adjoint_pressure", n_p))
    return OracleSystem("stokes", k, float(alpha), _canon(a),
                        np.concatenate([w_hat, p_hat, w_hat / alpha,
                                        p_hat / alpha]), fields,
                        _canon(mv))


def csr_residual(A, x, rhs=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    r = np.empty(A.shape[0])
    rh = None if rhs is None else np.ascontiguousarray(rhs, dtype=np.float64)
    lib().orc_residual(A.shape[0], _ptr(A.indptr), _ptr(A.indices),
                       _ptr(A.data), _ptr(x),
                       None if rh is None else _ptr(rh), _ptr(r))
    return r


def csr_matvec(A, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.shape[0])
    lib().orc_csr_matvec(A.shape[0], _ptr(A.indptr), _ptr(A.indices),
                         _ptr(A.data), _ptr(x), _ptr(y))
    return y


# ---------------------------------------------------------------------------
# transfers (transfer.py:22-143)
# ---------------------------------------------------------------------------

def p1_prolongation(kc):
    """Linear interpolation level kc -> kc+1: coarse vertices copy, edge
    midpoints average both ends (transfer.py:34-55, mesh.py:183-231)."""
    c, f = StructuredLevel(kc), StructuredLevel(kc + 1)
    fy, fx = np.divmod(np.arange(f.nv), f.n1)
    cx0, cy0 = fx // 2, fy // 2
    odd_x, odd_y = fx % 2 == 1, fy % 2 == 1
    a = cy0 * c.n1 + cx0                     # lower-left coarse end
    b = (cy0 + odd_y) * c.n1 + cx0 + odd_x   # upper-right coarse end
    own = ~(odd_x | odd_y)
    nnz = np.where(own, 1, 2)
    off = np.concatenate([[0], np.cumsum(nnz)]).astype(np.int64)
    cols = np.empty(off[-1], dtype=np.int64)
    vals = np.empty(off[-1])
    cols[off[:-1]] = a
    vals[off[:-1]] = np.where(own, 1.0, 0.5)
    mid = np.where(~own)[0]
    cols[off[mid] + 1] = b[mid]
    vals[off[mid] + 1] = 0.5
    return _canon(sp.csr_matrix((vals, cols, off), shape=(f.nv, c.nv)))


def _p2_shape_values(lam):
    l0, l1, l2 = lam[:, 0], lam[:, 1], lam[:, 2]
    return np.column_stack([l0 * (2 * l0 - 1), l1 * (2 * l1 - 1),
                            l2 * (2 * l2 - 1), 4 * l0 * l1, 4 * l1 * l2,
                            4 * l2 * l0])


def p2_prolongation(kc):
    """Nodal P2 interpolation between nested interior P2 spaces
    (transfer.py:58-97).  Points on a cell diagonal use the lower-right
    triangle (mesh.py:249-263)."""
    c, f = StructuredLevel(kc), StructuredLevel(kc + 1)
    f_int, _ = f.p2_interior()
    _, c_idx = c.p2_interior()
    px, py = f.p2_points()
    px, py = px[f_int], py[f_int]
    h = 1.0 / c.m
    cx = np.clip((px // h).astype(np.int64), 0, c.m - 1)
    cy = np.clip((py // h).astype(np.int64), 0, c.m - 1)
    s = (px - cx * h) / h
    t = (py - cy * h) / h
    upper = t > s
    lam = np.where(upper[:, None],
                   np.column_stack([1.0 - t, s, t - s]),
                   np.column_stack([1.0 - s, s - t, t]))
    w = _p2_shape_values(lam)
    tri = c.triangles()
    te = c.triangle_edges()
    tid = 2 * (cy * c.m + cx) + upper
    dofs = np.hstack([tri[tid], c.nv + te[tid]])
    cols = c_idx[dofs]
    keep = (w != 0.0) & (cols >= 0)
    rows = np.repeat(np.arange(f_int.size), 6).reshape(-1, 6)
    n_c = int((c_idx >= 0).sum())
    p = sp.coo_matrix((w[keep], (rows[keep], cols[keep])),
                      shape=(f_int.size, n_c))
    return _canon(p)


@dataclass
class OracleTransfer:
    P: sp.csr_matrix
    R: sp.csr_matrix


def system_transfer(coarse: OracleSystem, fine: OracleSystem):
    """Block-diagonal per-field transfer, R = P^T (transfer.py:100-143)."""
    kc = coarse.k
    if fine.problem == "poisson":
        p1 = p1_prolongation(kc)
        blocks = [p1, p1]
    else:
        p1, p2 = p1_prolongation(kc), p2_prolongation(kc)
        blocks = [p2, p2, p1, p2, p2, p1]
    P = _canon(sp.block_diag(blocks, format="csr"))
    R = _canon(P.T.tocsr())
    return OracleTransfer(P, R)


# ---------------------------------------------------------------------------
# smoothers (smoothers.py:179-285, kernels.py:17-66)
# ---------------------------------------------------------------------------

DEFAULT_TAU = {"poisson": 0.4, "stokes": 0.35}     # smoothers.py:25-29


class OracleSmoother:
    """Per-level smoother data: CSC mirror, row entries scaled by the
    column weight, normal-equation diagonal (smoothers.py:189-216)."""

    def __init__(self, system: OracleSystem, name="lsgs", tau=None):
        if name not in ("normal", "lsgs", "slsgs", "cgs"):
            raise ValueError(f"oracle smoother '{name}' not in scope")
        if name == "cgs" and system.problem != "poisson":
            raise ValueError("collective sweep needs a scalar control system")
        A = system.A
        self.system, self.name = system, name
        self.tau = tau if tau is not None else DEFAULT_TAU[system.problem]
        self.row_off, self.row_col = A.indptr, A.indices
        self.row_scaled = A.data / system.L[A.indices]
        csc = A.tocsc()
        csc.sort_indices()
        self.col_off = csc.indptr.astype(np.int64)
        self.col_row = csc.indices.astype(np.int64)
        self.col_val = np.ascontiguousarray(csc.data)
        rows = np.repeat(np.arange(system.n), np.diff(A.indptr))
        nd = np.zeros(system.n)
        np.add.at(nd, rows, A.data * self.row_scaled)
        if np.any(nd <= 0.0):
            raise ValueError("operator has an empty row")
        self.n_diag = nd
        self.weight = system.L
        self._update = np.empty(system.n)
        self.op_count = 0
        if name == "cgs":  # smoothers.py:217-219: diag(M), diag(K)
            nn = system.n // 2
            self.mass_diag = np.ascontiguousarray(A[:nn, :nn].diagonal())
            self.stiff_diag = np.ascontiguousarray(A[:nn, nn:].diagonal())

    def _args(self):
        return (self.system.n, _ptr(self.row_off), _ptr(self.row_col),
                _ptr(self.row_scaled), _ptr(self.col_off),
                _ptr(self.col_row), _ptr(self.col_val))

    def normal(self, x, r):
        self.op_count += lib().orc_normal_sweep(
            *self._args(), _ptr(self.weight), self.tau, _ptr(x), _ptr(r),
            _ptr(self._update))
        return x, r

    def lsgs(self, x, r, forward=True):
        self.op_count += lib().orc_lsgs_sweep(
            *self._args(), _ptr(self.n_diag), _ptr(x), _ptr(r),
            1 if forward else 0)
        return x, r

    def cgs(self, x, r):
        """kernels.collective_sweep via smoothers.py:288-295."""
        self.op_count += lib().orc_collective_sweep(
            self.system.n // 2, _ptr(self.col_off), _ptr(self.col_row),
            _ptr(self.col_val), _ptr(self.mass_diag), _ptr(self.stiff_diag),
            float(self.system.alpha), _ptr(x), _ptr(r))
        return x, r

    def sweep(self, x, r):
        """smoothers.py:226-244 for the NE family and CGS."""
        if self.name == "cgs":
            return self.cgs(x, r)
        if self.name == "normal":
            return self.normal(x, r)
        if self.name == "lsgs":
            return self.lsgs(x, r, True)
        self.lsgs(x, r, True)
        return self.lsgs(x, r, False)


def vanka_sweep(offsets, dofs, inverses, sizes, A, tau, x, r, forward=True):
    """kernels.vanka_sweep (kernels.py:99-131): multiplicative patch sweep
    with damping, in patch order (forward) or reversed; the downdate walks
    the column view of A (sparse.py ColumnView: CSC, rows ascending).
    Plain loops (small levels only)."""
    C = A.tocsc()
    C.sort_indices()
    n_patches = offsets.shape[0] - 1
    order = range(n_patches) if forward else range(n_patches - 1, -1, -1)
    ops = 0
    for p in order:
        lo, m = offsets[p], sizes[p]
        local_r = [r[dofs[lo + a]] for a in range(m)]
        local_s = []
        for a in range(m):
            acc = 0.0
            for b in range(m):
                acc += inverses[p, a, b] * local_r[b]
            local_s.append(tau * acc)
        for a in range(m):
            c = dofs[lo + a]
            sv = local_s[a]
            x[c] += sv
            for t in range(C.indptr[c], C.indptr[c + 1]):
                r[C.indices[t]] -= C.data[t] * sv
            ops += C.indptr[c + 1] - C.indptr[c]
    return ops


# ---------------------------------------------------------------------------
# coarse solve, cycle, solve loops (multigrid.py:67-204)
# ---------------------------------------------------------------------------

class OracleCoarse:
    """Dense partial-pivot LU of the coarsest operator; Stokes pins the first
    p and mu dof, projects the RHS and re-centres (multigrid.py:67-102)."""

    def __init__(self, system: OracleSystem):
        if system.n > 5000:
            raise ValueError("coarsest system too large")
        self.system = system
        dense = system.A.toarray()
        self.pinned = []
        if system.problem == "stokes":
            for name in ("pressure", "adjoint_pressure"):
                i = system.slice_of(name).start
                dense[i, :] = 0.0
                dense[:, i] = 0.0
                dense[i, i] = 1.0
                self.pinned.append(i)
        self.lu = scipy.linalg.lu_factor(dense)

    def solve(self, rhs):
        b = np.array(rhs, dtype=np.float64)
        if self.system.problem == "stokes":
            for name in ("pressure", "adjoint_pressure"):
                s = self.system.slice_of(name)
                b[s] -= b[s].mean()
            for i in self.pinned:
                b[i] = 0.0
        x = scipy.linalg.lu_solve(self.lu, b)
        return self.system.mean_project(x)


class OracleMultigrid:
    """V/W cycle over systems[0] (coarsest) .. systems[-1] (finest)
    (multigrid.py:105-159)."""

    def __init__(self, systems, transfers, smoother="lsgs", cycle="v",
                 nu_pre=2, nu_post=2, tau=None):
        self.systems, self.transfers = systems, transfers
        self.cycle_kind, self.nu_pre, self.nu_post = cycle, nu_pre, nu_post
        self.coarse = OracleCoarse(systems[0])
        self.states = [None] + [OracleSmoother(s, smoother, tau)
                                for s in systems[1:]]

    @property
    def finest(self):
        return self.systems[-1]

    def cycle(self, li, x, rhs):
        if li == 0:
            return self.coarse.solve(rhs)
        system, state = self.systems[li], self.states[li]
        tr = self.transfers[li - 1]
        r = system.residual(x, rhs)
        for _ in range(self.nu_pre):
            state.sweep(x, r)
        crhs = csr_matvec(tr.R, r)
        corr = np.zeros(self.systems[li - 1].n)
        for _ in range(1 if self.cycle_kind == "v" else 2):
            corr = self.cycle(li - 1, corr, crhs)
        x += csr_matvec(tr.P, corr)
        system.mean_project(x)
        r = system.residual(x, rhs)
        for _ in range(self.nu_post):
            state.sweep(x, r)
        return x


def build_oracle(problem, k_max, alpha, coarsest=1, **kw):
    """assemble_hierarchy + Multigrid (multigrid.py:207-225)."""
    make = poisson_system if problem == "poisson" else stokes_system
    systems = [make(k, alpha) for k in range(coarsest, k_max + 1)]
    transfers = [system_transfer(c, f)
                 for c, f in zip(systems[:-1], systems[1:])]
    return OracleMultigrid(systems, transfers, **kw)


def baseline_rhs(system: OracleSystem, seed, add_sine=False):
    """BASELINE.json inputs: y_D / v_D ~ U[-1,1] from
    default_rng(seed) in the reference layout (config 3 adds
    sin(pi x) sin(pi y) at the vertices); f = (M y_D, 0)."""
    rng = np.random.default_rng(seed)
    if system.problem == "poisson":
        lvl = StructuredLevel(system.k)
        yd = rng.uniform(-1.0, 1.0, lvl.nv)
        if add_sine:
            x, y = lvl.coords()
            yd = yd + np.sin(np.pi * x) * np.sin(np.pi * y)
        s = system.slice_of("state")
    else:
        s = system.slice_of("velocity")
        yd = rng.uniform(-1.0, 1.0, s.stop - s.start)
    f = np.zeros(system.n)
    f[s] = csr_matvec(system.mass, yd)
    return f


def baseline_solve(mg: OracleMultigrid, f, tol=1e-8, max_cycles=300,
                   keep_iterates=0):
    """x0 = 0; cycle; mean projection; stop at ||f-Ax||_2 <= tol ||f||_2
    (SURVEY.md §3.4).  Returns (x, rel_history, iterates)."""
    sysf = mg.finest
    x = np.zeros(sysf.n)
    nf = float(np.linalg.norm(f))
    hist, its = [], []
    for c in range(max_cycles):
        x = mg.cycle(len(mg.systems) - 1, x, f)
        sysf.mean_project(x)
        rel = float(np.linalg.norm(sysf.residual(x, f))) / nf
        hist.append(rel)
        if c < keep_iterates:
            its.append(x.copy())
        if rel <= tol or not np.isfinite(rel):
            break
    return x, hist, its


def reference_solve(mg: OracleMultigrid, seed=1234, tol=1e-6, max_it=200):
    """Reference protocol: rhs 0, x0 ~ U[-1,1], L-norm drop by tol
    (multigrid.py:161-204).  Returns the norm history."""
    sysf = mg.finest
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, sysf.n)
    sysf.mean_project(x)
    rhs = np.zeros(sysf.n)
    n0 = sysf.norm(x)
    hist = [n0]
    for _ in range(max_it):
        x = mg.cycle(len(mg.systems) - 1, x, rhs)
        sysf.mean_project(x)
        nrm = sysf.norm(x)
        hist.append(nrm)
        if nrm <= tol * n0 or nrm > 1e6 * n0 or not np.isfinite(nrm):
            break
    return hist
