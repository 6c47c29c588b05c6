"""Block systems of the two control problems, device-backed (host setup).

Reference: assembly.py (element matrices 22-183, Taylor-Hood elimination
186-201, FieldLayout 205-226, BlockSystem 229-267, builders 270-341,
pressure_mean_projection 381-388).

Poisson control, k >= 3, is held on the device as position-class stencil
tables (``p1_class_tables``): the operator never exists as a CSR at large
levels (L12 would need ~470M stored entries).  The tables reproduce the
reference's assembled values bit for bit: the 9 row classes are read off a
level-3 assembly done in the reference's element order, mass entries scale
exactly by powers of two across levels, and every derived quantity (K =
Laplace + mass, -M/alpha, L, row_scaled, n_diag) is formed with the same
floating-point operations the reference performs.  Stokes control and the
tiny Poisson levels go through a host CSR with the same conventions.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np
import scipy.sparse as sp

from . import _lib
from .mesh import StructuredMesh

__all__ = ["FieldLayout", "BlockSystem", "build_poisson_system",
           "build_stokes_system", "pressure_mean_projection",
           "assemble_p1", "assemble_taylor_hood", "p1_class_tables"]

STRUCTURED_MIN_LEVEL = 3


# ---------------------------------------------------------------------------
# layout
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class FieldLayout:
    """Ordered fields with global offsets (assembly.py:205-226)."""

    names: tuple
    counts: tuple
    kinds: tuple

    @property
    def n(self):
        return int(sum(self.counts))

    def offset(self, name):
        return int(sum(self.counts[:self.names.index(name)]))

    def slice_of(self, name):
        off = self.offset(name)
        return slice(off, off + self.counts[self.names.index(name)])

    def offsets(self):
        return np.concatenate([[0], np.cumsum(self.counts)]).astype(np.int64)


# ---------------------------------------------------------------------------
# element matrices
# ---------------------------------------------------------------------------

def _canonical(m):
    c = m.tocsr().copy()
    c.sum_duplicates()
    c.sort_indices()
    c.eliminate_zeros()
    return c


def _triangle_pair(h):
    """The two congruent triangles of the pattern (lower-right, upper-left)."""
    return ([(0, 0), (h, 0), (h, h)], [(0, 0), (h, h), (0, h)])


def _p1_element(pts):
    """P1 mass and pure-Laplace stiffness of a triangle, in the reference's
    floating-point form (assembly.py:97-118)."""
    (x0, y0), (x1, y1), (x2, y2) = [(float(a), float(b)) for a, b in pts]
    b = np.array([y1 - y2, y2 - y0, y0 - y1])
    c = np.array([x2 - x1, x0 - x2, x1 - x0])
    area = 0.5 * ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0))
    mass = (np.ones((3, 3)) + np.eye(3)) * (area / 12.0)
    lap = (b[:, None] * b[None, :] + c[:, None] * c[None, :]) / (4.0 * area)
    return mass, lap


def _scatter(row_dofs, col_dofs, per_type, shape):
    """Element-by-element COO scatter (triangle order, local row-major), then
    CSR; duplicates are summed by scipy exactly as in the reference."""
    nt, a = row_dofs.shape
    b = col_dofs.shape[1]
    vals = np.empty((nt, a * b))
    vals[0::2] = per_type[0].reshape(1, -1)
    vals[1::2] = per_type[1].reshape(1, -1)
    rows = np.repeat(row_dofs, b, axis=1).ravel()
    cols = np.tile(col_dofs, (1, a)).ravel()
    return sp.coo_matrix((vals.ravel(), (rows, cols)), shape=shape).tocsr()


def assemble_p1(mesh: StructuredMesh):
    """(M, K) with K = Laplace + mass (assembly.py:121-131), canonical CSR."""
    tri = mesh.triangles()
    lo, up = _triangle_pair(mesh.h)
    m_lo, l_lo = _p1_element(lo)
    m_up, l_up = _p1_element(up)
    shape = (mesh.n_vertices, mesh.n_vertices)
    mass = _scatter(tri, tri, (m_lo, m_up), shape)
    lap = _scatter(tri, tri, (l_lo, l_up), shape)
    return _canonical(mass), _canonical(lap + mass)


def _p2_element_exact(pts):
    """Taylor-Hood element blocks in closed form with exact rationals, rounded
    once: P2 mass, P2 Laplace, and the P1 x P2 negative divergence (x, y).
    Local P2 order: vertices 0,1,2 then midpoints of edges (0,1), (1,2),
    (2,0) (assembly.py:39-66).  The reference integrates the same
    polynomials with a degree-4 rule (assembly.py:22-36, 134-183)."""
    P = [(Fraction(x), Fraction(y)) for x, y in pts]
    (x0, y0), (x1, y1), (x2, y2) = P
    det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    A = det / 2
    gx = [(y1 - y2) / det, (y2 - y0) / det, (y0 - y1) / det]
    gy = [(x2 - x1) / det, (x0 - x2) / det, (x1 - x0) / det]
    g = [[gx[i] * gx[j] + gy[i] * gy[j] for j in range(3)] for i in range(3)]

    def I2(i, j):                       # integral of lambda_i lambda_j
        return A / 6 if i == j else A / 12
    edges = ((0, 1), (1, 2), (2, 0))
    opposite = {0: 1, 1: 2, 2: 0}       # vertex -> index of opposite edge
    M = [[Fraction(0)] * 6 for _ in range(6)]
    S = [[Fraction(0)] * 6 for _ in range(6)]
    for i in range(3):
        for j in range(3):
            M[i][j] = A / 180 * (6 if i == j else -1)
            S[i][j] = A * g[i][j] * (1 if i == j else Fraction(-1, 3))
        for e, (a, b) in enumerate(edges):
            M[i][3 + e] = M[3 + e][i] = (A / 180 * -4 if opposite[i] == e
                                         else Fraction(0))
            s = Fraction(0)
            if i == a:
                s = 4 * A / 3 * g[i][b]
            elif i == b:
                s = 4 * A / 3 * g[i][a]
            S[i][3 + e] = S[3 + e][i] = s
    for e, (i, j) in enumerate(edges):
        for f, (k, l) in enumerate(edges):
            M[3 + e][3 + f] = A / 180 * (32 if e == f else 16)
            S[3 + e][3 + f] = 16 * (g[i][k] * I2(j, l) + g[i][l] * I2(j, k)
                                    + g[j][k] * I2(i, l) + g[j][l] * I2(i, k))
    Dx = [[Fraction(0)] * 6 for _ in range(3)]
    Dy = [[Fraction(0)] * 6 for _ in range(3)]
    for p in range(3):
        for i in range(3):
            if p == i:
                Dx[p][i] = -gx[i] * A / 3
                Dy[p][i] = -gy[i] * A / 3
        for e, (i, j) in enumerate(edges):
            Dx[p][3 + e] = -4 * (gx[i] * I2(p, j) + gx[j] * I2(p, i))
            Dy[p][3 + e] = -4 * (gy[i] * I2(p, j) + gy[j] * I2(p, i))
    f = np.vectorize(float)
    return f(np.array(M)), f(np.array(S)), f(np.array(Dx)), f(np.array(Dy))


def assemble_taylor_hood(mesh: StructuredMesh):
    """(mass, laplace, D) on the interior P2 dofs; D = [Dx | Dy] maps the
    two-component interior velocity to the P1 pressures
    (assembly.py:186-201)."""
    tri = mesh.triangles()
    p2 = np.hstack([tri, mesh.n_vertices + mesh.triangle_edge_ids()])
    lo, up = _triangle_pair(Fraction(1, mesh.m))
    e_lo, e_up = _p2_element_exact(lo), _p2_element_exact(up)
    n2 = mesh.n_vertices + mesh.n_edges
    full = [_scatter(p2, p2, (e_lo[0], e_up[0]), (n2, n2)),
            _scatter(p2, p2, (e_lo[1], e_up[1]), (n2, n2))]
    dx = _scatter(tri, p2, (e_lo[2], e_up[2]), (mesh.n_vertices, n2))
    dy = _scatter(tri, p2, (e_lo[3], e_up[3]), (mesh.n_vertices, n2))
    keep, _ = mesh.p2_interior()
    mass = _canonical(full[0][keep][:, keep])
    lap = _canonical(full[1][keep][:, keep])
    div = _canonical(sp.hstack([dx[:, keep], dy[:, keep]]))
    return mass, lap, div


# ---------------------------------------------------------------------------
# P1 position-class tables (structured device path)
# ---------------------------------------------------------------------------

_OFF7 = ((-1, -1), (0, -1), (-1, 0), (0, 0), (1, 0), (0, 1), (1, 1))
_LOW9 = ((-2, -2), (-1, -2), (0, -2), (-2, -1), (-1, -1), (0, -1), (1, -1),
         (-2, 0), (-1, 0))
_REP = (0, 1, 2, 4, 6, 7, 8)     # axis class -> coordinate on the 9x9 grid
_REP_K = 3


@lru_cache(maxsize=1)
def _rep_blocks():
    mesh = StructuredMesh(_REP_K)
    tri = mesh.triangles()
    lo, up = _triangle_pair(mesh.h)
    m_lo, l_lo = _p1_element(lo)
    m_up, l_up = _p1_element(up)
    shape = (mesh.n_vertices, mesh.n_vertices)
    mass = _canonical(_scatter(tri, tri, (m_lo, m_up), shape)).toarray()
    lap = _scatter(tri, tri, (l_lo, l_up), shape)
    lap.sum_duplicates()
    return mass, lap.toarray()


def p1_class_tables(k, alpha):
    """Stencil tables of level k (layout in csrc/ocmg_p1.cuh and
    csrc/ocmg_wavefront.cuh), bit-identical to the reference's CSR values."""
    if k < _REP_K:
        raise ValueError("structured tables need k >= 3")
    M3, LAP3 = _rep_blocks()
    n1 = 2 ** _REP_K + 1
    scale = 4.0 ** (_REP_K - k)          # h^2 scaling, exact
    sa = float(np.sqrt(alpha))
    ia = 1 / alpha                       # scipy divides by multiplying

    def vid(ix, iy):
        if 0 <= ix < n1 and 0 <= iy < n1:
            return iy * n1 + ix
        return None

    def m(v, u):
        return M3[v, u] * scale

    def kk(v, u):
        return LAP3[v, u] + M3[v, u] * scale

    def L(v):
        w = m(v, v) + kk(v, v) * sa
        return (w, w / alpha)

    A = np.zeros((49, 2, 14))
    W = np.zeros((49, 2, 14))
    Lt = np.zeros((49, 2))
    ND = np.zeros((49, 2))
    WF = np.zeros((49, 38))
    for c in range(49):
        cy, cx = divmod(c, 7)
        ix, iy = _REP[cx], _REP[cy]
        v = vid(ix, iy)
        nbrs = [vid(ix + dx, iy + dy) for dx, dy in _OFF7]
        for d, u in enumerate(nbrs):
            if u is None:
                continue
            A[c, 0, d], A[c, 0, 7 + d] = m(v, u), kk(v, u)
            A[c, 1, d], A[c, 1, 7 + d] = kk(v, u), (-m(v, u)) * ia
            Lu = L(u)
            for b in range(2):
                W[c, b, d] = A[c, b, d] / Lu[0]
                W[c, b, 7 + d] = A[c, b, 7 + d] / Lu[1]
        Lt[c] = L(v)
        for b in range(2):
            acc = 0.0
            for t in range(14):
                if nbrs[t % 7] is not None:
                    acc += A[c, b, t] * W[c, b, t]
            ND[c, b] = acc

        # delta-form normal-equation coefficients N = A^T L^-1 A
        def n_entry(u, field):
            if u is None:
                return 0.0
            s = 0.0
            for dx, dy in _OFF7:
                w = vid(ix + dx, iy + dy)
                if w is None or abs((u % n1) - (w % n1)) > 1 \
                        or abs((u // n1) - (w // n1)) > 1:
                    continue
                du = ((u % n1) - (w % n1), (u // n1) - (w // n1))
                if du not in _OFF7:
                    continue
                Lw = L(w)
                if field == 0:
                    s += m(w, v) * m(w, u) / Lw[0] + kk(w, v) * kk(w, u) / Lw[1]
                else:
                    s += (kk(w, v) * kk(w, u) / Lw[0]
                          + ((-m(w, v)) * ia) * ((-m(w, u)) * ia) / Lw[1])
            return s
        for j, (dx, dy) in enumerate(_LOW9):
            lo_u = vid(ix + dx, iy + dy)
            up_u = vid(ix - dx, iy - dy)
            WF[c, j] = n_entry(lo_u, 0)
            WF[c, 9 + j] = n_entry(lo_u, 1)
            WF[c, 18 + j] = n_entry(up_u, 0)
            WF[c, 27 + j] = n_entry(up_u, 1)
        WF[c, 36] = 1.0 / ND[c, 0]
        WF[c, 37] = 1.0 / ND[c, 1]
    out = np.concatenate([A.ravel(), W.ravel(), Lt.ravel(), ND.ravel(),
                          WF.ravel()])
    assert out.size == _lib.P1_TABLE_DOUBLES + _lib.WF_TABLE_DOUBLES
    return out


def p1_norm_diag(k, alpha):
    """Full norm_diag vector of a structured level (host, from the tables)."""
    t = p1_class_tables(k, alpha)
    Lt = t[49 * 56:49 * 56 + 98].reshape(49, 2)
    n1 = 2 ** k + 1
    ax = np.full(n1, 3)
    ax[:3] = [0, 1, 2]
    ax[-3:] = [4, 5, 6]
    c = (7 * ax[:, None] + ax[None, :]).ravel()
    return np.concatenate([Lt[c, 0], Lt[c, 1]])


# ---------------------------------------------------------------------------
# device-backed block system
# ---------------------------------------------------------------------------

class _Handle:
    """Owns a C handle; destroyed with the Python object."""

    def __init__(self, ptr, destroy):
        self.ptr, self._destroy = ptr, destroy

    def __del__(self):
        try:
            if self.ptr:
                getattr(_lib.load(), self._destroy)(self.ptr)
        except Exception:
            pass


class BlockSystem:
    """One level of an all-at-once control system (assembly.py:229-267).

    ``matrix`` (host scipy CSR) exists for CSR-backed levels and on request
    (``to_scipy()``) for small structured ones; the device operator is
    ``handle``.  Vectors are CUDA fp64 tensors in the reference layout;
    numpy arrays are accepted and copied through (drop-in convenience).
    """

    def __init__(self, *, problem, level, alpha, layout, handle, structured,
                 mesh, matrix=None, norm_diag=None, mass=None,
                 n_velocity_scalar=None):
        self.problem = problem
        self.level = level
        self.alpha = float(alpha)
        self.layout = layout
        self._h = handle
        self.structured = structured
        self.mesh = mesh
        self.matrix = matrix
        self._norm_diag = norm_diag
        self.mass = mass
        self.n_velocity_scalar = n_velocity_scalar

    @property
    def handle(self):
        return self._h.ptr

    @property
    def n(self):
        return self.layout.n

    @property
    def nnz(self):
        return int(_lib.load().ocmg_level_nnz(self.handle))

    @property
    def norm_diag(self):
        if self._norm_diag is None and self.structured:
            self._norm_diag = p1_norm_diag(self.level, self.alpha)
        return self._norm_diag

    def to_scipy(self):
        if self.matrix is None:
            if self.level > 10:
                raise ValueError("refusing to materialise a CSR above level 10")
            self.matrix = _poisson_csr(StructuredMesh(self.level), self.alpha)[0]
        return self.matrix

    def residual(self, x, rhs=None):
        """r = rhs - A x (assembly.py:259-263), on the device."""
        from ._vec import as_device, back
        xd, was_np = as_device(x, self.n)
        fd = as_device(rhs, self.n)[0] if rhs is not None else None
        import torch
        r = torch.empty_like(xd)
        _lib.call("ocmg_residual", self.handle, _lib.dptr(xd),
                  _lib.dptr(fd), _lib.dptr(r), _lib.stream_ptr())
        return back(r, was_np)

    def norm(self, x):
        """sqrt(sum L_i x_i^2) (assembly.py:265-267)."""
        from ._vec import as_device, device_scalar
        xd, _ = as_device(x, self.n)
        out = device_scalar()
        _lib.call("ocmg_norm2", self.handle, _lib.dptr(xd), 1,
                  _lib.dptr(out), _lib.stream_ptr())
        return float(np.sqrt(out.item()))


def _poisson_csr(mesh, alpha):
    mass, stiff = assemble_p1(mesh)
    a = sp.bmat([[mass, stiff], [stiff, -mass / alpha]], format="csr")
    w = mass + np.sqrt(alpha) * stiff
    wd = w.diagonal()
    return _canonical(a), np.concatenate([wd, wd / alpha]), mass


def build_poisson_system(level, alpha):
    """Poisson control [[M, K], [K, -M/alpha]] (assembly.py:270-290)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    _lib.require_cuda()
    mesh = StructuredMesh(level)
    nv = mesh.n_vertices
    layout = FieldLayout(("state", "adjoint"), (nv, nv), ("p1", "p1"))
    if level >= STRUCTURED_MIN_LEVEL:
        tab = np.ascontiguousarray(p1_class_tables(level, alpha))
        h = _lib.new_handle()
        _lib.call("ocmg_level_create_p1", int(level), float(alpha),
                  _lib.hptr(tab), tab.size, ctypes.byref(h))
        return BlockSystem(problem="poisson", level=level, alpha=alpha,
                           layout=layout,
                           handle=_Handle(h, "ocmg_level_destroy"),
                           structured=True, mesh=mesh)
    a, L, mass = _poisson_csr(mesh, alpha)
    h = _create_csr_level(_lib.POISSON, a, L, layout, 0)
    # the control weight itself (the CGS 2x2 solve divides by it)
    _lib.call("ocmg_level_set_alpha", h.ptr, float(alpha))
    return BlockSystem(problem="poisson", level=level, alpha=alpha,
                       layout=layout, handle=h, structured=False, mesh=mesh,
                       matrix=a, norm_diag=L, mass=mass)


# generic levels get a greedy distance-2 colouring (multicolour NE-GS) up to
# this many rows (host time grows with nnz x row length: ~6 s for the 18.9M
# rows of Stokes L10)
COLOURING_MAX_ROWS = 25_000_000


def _create_csr_level(problem, a, L, layout, pmask, colouring=True):
    off = np.ascontiguousarray(a.indptr, dtype=np.int64)
    col = np.ascontiguousarray(a.indices, dtype=np.int64)
    val = np.ascontiguousarray(a.data, dtype=np.float64)
    Ld = np.ascontiguousarray(L, dtype=np.float64)
    fo = layout.offsets()
    h = _lib.new_handle()
    _lib.call("ocmg_level_create_csr", problem, a.shape[0], _lib.hptr(off),
              _lib.hptr(col), _lib.hptr(val), _lib.hptr(Ld),
              len(layout.counts), _lib.hptr(fo), pmask,
              1 if (colouring and a.shape[0] <= COLOURING_MAX_ROWS) else 0,
              ctypes.byref(h))
    return _Handle(h, "ocmg_level_destroy")


def build_stokes_system(level, alpha):
    """Stokes velocity tracking, Taylor-Hood (assembly.py:293-341)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if level < 1:
        raise ValueError("velocity tracking needs mesh level >= 1")
    _lib.require_cuda()
    mesh = StructuredMesh(level)
    ms, ks, d = assemble_taylor_hood(mesh)
    mv = sp.block_diag([ms, ms], format="csr")
    kv = sp.block_diag([ks, ks], format="csr")
    dt = d.T.tocsr()
    a = _canonical(sp.bmat([[mv, None, kv, dt], [None, None, d, None],
                            [kv, dt, -mv / alpha, None],
                            [d, None, None, None]], format="csr"))
    ws = ms + np.sqrt(alpha) * ks
    w_hat = np.concatenate([ws.diagonal(), ws.diagonal()])
    winv = 1.0 / w_hat
    rows = np.repeat(np.arange(d.shape[0]), np.diff(d.indptr))
    tri = np.zeros(d.shape[0])
    np.add.at(tri, rows, d.data ** 2 * winv[d.indices])   # sparse.py:239-255
    p_hat = alpha * tri
    n_int, n_p = ms.shape[0], mesh.n_vertices
    layout = FieldLayout(("velocity", "pressure", "adjoint_velocity",
                          "adjoint_pressure"),
                         (2 * n_int, n_p, 2 * n_int, n_p),
                         ("p2", "p1", "p2", "p1"))
    L = np.concatenate([w_hat, p_hat, w_hat / alpha, p_hat / alpha])
    h = _create_csr_level(_lib.STOKES, a, L, layout, 0b1010)
    return BlockSystem(problem="stokes", level=level, alpha=alpha,
                       layout=layout, handle=h, structured=False, mesh=mesh,
                       matrix=a, norm_diag=L, mass=_canonical(mv),
                       n_velocity_scalar=n_int)


def pressure_mean_projection(system, x):
    """Remove the constant modes of both pressure fields in place
    (assembly.py:381-388); no-op for Poisson."""
    if system.problem != "stokes":
        return x
    from ._vec import as_device, back_inplace
    xd, was_np = as_device(x, system.n)
    _lib.call("ocmg_mean_project", system.handle, _lib.dptr(xd),
              _lib.stream_ptr())
    back_inplace(xd, x, was_np)
    return x
