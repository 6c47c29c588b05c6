"""Grid transfers between consecutive nested levels (transfer.py:1-143).

Prolongation is the exact embedding of the coarse finite element space;
restriction is its transpose (scale 1).  Poisson control uses the structured
block-P1 kernels (no matrix stored); Stokes control uploads the block
diagonal [P2, P2, P1, P2, P2, P1] as a CSR and the device builds R = P^T.
"""
from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._vec import as_device, back, zeros
from .assembly import _Handle, _canonical
from .mesh import StructuredMesh

__all__ = ["TransferPair", "p1_prolongation", "p2_prolongation",
           "system_transfer"]


def p1_prolongation(coarse: StructuredMesh, fine: StructuredMesh):
    """Linear interpolation (transfer.py:34-55): a fine vertex on a coarse
    vertex copies it, an edge midpoint averages the two ends."""
    if fine.level != coarse.level + 1:
        raise ValueError("meshes are not consecutive refinement levels")
    fy, fx = np.divmod(np.arange(fine.n_vertices), fine.n1)
    ox, oy = fx & 1, fy & 1
    a = (fy >> 1) * coarse.n1 + (fx >> 1)
    b = ((fy >> 1) + oy) * coarse.n1 + (fx >> 1) + ox
    mid = (ox | oy).astype(bool)
    rows = np.concatenate([np.arange(fine.n_vertices), np.flatnonzero(mid)])
    cols = np.concatenate([a, b[mid]])
    vals = np.concatenate([np.where(mid, 0.5, 1.0), np.full(mid.sum(), 0.5)])
    return _canonical(sp.coo_matrix((vals, (rows, cols)),
                                    shape=(fine.n_vertices,
                                           coarse.n_vertices)))


def p2_prolongation(coarse: StructuredMesh, fine: StructuredMesh):
    """Nodal P2 interpolation between interior P2 spaces (transfer.py:58-97);
    points on a cell diagonal use the lower-right coarse triangle
    (mesh.py:249-263).  All weights are dyadic, hence exact."""
    if fine.level != coarse.level + 1:
        raise ValueError("meshes are not consecutive refinement levels")
    f_keep, _ = fine.p2_interior()
    _, c_pos = coarse.p2_interior()
    px, py = fine.p2_points()
    px, py = px[f_keep], py[f_keep]
    h = coarse.h
    cx = np.clip((px // h).astype(np.int64), 0, coarse.m - 1)
    cy = np.clip((py // h).astype(np.int64), 0, coarse.m - 1)
    s, t = (px - cx * h) / h, (py - cy * h) / h
    upper = t > s
    l0 = np.where(upper, 1.0 - t, 1.0 - s)
    l1 = np.where(upper, s, s - t)
    l2 = np.where(upper, t - s, t)
    w = np.column_stack([l0 * (2 * l0 - 1), l1 * (2 * l1 - 1),
                         l2 * (2 * l2 - 1), 4 * l0 * l1, 4 * l1 * l2,
                         4 * l2 * l0])
    tri = coarse.triangles()
    te = coarse.triangle_edge_ids()
    tid = 2 * (cy * coarse.m + cx) + upper
    cols = c_pos[np.hstack([tri[tid], coarse.n_vertices + te[tid]])]
    keep = (w != 0.0) & (cols >= 0)
    rows = np.broadcast_to(np.arange(f_keep.size)[:, None], w.shape)
    n_c = int((c_pos >= 0).sum())
    return _canonical(sp.coo_matrix((w[keep], (rows[keep], cols[keep])),
                                    shape=(f_keep.size, n_c)))


class _Operator:
    """Device action of P (prolongation) or R = P^T (restriction) with the
    reference's SparseMatrix-like surface (shape, matvec)."""

    def __init__(self, pair, which):
        self._pair, self._which = pair, which

    @property
    def shape(self):
        nf, nc = self._pair.n_fine, self._pair.n_coarse
        return (nf, nc) if self._which == "P" else (nc, nf)

    @property
    def nrows(self):
        return self.shape[0]

    @property
    def ncols(self):
        return self.shape[1]

    def matvec(self, x):
        xd, was_np = as_device(x, self.ncols)
        if self._which == "P":
            y = zeros(self.nrows)
            self._pair.prolong_add(xd, y)
        else:
            import torch
            y = torch.empty(self.nrows, dtype=torch.float64, device="cuda")
            self._pair.restrict(xd, y)
        return back(y, was_np)

    def to_scipy(self):
        P = self._pair.host_prolongation()
        return P if self._which == "P" else _canonical(P.T)


class TransferPair:
    """Prolongation and its exact transpose (transfer.py:22-31)."""

    def __init__(self, handle, n_fine, n_coarse, host_builder):
        self._h = handle
        self.n_fine, self.n_coarse = n_fine, n_coarse
        self._host_builder = host_builder
        self.prolongation = _Operator(self, "P")
        self.restriction = _Operator(self, "R")

    @property
    def handle(self):
        return self._h.ptr

    def host_prolongation(self):
        return self._host_builder()

    def restrict(self, rf, rc):
        """rc = R rf on the device (multigrid.py:148)."""
        _lib.call("ocmg_restrict", self.handle, _lib.dptr(rf), _lib.dptr(rc),
                  _lib.stream_ptr())

    def prolong_add(self, c, xf):
        """xf += P c on the device (multigrid.py:153)."""
        _lib.call("ocmg_prolong_add", self.handle, _lib.dptr(c),
                  _lib.dptr(xf), _lib.stream_ptr())


def _block_host(layout, per_field):
    blocks = []
    for kind, p in zip(layout.kinds, per_field):
        blocks.extend([p, p] if kind == "p2" else [p])
    return _canonical(sp.block_diag(blocks, format="csr"))


def system_transfer(coarse_system, fine_system):
    """Transfer pair for two consecutive assembled systems
    (transfer.py:135-143)."""
    if coarse_system.problem != fine_system.problem:
        raise ValueError("systems solve different problems")
    cm, fm = coarse_system.mesh, fine_system.mesh
    if fm.level != cm.level + 1:
        raise ValueError("meshes are not consecutive refinement levels")
    if fine_system.problem == "poisson":
        h = _lib.new_handle()
        _lib.call("ocmg_transfer_create_p1", cm.level, 2, ctypes.byref(h))

        def host():
            p = p1_prolongation(cm, fm)
            return _canonical(sp.block_diag([p, p], format="csr"))
        return TransferPair(_Handle(h, "ocmg_transfer_destroy"),
                            fine_system.n, coarse_system.n, host)
    p1 = p1_prolongation(cm, fm)
    p2 = p2_prolongation(cm, fm)
    P = _block_host(fine_system.layout, [p2, p1, p2, p1])
    if P.shape != (fine_system.n, coarse_system.n):
        raise ValueError("transfer does not match the system layouts")
    off = np.ascontiguousarray(P.indptr, dtype=np.int64)
    col = np.ascontiguousarray(P.indices, dtype=np.int64)
    val = np.ascontiguousarray(P.data, dtype=np.float64)
    h = _lib.new_handle()
    _lib.call("ocmg_transfer_create_csr", P.shape[0], P.shape[1],
              _lib.hptr(off), _lib.hptr(col), _lib.hptr(val), ctypes.byref(h))
    return TransferPair(_Handle(h, "ocmg_transfer_destroy"), fine_system.n,
                        coarse_system.n, lambda: P)
