"""Vanka patch smoother: patches and their local
inverses built on the host exactly as the reference builds them
(smoothers.py:87-176, kernels.py:134-151), the multiplicative sweep
(kernels.py:99-131) on the device (``ocmg_vanka_sweep``).

A patch is the velocity / adjoint-velocity dofs at a vertex and on its
incident edges plus the vertex's pressure and adjoint-pressure dofs.  The
local matrices are gathered from the level's operator, diagonally scaled,
inverted with numpy (LAPACK, as the reference) and rescaled, so the inverses
are the reference's bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

# patches x (largest patch)^2 above which the host build is refused (the
# dense inverses alone are 8 bytes each)
MAX_INVERSE_ENTRIES = 300_000_000


@dataclass
class VankaPatches:
    """smoothers.py:62-84: concatenated patch dofs, sizes, padded local
    inverses, and the vertex of each patch."""
    offsets: np.ndarray
    dofs: np.ndarray
    sizes: np.ndarray
    inverses: np.ndarray
    vertex_ids: np.ndarray

    @property
    def n_patches(self):
        return self.sizes.shape[0]

    def dofs_of(self, p):
        return self.dofs[self.offsets[p]:self.offsets[p + 1]]


def _edges(mesh):
    """(ne, 2) sorted vertex pairs in the reference's lexicographic edge
    order (mesh.py:159-166): per lower vertex, horizontal, vertical,
    diagonal -- the numbering of the structured edge table."""
    n1 = mesh.n1
    e = mesh._edge_table
    lo = np.repeat(np.arange(mesh.n_vertices), 3)
    kind = np.tile(np.arange(3), mesh.n_vertices)
    have = e.ravel() >= 0
    hi = lo + np.array([1, n1, n1 + 1])[kind]
    out = np.empty((mesh.n_edges, 2), dtype=np.int64)
    out[e.ravel()[have]] = np.column_stack([lo[have], hi[have]])
    return out


def _vertex_edge_adjacency(mesh, edges):
    """mesh.py:62-70."""
    ne = edges.shape[0]
    both = np.concatenate([edges[:, 0], edges[:, 1]])
    eidx = np.tile(np.arange(ne), 2)
    order = np.argsort(both, kind="stable")
    counts = np.bincount(both, minlength=mesh.n_vertices)
    offsets = np.concatenate([[0], np.cumsum(counts)])
    return offsets, eidx[order]


def _patch_scalars(mesh, p2i):
    """Per vertex, the interior scalar P2 dofs of its patch as a padded
    (nv, 7) matrix (-1 = none) plus the count per vertex.  The order is the
    reference's (smoothers.py:87-176): the vertex's own dof, then its
    incident edges in vertex-edge adjacency order (mesh.py:62-70).  Vertices
    whose vertex and incident-edge dofs are all eliminated (the corners) take
    the interior edge dofs of the triangles around them, in edge order."""
    nv = mesh.n_vertices
    edges = _edges(mesh)
    adj_off, adj_edges = _vertex_edge_adjacency(mesh, edges)
    deg = np.diff(adj_off)
    width = 1 + int(deg.max())
    cand = np.full((nv, width), -1, dtype=np.int64)
    cand[:, 0] = p2i[:nv]
    owner = np.repeat(np.arange(nv), deg)
    cand[owner, 1 + np.arange(adj_edges.size) - adj_off[owner]] = \
        p2i[nv + adj_edges]
    # push the eliminated (-1) entries to the end of each row, keeping order
    keep = cand >= 0
    cand = np.take_along_axis(cand, np.argsort(~keep, axis=1, kind="stable"),
                              axis=1)
    count = keep.sum(axis=1)
    empty = np.flatnonzero(count == 0)
    if empty.size:
        tris, tri_edges = mesh.triangles(), mesh.triangle_edge_ids()
        for v in empty:                       # at most the 4 corners
            around = np.unique(tri_edges[(tris == v).any(axis=1)])
            extra = p2i[nv + around]
            extra = extra[extra >= 0]
            if extra.size > width:
                raise ValueError("corner patch wider than the padding")
            cand[v, :extra.size] = extra
            count[v] = extra.size
    return cand, count


def _patch_dofs(system, cand, count):
    """Concatenated global dofs of all patches, vertex order: [v_x, v_y,
    adjoint v_x, adjoint v_y] over the patch's scalar dofs, then the
    vertex's pressure and adjoint-pressure dofs."""
    lay = system.layout
    n_s = system.n_velocity_scalar
    bases = np.array([lay.offset("velocity"), lay.offset("velocity") + n_s,
                      lay.offset("adjoint_velocity"),
                      lay.offset("adjoint_velocity") + n_s], dtype=np.int64)
    verts = np.flatnonzero(count > 0)
    sizes = 4 * count[verts] + 2
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dofs = np.empty(int(offsets[-1]), dtype=np.int64)
    for c in np.unique(count[verts]):         # one vectorised pass per size
        rows = np.flatnonzero(count[verts] == c)
        v = verts[rows]
        vel = (bases[:, None, None] + cand[v, :c][None]).transpose(1, 0, 2)
        block = np.concatenate(
            [vel.reshape(rows.size, 4 * c),
             (lay.offset("pressure") + v)[:, None],
             (lay.offset("adjoint_pressure") + v)[:, None]], axis=1)
        dofs[offsets[rows][:, None] + np.arange(4 * c + 2)] = block
    return offsets, dofs, sizes.astype(np.int64), verts.astype(np.int64)


def _gather_local(a, offsets, dofs, sizes, mmax):
    """out[p, i, j] = A[dofs_i, dofs_j] (stored entries, else 0), padded to
    mmax (kernels.py:134-151), by batched CSR lookups of all (i, j) pairs of
    equally sized patches."""
    n_p = sizes.size
    out = np.zeros((n_p, mmax, mmax))
    for m in np.unique(sizes):
        rows = np.flatnonzero(sizes == m)
        ii, jj = np.divmod(np.arange(m * m), m)
        step = max(1, 4_000_000 // (m * m))
        for c0 in range(0, rows.size, step):
            rr = rows[c0:c0 + step]
            d = dofs[offsets[rr][:, None] + np.arange(m)]       # (b, m)
            vals = np.asarray(a[d[:, ii].ravel(), d[:, jj].ravel()]).ravel()
            out[rr[:, None], ii, jj] = vals.reshape(rr.size, m * m)
    return out


def build_vanka_patches(system):
    """Vanka patches of a Stokes level and their local inverses
    (smoothers.py:87-176)."""
    if system.problem != "stokes":
        raise ValueError("patches are built for velocity tracking systems")
    mesh = system.mesh
    _, p2i = mesh.p2_interior()
    cand, count = _patch_scalars(mesh, np.asarray(p2i, dtype=np.int64))
    offsets, dofs, sizes, vertex_ids = _patch_dofs(system, cand, count)
    n_patches = sizes.size
    mmax = int(sizes.max())
    if n_patches * mmax * mmax > MAX_INVERSE_ENTRIES:
        raise ValueError(f"{n_patches} patches of up to {mmax} dofs: the "
                         "dense local inverses are too large for this level")
    mats = _gather_local(system.to_scipy().tocsr(), offsets, dofs, sizes,
                         mmax)
    # pad with the identity, then scale -> invert -> rescale; this sequence
    # is the reference's op for op (smoothers.py:155-176), which is what
    # makes the inverses bit-identical
    pad = np.arange(mmax)[None, :] >= sizes[:, None]
    mats[pad[:, :, None] & pad[:, None, :] &
         np.eye(mmax, dtype=bool)[None]] = 1.0
    diag = np.abs(np.einsum("pii->pi", mats))
    scale = 1.0 / np.sqrt(np.where(diag > 0.0, diag, 1.0))
    scaled = mats * scale[:, :, None] * scale[:, None, :]
    try:
        inv = np.linalg.inv(scaled)
    except np.linalg.LinAlgError:
        bad = next(p for p in range(n_patches)
                   if np.linalg.matrix_rank(scaled[p]) < mmax)
        raise _lib.SingularMatrixError(
            f"singular local matrix for patch {bad} "
            f"(vertex {vertex_ids[bad]})") from None
    inverses = inv * scale[:, :, None] * scale[:, None, :]
    finite = np.isfinite(inverses).all(axis=(1, 2))
    if not finite.all():
        bad = int(np.flatnonzero(~finite)[0])
        raise _lib.SingularMatrixError(f"non-finite local inverse for patch "
                                       f"{bad} (vertex {vertex_ids[bad]})")
    return VankaPatches(offsets=offsets, dofs=dofs, sizes=sizes,
                        inverses=inverses, vertex_ids=vertex_ids)


def attach(system, patches):
    """Upload the patches to the level (ocmg_level_set_vanka): dofs, padded
    inverses and the dependency schedule of the multiplicative sweep."""
    off = np.ascontiguousarray(patches.offsets, dtype=np.int64)
    dofs = np.ascontiguousarray(patches.dofs, dtype=np.int64)
    inv = np.ascontiguousarray(patches.inverses, dtype=np.float64)
    _lib.call("ocmg_level_set_vanka", system.handle, int(patches.n_patches),
              int(inv.shape[1]), _lib.hptr(off), _lib.hptr(dofs), _lib.hptr(inv))
