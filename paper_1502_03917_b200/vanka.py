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


def build_vanka_patches(system):
    """smoothers.py:87-176."""
    if system.problem != "stokes":
        raise ValueError("patches are built for velocity tracking systems")
    mesh = system.mesh
    layout = system.layout
    _, p2i = mesh.p2_interior()
    n_s = system.n_velocity_scalar
    off_v = layout.offset("velocity")
    off_p = layout.offset("pressure")
    off_av = layout.offset("adjoint_velocity")
    off_ap = layout.offset("adjoint_pressure")
    nv = mesh.n_vertices
    edges = _edges(mesh)
    adj_off, adj_edges = _vertex_edge_adjacency(mesh, edges)
    tris = mesh.triangles()
    tri_edges = mesh.triangle_edge_ids()

    offsets = [0]
    dofs = []
    vertex_ids = []
    for v in range(nv):
        scalar = []
        if p2i[v] >= 0:
            scalar.append(p2i[v])
        for e in adj_edges[adj_off[v]:adj_off[v + 1]]:
            idx = p2i[nv + e]
            if idx >= 0:
                scalar.append(idx)
        if not scalar:
            # corners whose incident edges are all on the boundary: the
            # interior edge midpoints of the triangles at the vertex
            t = np.where((tris == v).any(axis=1))[0]
            for e in np.unique(tri_edges[t]):
                idx = p2i[nv + e]
                if idx >= 0:
                    scalar.append(idx)
        if not scalar:
            continue
        patch = []
        for base in (off_v, off_av):
            patch.extend(base + i for i in scalar)
            patch.extend(base + n_s + i for i in scalar)
        patch.append(off_p + v)
        patch.append(off_ap + v)
        dofs.extend(patch)
        offsets.append(len(dofs))
        vertex_ids.append(v)

    offsets = np.asarray(offsets, dtype=np.int64)
    dofs = np.asarray(dofs, dtype=np.int64)
    sizes = np.diff(offsets)
    vertex_ids = np.asarray(vertex_ids, dtype=np.int64)
    n_patches = sizes.shape[0]
    mmax = int(sizes.max())
    if n_patches * mmax * mmax > MAX_INVERSE_ENTRIES:
        raise ValueError(f"{n_patches} patches of up to {mmax} dofs: the "
                         "dense local inverses are too large for this level")

    # gather_patch_matrices (kernels.py:134-151): out[p, a, b] = A[dofs_a,
    # dofs_b] for the stored entries, in chunks of patches
    a = system.to_scipy()
    mats = np.zeros((n_patches, mmax, mmax))
    chunk = max(1, 4_000_000 // (mmax * mmax))
    for p0 in range(0, n_patches, chunk):
        p1 = min(n_patches, p0 + chunk)
        for p in range(p0, p1):
            d = dofs[offsets[p]:offsets[p + 1]]
            m = d.size
            mats[p, :m, :m] = a[d][:, d].toarray()

    # smoothers.py:155-176: identity padding, symmetric diagonal scaling,
    # inversion, rescaling
    for p in range(n_patches):
        mats[p, sizes[p]:, sizes[p]:] = np.eye(mmax - sizes[p])
    diag = np.abs(np.einsum("pii->pi", mats))
    scale = 1.0 / np.sqrt(np.where(diag > 0.0, diag, 1.0))
    scaled = mats * scale[:, :, None] * scale[:, None, :]
    try:
        inv = np.linalg.inv(scaled)
    except np.linalg.LinAlgError:
        for p in range(n_patches):
            try:
                np.linalg.inv(scaled[p])
            except np.linalg.LinAlgError:
                raise _lib.SingularMatrixError(
                    f"singular local matrix for patch {p} "
                    f"(vertex {vertex_ids[p]})") from None
        raise
    inverses = inv * scale[:, :, None] * scale[:, None, :]
    if not np.all(np.isfinite(inverses)):
        bad = np.where(~np.isfinite(inverses).all(axis=(1, 2)))[0][0]
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
