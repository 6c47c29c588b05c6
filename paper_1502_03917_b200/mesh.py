"""Structured unit-square levels and their dof numbering (host setup).

Level k: (2^k+1)^2 vertices, h = 2^-k, every cell split along its SW-NE
diagonal; vertex (ix, iy) has index iy*(2^k+1)+ix (mesh.py:139-180).  The
numbering here is the reference's, so device vectors use the reference's
global layout unchanged.  P2 dofs are the vertices followed by the edges in
lexicographic (lo, hi) order -- per lower vertex: horizontal, vertical,
diagonal (mesh.py:159-166, 273-281) -- with boundary dofs eliminated.
"""
from __future__ import annotations

from functools import cached_property

import numpy as np

MAX_LEVEL = 14   # the reference stops at 9 (mesh.py:16); device levels go further


class StructuredMesh:
    """Geometry and numbering of one level (no per-triangle arrays kept)."""

    def __init__(self, level: int):
        if not 0 <= level <= MAX_LEVEL:
            raise ValueError(f"level must be in [0, {MAX_LEVEL}], got {level}")
        self.level = int(level)
        self.m = 2 ** self.level
        self.n1 = self.m + 1

    @property
    def h(self):
        return 2.0 ** (-self.level)

    @property
    def n_vertices(self):
        return self.n1 * self.n1

    def vertex_xy(self):
        t = np.linspace(0.0, 1.0, self.n1)
        return np.tile(t, self.n1), np.repeat(t, self.n1)

    # -- triangles: cells x-fastest, lower-right (v00,v10,v11) then
    #    upper-left (v00,v11,v01) ------------------------------------------
    def triangles(self):
        m, n1 = self.m, self.n1
        v00 = (np.arange(m)[None, :] + n1 * np.arange(m)[:, None]).ravel()
        out = np.empty((2 * m * m, 3), dtype=np.int64)
        out[0::2, 0], out[0::2, 1], out[0::2, 2] = v00, v00 + 1, v00 + n1 + 1
        out[1::2, 0], out[1::2, 1], out[1::2, 2] = v00, v00 + n1 + 1, v00 + n1
        return out

    # -- edges ---------------------------------------------------------------
    @cached_property
    def _edge_table(self):
        """(n_vertices, 3) edge id of the horizontal / vertical / diagonal
        edge whose lower end is the vertex, -1 where it does not exist."""
        m = self.m
        iy, ix = np.divmod(np.arange(self.n_vertices), self.n1)
        present = np.column_stack([ix < m, iy < m, (ix < m) & (iy < m)])
        ids = np.cumsum(present.ravel()) - 1
        return np.where(present.ravel(), ids, -1).reshape(-1, 3)

    @property
    def n_edges(self):
        return 3 * self.m * self.m + 2 * self.m

    def triangle_edge_ids(self):
        """Edge ids of local edges (0,1), (1,2), (2,0) per triangle."""
        e = self._edge_table
        tri = self.triangles()
        out = np.empty_like(tri)
        lo, up = tri[0::2], tri[1::2]
        out[0::2] = np.column_stack([e[lo[:, 0], 0], e[lo[:, 1], 1],
                                     e[lo[:, 0], 2]])
        out[1::2] = np.column_stack([e[up[:, 0], 2], e[up[:, 2], 0],
                                     e[up[:, 0], 1]])
        return out

    def p2_dirichlet_mask(self):
        """True for P2 dofs (vertices, then edges) on the boundary."""
        m = self.m
        iy, ix = np.divmod(np.arange(self.n_vertices), self.n1)
        vb = (ix == 0) | (ix == m) | (iy == 0) | (iy == m)
        e = self._edge_table
        eb = np.zeros(self.n_edges, dtype=bool)
        hv = e[:, 0] >= 0
        eb[e[hv, 0]] = (iy[hv] == 0) | (iy[hv] == m)
        vv = e[:, 1] >= 0
        eb[e[vv, 1]] = (ix[vv] == 0) | (ix[vv] == m)
        return np.concatenate([vb, eb])

    def p2_interior(self):
        """(interior dof ids, dof -> interior position or -1)."""
        bnd = self.p2_dirichlet_mask()
        keep = np.flatnonzero(~bnd)
        pos = np.full(bnd.size, -1, dtype=np.int64)
        pos[keep] = np.arange(keep.size)
        return keep, pos

    def p2_points(self):
        x, y = self.vertex_xy()
        e = self._edge_table
        lo = np.repeat(np.arange(self.n_vertices), 3)[e.ravel() >= 0]
        kind = np.tile(np.arange(3), self.n_vertices)[e.ravel() >= 0]
        hi = lo + np.array([1, self.n1, self.n1 + 1])[kind]
        return (np.concatenate([x, 0.5 * (x[lo] + x[hi])]),
                np.concatenate([y, 0.5 * (y[lo] + y[hi])]))

    def p2_interior_count(self):
        return int((~self.p2_dirichlet_mask()).sum())
