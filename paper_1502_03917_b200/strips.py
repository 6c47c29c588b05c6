"""Strip partition of the fine levels across ranks.

One process per GPU; rank p owns the mesh rows [y0, y1) of a structured P1
level (all fields of a vertex on the same rank, rows split as evenly as
possible).  The multicolour NE-GS sweep needs 29 ghost rows of the residual
on each side: the pipelined kernel recomputes a 28-row halo (2 rows per
colour x 14 colours) and reads one more row.  One sweep is then

    exchange_ghosts(r_in)            # one send/recv pair per neighbour
    ocmg_ne_gs_sweep_strip(...)      # the single-GPU kernel on the slab

with no other communication; the union of the ranks' strips is
bit-identical to the single-GPU sweep.  The exchange uses torch.distributed
point-to-point calls: NCCL (NVLink) for CUDA tensors, gloo for CPU tensors
(the CPU tests).  The exact-order (wavefront) sweep does not shard: its
critical path of 3*2^k+8 steps is the same on any partition.

Vocabulary: a *strip* is a rank's own rows, a *slab* is the strip plus its
ghost rows, stored as a (2, slab_rows, n1) fp64 tensor (field-major, like the
reference's global layout restricted to those rows).
"""
from __future__ import annotations

import ctypes

from . import _lib

GHOST = 29


class StripPartition:
    """Rows of an n1 x n1 vertex grid split over `world_size` ranks."""

    def __init__(self, n1, world_size, rank, ghost=GHOST):
        if world_size < 1 or not 0 <= rank < world_size:
            raise ValueError(f"bad rank {rank} of {world_size}")
        base, rem = divmod(n1, world_size)
        if base < ghost and world_size > 1:
            raise ValueError(
                f"{world_size} strips of a {n1}-row grid are thinner than the "
                f"{ghost} ghost rows a multicolour sweep needs")
        self.n1, self.world_size, self.rank, self.ghost = n1, world_size, rank, ghost
        self.bounds = []
        y = 0
        for p in range(world_size):
            h = base + (1 if p < rem else 0)
            self.bounds.append((y, y + h))
            y += h
        self.y0, self.y1 = self.bounds[rank]
        self.s0 = max(0, self.y0 - ghost)
        self.s1 = min(n1, self.y1 + ghost)

    @property
    def rows(self):
        return self.y1 - self.y0

    @property
    def slab_rows(self):
        return self.s1 - self.s0

    def own(self, slab):
        """View of the strip's own rows inside a slab tensor."""
        return slab[:, self.y0 - self.s0:self.y1 - self.s0]

    def scatter(self, glob):
        """Slab of a global (2*n1*n1,) vector (for tests and setup)."""
        g = glob.reshape(2, self.n1, self.n1)
        return g[:, self.s0:self.s1].contiguous()

    def scatter_own(self, glob):
        g = glob.reshape(2, self.n1, self.n1)
        return g[:, self.y0:self.y1].contiguous()


def ghost_plan(part):
    """(peer, own rows to send, ghost rows to receive) per neighbour, as
    slab-relative row ranges."""
    plan = []
    g, s0 = part.ghost, part.s0
    if part.rank > 0:  # lower neighbour: it needs my first g rows
        plan.append((part.rank - 1,
                     (part.y0 - s0, part.y0 - s0 + g),
                     (part.s0 - s0, part.y0 - s0)))
    if part.rank < part.world_size - 1:  # upper neighbour: my last g rows
        plan.append((part.rank + 1,
                     (part.y1 - s0 - g, part.y1 - s0),
                     (part.y1 - s0, part.s1 - s0)))
    return plan


def exchange_ghosts(slab, part, group=None):
    """Refresh the ghost rows of `slab` (2, slab_rows, n1) from the
    neighbouring ranks (torch.distributed point-to-point)."""
    import torch
    import torch.distributed as dist
    if part.world_size == 1:
        return
    sends, recvs = [], []
    for peer, (a, b), (c, d) in ghost_plan(part):
        sbuf = slab[:, a:b].contiguous()
        rbuf = torch.empty_like(slab[:, c:d])
        sends.append(dist.isend(sbuf, peer, group=group))
        recvs.append((dist.irecv(rbuf, peer, group=group), rbuf, c, d))
    for req, rbuf, c, d in recvs:
        req.wait()
        slab[:, c:d].copy_(rbuf)
    for req in sends:
        req.wait()


class LoopbackExchange:
    """All ranks' slabs in one process, ghosts copied between them: runs the
    strip sweeps of every rank on one GPU, one after another, to check the
    decomposition (no rank waits on another inside a kernel)."""

    def __init__(self, parts):
        self.parts = parts

    def exchange(self, slabs):
        for part, slab in zip(self.parts, slabs):
            for peer, _, (c, d) in ghost_plan(part):
                src = self.parts[peer]
                rows = slice(part.s0 + c - src.s0, part.s0 + d - src.s0)
                slab[:, c:d].copy_(slabs[peer][:, rows])


def strip_sweep(system, part, x_own, r_in, r_out, forward=True, stream=None):
    """One multicolour NE-GS sweep of this rank's strip (ghosts of r_in must
    be current).  system: the structured level (every rank builds the same
    level handle; only its coefficient tables are used)."""
    n1 = part.n1
    if x_own.shape != (2, part.rows, n1) or r_in.shape != (2, part.slab_rows, n1) \
            or r_out.shape != r_in.shape:
        raise ValueError("strip tensors have the wrong shape")
    ops = ctypes.c_int64()
    _lib.call("ocmg_ne_gs_sweep_strip", system.handle, 1 if forward else 0,
              part.y0, part.y1, part.s0, part.s1, _lib.dptr(x_own),
              _lib.dptr(r_in), _lib.dptr(r_out),
              stream if stream is not None else _lib.stream_ptr(),
              ctypes.byref(ops))
    return ops.value


class StripSmoother:
    """Multicolour NE-GS on a strip-partitioned structured level: ghost
    exchange + one kernel per sweep, residual ping-pong between two slabs."""

    def __init__(self, system, part, group=None):
        import torch
        if not getattr(system, "structured", False):
            raise ValueError("strip partition needs a structured P1 level")
        self.system, self.part, self.group = system, part, group
        self.spare = torch.empty((2, part.slab_rows, part.n1),
                                 dtype=torch.float64, device="cuda")

    def sweep(self, x_own, r_slab, forward=True):
        """Returns the slab holding the new residual (r_slab or the spare;
        the other becomes the spare)."""
        exchange_ghosts(r_slab, self.part, self.group)
        out = self.spare
        strip_sweep(self.system, self.part, x_own, r_slab, out, forward)
        self.spare = r_slab
        return out
