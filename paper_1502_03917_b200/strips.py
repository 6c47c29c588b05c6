"""Strip partition of the fine levels across ranks.

One process per GPU; rank p owns the mesh rows [y0, y1) of a structured P1
level (all fields of a vertex on the same rank, rows split as evenly as
possible).  The multicolour NE-GS sweep needs 15 ghost rows of the residual
on each side: the pipelined kernel recomputes a 14-row halo (2 rows per
colour x 7 vertex colours) and reads one more row.  One sweep is then

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

GHOST = 15


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
    # one grouped batch (ncclGroupStart/End under NCCL): both neighbours
    # send first, which ungrouped NCCL point-to-point calls may deadlock on
    ops, recvs = [], []
    for peer, (a, b), (c, d) in ghost_plan(part):
        sbuf = slab[:, a:b].contiguous()
        rbuf = torch.empty_like(slab[:, c:d])
        ops.append(dist.P2POp(dist.isend, sbuf, peer, group=group))
        ops.append(dist.P2POp(dist.irecv, rbuf, peer, group=group))
        recvs.append((rbuf, c, d))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for rbuf, c, d in recvs:
        slab[:, c:d].copy_(rbuf)


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


def strip_sweep(system, part, x, r_in, r_out, forward=True, stream=None):
    """One multicolour NE-GS sweep of this rank's strip (ghosts of r_in must
    be current).  x, r_in, r_out: slabs (2, slab_rows, n1) -- or full-size
    level vectors with part.s0 = 0, part.s1 = n1 (see StripMultigrid).
    system: the structured level (every rank builds the same level handle;
    only its coefficient tables are used)."""
    n1 = part.n1
    shape = (2, part.s1 - part.s0, n1)
    for t in (x, r_in, r_out):
        if tuple(t.reshape(2, -1, n1).shape) != shape:
            raise ValueError("strip tensors have the wrong shape")
    ops = ctypes.c_int64()
    _lib.call("ocmg_ne_gs_sweep_strip", system.handle, 1 if forward else 0,
              part.y0, part.y1, part.s0, part.s1, _lib.dptr(x),
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

    def sweep(self, x_slab, r_slab, forward=True):
        """Returns the slab holding the new residual (r_slab or the spare;
        the other becomes the spare)."""
        exchange_ghosts(r_slab, self.part, self.group)
        out = self.spare
        strip_sweep(self.system, self.part, x_slab, r_slab, out, forward)
        self.spare = r_slab
        return out


# ---------------------------------------------------------------------------
# Strip-partitioned multigrid cycle (Poisson control, multicolour NE-GS)
# ---------------------------------------------------------------------------

def nested_bounds(n1_levels, world_size, ghost=GHOST):
    """Row bounds per rank for a coarse-to-fine list of grid sizes, nested
    (fine strip [2 y0, 2 y1), the last clipped to n1): a coarse row and the
    fine rows it restricts from live on the same rank.  Returns (first
    partitioned index, bounds per level) -- levels below stay whole."""
    first = None
    for i, n1 in enumerate(n1_levels):
        if n1 // world_size >= ghost:
            first = i
            break
    if first is None:
        raise ValueError("no level is wide enough to split over "
                         f"{world_size} ranks")
    bounds = [None] * len(n1_levels)
    base = StripPartition(n1_levels[first], world_size, 0, ghost).bounds
    bounds[first] = base
    for i in range(first + 1, len(n1_levels)):
        n1 = n1_levels[i]
        bounds[i] = [(2 * a, min(2 * b, n1)) for a, b in bounds[i - 1]]
        bounds[i][-1] = (bounds[i][-1][0], n1)
    return first, bounds


def _rows(v, n1, a, b):
    """Per-field contiguous views of the rows [a, b) of a full-size level
    vector (2 n1^2,)."""
    N = n1 * n1
    return [v[f * N + a * n1:f * N + b * n1] for f in range(2)]


class LoopbackComm:
    """Every rank's state in this process: exchanges are copies.  Lets one
    GPU run the partitioned cycle rank after rank and compare it with the
    single-GPU cycle (no kernel ever waits on another rank)."""

    def exchange(self, states, level, name, g):
        for st in states:
            y0, y1 = st.bounds[level]
            n1 = st.n1[level]
            v = getattr(st, name)[level]
            for peer in (st.rank - 1, st.rank + 1):
                if 0 <= peer < len(states):
                    a, b = (y0 - g, y0) if peer < st.rank else (y1, y1 + g)
                    src = getattr(states[peer], name)[level]
                    for dst_f, src_f in zip(_rows(v, n1, a, b), _rows(src, n1, a, b)):
                        dst_f.copy_(src_f)

    def allgather(self, states, level, name):
        for st in states:
            v = getattr(st, name)[level]
            n1 = st.n1[level]
            for peer in states:
                if peer is st:
                    continue
                a, b = peer.bounds[level]
                src = getattr(peer, name)[level]
                for dst_f, src_f in zip(_rows(v, n1, a, b), _rows(src, n1, a, b)):
                    dst_f.copy_(src_f)

    def allreduce(self, values):
        total = sum(values)
        return [total] * len(values)


class DistComm:
    """One rank per process, torch.distributed (NCCL over NVLink for CUDA
    tensors): ghost rows by grouped isend/irecv straight into the full-size
    vectors, the gather by one padded all_gather_into_tensor, sums by
    all_reduce."""

    def __init__(self, group=None, device="cuda"):
        self.group, self.device = group, device

    def exchange(self, states, level, name, g):
        import torch.distributed as dist
        (st,) = states
        y0, y1 = st.bounds[level]
        n1 = st.n1[level]
        v = getattr(st, name)[level]
        ops = []
        for peer in (st.rank - 1, st.rank + 1):
            if not 0 <= peer < st.world_size:
                continue
            snd = (y0, y0 + g) if peer < st.rank else (y1 - g, y1)
            rcv = (y0 - g, y0) if peer < st.rank else (y1, y1 + g)
            for s_f, r_f in zip(_rows(v, n1, *snd), _rows(v, n1, *rcv)):
                ops.append(dist.P2POp(dist.isend, s_f, peer, group=self.group))
                ops.append(dist.P2POp(dist.irecv, r_f, peer, group=self.group))
        # grouped (ncclGroupStart/End): both neighbours post sends first
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def allgather(self, states, level, name):
        """One all_gather_into_tensor of every rank's rows (both fields),
        each padded to the longest strip, then scattered into place."""
        import torch
        import torch.distributed as dist
        (st,) = states
        v = getattr(st, name)[level]
        n1 = st.n1[level]
        bnds = st.all_bounds[level]
        mrows = max(b - a for a, b in bnds)
        a, b = bnds[st.rank]
        send = torch.zeros(2, mrows, n1, dtype=v.dtype, device=v.device)
        for f, rows in enumerate(_rows(v, n1, a, b)):
            send[f, :b - a] = rows.view(b - a, n1)
        recv = torch.empty(st.world_size * 2 * mrows * n1, dtype=v.dtype,
                           device=v.device)
        dist.all_gather_into_tensor(recv, send.reshape(-1), group=self.group)
        recv = recv.view(st.world_size, 2, mrows, n1)
        for p, (a, b) in enumerate(bnds):
            if p == st.rank:
                continue
            for f, rows in enumerate(_rows(v, n1, a, b)):
                rows.copy_(recv[p, f, :b - a].reshape(-1))

    def allreduce(self, values):
        import torch
        import torch.distributed as dist
        t = torch.tensor(values, dtype=torch.float64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return t.tolist()


class _RankState:
    def __init__(self, rank, world_size, n1s, all_bounds, first, device="cuda"):
        import torch
        self.rank, self.world_size = rank, world_size
        self.n1 = n1s
        self.all_bounds = all_bounds
        self.bounds = [b[rank] if b is not None else None for b in all_bounds]

        def vec(i):
            return torch.zeros(2 * n1s[i] ** 2, dtype=torch.float64, device=device)
        L = len(n1s)
        # x, f on every level from the gather level up; r, r2 where smoothed
        self.x = [vec(i) if i >= first - 1 else None for i in range(L)]
        self.f = [vec(i) if i >= first - 1 else None for i in range(L)]
        # (bounds[first-1] are the gathered level's rows this rank restricts)
        self.r = [vec(i) if i >= first else None for i in range(L)]
        self.r2 = [vec(i) if i >= first else None for i in range(L)]


def partition(mg, n_gpus=None, collapse_threshold=None):
    """The strip-partitioned cycle of ``mg`` over ``n_gpus`` ranks.  Under
    torch.distributed (one process per GPU, torchrun) this process drives its
    own rank and exchanges over the process group (n_gpus, if given, must be
    the world size); without it one process drives all n_gpus ranks on its
    GPU with loopback exchanges (bit-identical to the single-GPU cycle)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        ws = dist.get_world_size()
        if n_gpus is not None and n_gpus != ws:
            raise ValueError(f"n_gpus={n_gpus} but the process group has {ws} ranks")
        return StripMultigrid(mg, ws, [dist.get_rank()], DistComm(),
                              collapse_threshold=collapse_threshold)
    if n_gpus is None or n_gpus < 1:
        raise ValueError("n_gpus is required outside torch.distributed")
    return StripMultigrid(mg, n_gpus, list(range(n_gpus)), LoopbackComm(),
                          collapse_threshold=collapse_threshold)


class StripMultigrid:
    """The BASELINE V/W cycle with its fine levels split into row strips
    (SURVEY.md §8(e)).  Levels whose strips would be thinner than the 15
    ghost rows of a sweep are gathered: every rank applies the same
    single-GPU coarse correction to them (ocmg_coarse_correction).

    Per partitioned level visit: x ghost (1 row) -> residual rows; per sweep
    r ghost (15 rows) -> strip sweep (residual ping-pong); r ghost (1 row) ->
    restriction rows; coarse visit(s); coarse x ghost (1 row) -> prolongation
    rows; residual; post-sweeps.  Every row is computed with the single-GPU
    kernels' arithmetic, so the iterate is bit-identical to Multigrid's.

    mg: a Poisson Multigrid with gs_mode="multicolour" (it supplies the
    levels, transfers and the gathered sub-hierarchy).  ranks: the ranks
    this process drives (one with DistComm; all of them with LoopbackComm).
    """

    def __init__(self, mg, world_size, ranks, comm, collapse_threshold=None):
        """collapse_threshold: levels with fewer unknowns than this stay on
        every rank whole (the coarse end of the cycle "collapsed onto a
        single GPU", SURVEY.md §5 / north_star (4)), on top of the levels
        whose strips would be thinner than a sweep's ghost rows."""
        cfg = mg.config
        self.jacobi = cfg.smoother.name == "normal"
        if not self.jacobi and (cfg.gs_mode != "multicolour" or
                                cfg.smoother.name not in ("lsgs", "slsgs")):
            raise ValueError("strip cycles run multicolour NE-GS or NE-Jacobi "
                             "smoothers")
        self.tau = cfg.smoother.tau
        self.mg, self.comm = mg, comm
        n1s = [2 ** s.level + 1 for s in mg.systems]
        first, bounds = nested_bounds(n1s, world_size)
        # levels the single-GPU cycle has collapsed into a dense coarse
        # correction are never visited: the partition starts above them
        col = ctypes.c_int()
        _lib.call("ocmg_hierarchy_collapsed_level", mg.native().handle, ctypes.byref(col))
        first = max(first, col.value + 1)
        if collapse_threshold is not None:
            big = [i for i, s in enumerate(mg.systems) if s.n >= collapse_threshold]
            if not big:
                raise ValueError("collapse_threshold leaves no level to partition")
            first = max(first, big[0])
        if first < 2:
            raise ValueError("partitioned levels must leave a gathered "
                             "sub-hierarchy of at least one smoothed level")
        # partitioned levels and the gathered one they restrict into are
        # structured; below that any level kind runs (the gathered
        # sub-cycle is the single-GPU ocmg_cycle)
        if not all(getattr(s, "structured", False) for s in mg.systems[first - 1:]):
            raise ValueError("strip cycles need structured Poisson levels")
        self.first, self.gather = first, first - 1
        # each rank restricts the gathered level's rows that its fine strip
        # covers: coarse row c reads fine rows 2c-1 .. 2c+1 (one ghost row)
        bounds[first - 1] = [((a + 1) // 2, (b + 1) // 2) for a, b in bounds[first]]
        self.n1s = n1s
        self.states = [_RankState(r, world_size, n1s, bounds, first) for r in ranks]
        self.w = cfg.cycle == "w"
        self.nu_pre, self.nu_post = cfg.nu_pre, cfg.nu_post
        self.slsgs = cfg.smoother.name == "slsgs"

    # -- per-level operations on every driven rank --------------------------
    def _resid(self, i):
        self.comm.exchange(self.states, i, "x", 1)
        sysi = self.mg.systems[i]
        for st in self.states:
            y0, y1 = st.bounds[i]
            _lib.call("ocmg_residual_rows", sysi.handle, _lib.dptr(st.x[i]),
                      _lib.dptr(st.f[i]), _lib.dptr(st.r[i]), y0, y1,
                      _lib.stream_ptr())

    def _sweep(self, i, forward):
        self.comm.exchange(self.states, i, "r", GHOST)
        sysi = self.mg.systems[i]
        n1 = self.n1s[i]
        for st in self.states:
            y0, y1 = st.bounds[i]
            ops = ctypes.c_int64()
            _lib.call("ocmg_ne_gs_sweep_strip", sysi.handle, 1 if forward else 0,
                      y0, y1, 0, n1, _lib.dptr(st.x[i]), _lib.dptr(st.r[i]),
                      _lib.dptr(st.r2[i]), _lib.stream_ptr(), ctypes.byref(ops))
            st.r[i], st.r2[i] = st.r2[i], st.r[i]

    def _jacobi(self, i):
        """NE-Jacobi on the strips (kernels.py:17-39): r ghost (1 row) -> p
        of the own rows -> p ghost (1 row) -> x += p, r -= A p on the own
        rows; the arithmetic of the single-GPU halves row for row."""
        sysi = self.mg.systems[i]
        self.comm.exchange(self.states, i, "r", 1)
        for st in self.states:
            y0, y1 = st.bounds[i]
            _lib.call("ocmg_ne_jacobi_p_rows", sysi.handle, float(self.tau),
                      _lib.dptr(st.r[i]), _lib.dptr(st.r2[i]), y0, y1,
                      _lib.stream_ptr())
        self.comm.exchange(self.states, i, "r2", 1)
        for st in self.states:
            y0, y1 = st.bounds[i]
            _lib.call("ocmg_ne_jacobi_apply_rows", sysi.handle, _lib.dptr(st.r2[i]),
                      _lib.dptr(st.x[i]), _lib.dptr(st.r[i]), y0, y1,
                      _lib.stream_ptr())

    def _smooth(self, i, nu):
        for _ in range(nu):
            if self.jacobi:
                self._jacobi(i)
                continue
            self._sweep(i, True)
            if self.slsgs:
                self._sweep(i, False)

    def _visit(self, i):
        self._resid(i)
        self._smooth(i, self.nu_pre)
        self.comm.exchange(self.states, i, "r", 1)
        t = self.mg.transfers[i - 1]
        for st in self.states:
            cy0, cy1 = st.bounds[i - 1]
            _lib.call("ocmg_restrict_rows", t.handle, _lib.dptr(st.r[i]),
                      _lib.dptr(st.f[i - 1]), cy0, cy1, _lib.stream_ptr())
        if i - 1 == self.gather:
            # the gathered coarse end: every rank applies the single-GPU
            # coarse correction (rec sub-cycles, or the collapsed map) to the
            # whole gathered right-hand side -- the call ocmg_cycle makes
            self.comm.allgather(self.states, i - 1, "f")
            h = self.mg.native().handle
            for st in self.states:
                _lib.call("ocmg_coarse_correction", h, i, _lib.dptr(st.f[i - 1]),
                          _lib.dptr(st.x[i - 1]), _lib.stream_ptr())
        else:
            for st in self.states:
                st.x[i - 1].zero_()
            rec = 2 if (self.w and i - 1 > 0) else 1
            for _ in range(rec):
                self._visit(i - 1)
        if i - 1 >= self.first:
            self.comm.exchange(self.states, i - 1, "x", 1)
        for st in self.states:
            fy0, fy1 = st.bounds[i]
            _lib.call("ocmg_prolong_add_rows", t.handle, _lib.dptr(st.x[i - 1]),
                      _lib.dptr(st.x[i]), fy0, fy1, _lib.stream_ptr())
        self._resid(i)
        self._smooth(i, self.nu_post)

    def cycle(self):
        self._visit(len(self.n1s) - 1)

    def load(self, f_full, x_full=None):
        """Copy the finest rhs (and start vector) rows into the rank states
        (f_full / x_full: full-size device vectors)."""
        top = len(self.n1s) - 1
        for st in self.states:
            st.f[top].copy_(f_full)
            if x_full is None:
                st.x[top].zero_()
            else:
                st.x[top].copy_(x_full)

    def gather_x(self):
        """The finest iterate assembled from the ranks' own rows (loopback)."""
        import torch
        top = len(self.n1s) - 1
        n1 = self.n1s[top]
        out = torch.empty_like(self.states[0].x[top])
        for st in self.states:
            y0, y1 = st.bounds[top]
            for o, s in zip(_rows(out, n1, y0, y1), _rows(st.x[top], n1, y0, y1)):
                o.copy_(s)
        return out

    def solve(self, tol=1e-8, max_cycles=300):
        """BASELINE protocol on the partition: rel = ||f - A x|| / ||f||
        from the ranks' own rows (all_reduce), stop at tol."""
        top = len(self.n1s) - 1
        n1 = self.n1s[top]

        def own_sumsq(vecs):
            vals = []
            for st, v in zip(self.states, vecs):
                y0, y1 = st.bounds[top]
                vals.append(float(sum((t * t).sum() for t in _rows(v, n1, y0, y1))))
            return self.comm.allreduce(vals)[0]
        fn = own_sumsq([st.f[top] for st in self.states]) ** 0.5
        hist = []
        for _ in range(max_cycles):
            self.cycle()
            self._resid(top)
            rel = own_sumsq([st.r[top] for st in self.states]) ** 0.5 / fn
            hist.append(rel)
            if rel <= tol:
                break
        return hist
