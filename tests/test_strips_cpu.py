"""Strip partition + ghost exchange on CPU: the partition
arithmetic and a world-size-2 gloo exchange.  The strip kernel itself is
checked on the GPU (tests/test_gpu_parity.py::test_strip_sweeps_*)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1502_03917_b200.strips import (GHOST, StripPartition,  # noqa: E402
                                          ghost_plan)


@pytest.mark.parametrize("n1,ws", [(65, 2), (65, 4), (257, 3), (1025, 8),
                                   (4097, 8), (4097, 5)])
def test_partition_tiles_rows_and_plans_match(n1, ws):
    parts = [StripPartition(n1, ws, p) for p in range(ws)]
    assert parts[0].y0 == 0 and parts[-1].y1 == n1
    for a, b in zip(parts, parts[1:]):
        assert a.y1 == b.y0
    assert max(p.rows for p in parts) - min(p.rows for p in parts) <= 1
    for p in parts:
        assert p.s0 == max(0, p.y0 - GHOST) and p.s1 == min(n1, p.y1 + GHOST)
        for peer, (a, b), (c, d) in ghost_plan(p):
            # what I receive from `peer` is exactly what `peer` sends me
            q = parts[peer]
            mine = [(pp, snd) for pp, snd, _ in ghost_plan(q) if pp == p.rank]
            assert len(mine) == 1
            qa, qb = mine[0][1]
            assert (q.s0 + qa, q.s0 + qb) == (p.s0 + c, p.s0 + d)
            assert b - a == d - c == GHOST


def test_partition_rejects_thin_strips():
    with pytest.raises(ValueError):
        StripPartition(33, 4, 0)  # 8-row strips < GHOST


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, n1, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        from paper_1502_03917_b200.strips import exchange_ghosts
        part = StripPartition(n1, ws, rank)
        rows = torch.arange(n1, dtype=torch.float64)
        glob = (rows[None, :, None] * 1000 + torch.arange(n1)[None, None, :]
                + torch.tensor([0.0, 1e7])[:, None, None]).expand(2, n1, n1)
        slab = torch.full((2, part.slab_rows, n1), -1.0, dtype=torch.float64)
        part.own(slab).copy_(glob[:, part.y0:part.y1])
        exchange_ghosts(slab, part)
        ok = torch.equal(slab, glob[:, part.s0:part.s1])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("ws", [2])
def test_gloo_ghost_exchange(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, 97, q))
             for r in range(ws)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(ws)}, res


def _dist_comm_worker(rank, ws, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        from paper_1502_03917_b200.strips import DistComm, _RankState, nested_bounds
        n1s = [17, 33, 65, 129]
        first, bounds = nested_bounds(n1s, ws)
        bounds[first - 1] = [((a + 1) // 2, (b + 1) // 2) for a, b in bounds[first]]
        st = _RankState(rank, ws, n1s, bounds, first, device="cpu")
        comm = DistComm(device="cpu")
        ok = True
        # ghost exchange on the finest level: own rows hold the global index
        top = len(n1s) - 1
        n1 = n1s[top]
        glob = torch.arange(2 * n1 * n1, dtype=torch.float64)
        y0, y1 = st.bounds[top]
        for fld in range(2):
            a, b = fld * n1 * n1 + y0 * n1, fld * n1 * n1 + y1 * n1
            st.x[top][a:b] = glob[a:b]
        comm.exchange([st], top, "x", 2)
        for fld in range(2):
            lo = max(0, y0 - 2) * n1 + fld * n1 * n1
            hi = min(n1, y1 + 2) * n1 + fld * n1 * n1
            ok &= torch.equal(st.x[top][lo:hi], glob[lo:hi])
        # all-gather of the gathered level's contributions
        g = first - 1
        c0, c1 = st.bounds[g]
        m = n1s[g]
        for fld in range(2):
            a, b = fld * m * m + c0 * m, fld * m * m + c1 * m
            st.f[g][a:b] = torch.arange(a, b, dtype=torch.float64)
        comm.allgather([st], g, "f")
        ok &= torch.equal(st.f[g], torch.arange(2 * m * m, dtype=torch.float64))
        s = comm.allreduce([float(rank + 1)])
        ok &= s[0] == ws * (ws + 1) / 2
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_gloo_dist_comm_exchange_gather_reduce():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_comm_worker, args=(r, ws, port, q))
             for r in range(ws)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(ws)}, res


def test_nested_bounds_tile_and_nest():
    from paper_1502_03917_b200.strips import nested_bounds
    n1s = [2 ** k + 1 for k in range(3, 13)]
    for ws in (2, 4, 8):
        first, b = nested_bounds(n1s, ws)
        assert n1s[first] // ws >= GHOST and n1s[first - 1] // ws < GHOST
        for i in range(first, len(n1s)):
            assert b[i][0][0] == 0 and b[i][-1][1] == n1s[i]
            assert all(p[1] == q[0] for p, q in zip(b[i], b[i][1:]))
            assert min(y1 - y0 for y0, y1 in b[i]) >= GHOST
            if i > first:
                assert all(f[0] == 2 * c[0] for f, c in zip(b[i], b[i - 1]))
