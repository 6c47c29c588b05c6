#!/usr/bin/env python
"""Benchmark: fp64 NE-GS sweep throughput (DOF-updates/s) on Poisson control.

Headline workload (BASELINE.json configs[2], the north_star target): level 12
(4097 x 4097 P1 nodes, 33,570,818 unknowns, fp64, alpha = 1e-6), one step =
one forward NE-GS sweep over the finest level through the public sweep call
(default: distance-2 multicolour mode; --mode wavefront = the reference's
exact order, also reported under "modes"), x and r resident in HBM (537 MB >
the 126 MB L2, so no flush is needed between steps).  Also reported: every hot kernel of the cycle on
the same level, the time to 1e-8 of a multigrid solve, the end-to-end sweep
through the public API with host buffers, the CPU oracle on the host, and
the clocks seen during the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): every rank sweeps its own level-12
replica ("replicas only" for the exact-order sweep); time is
the max over ranks, value the whole-job throughput.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("fp64 DOF-updates/s per NE-GS sweep; multigrid time to 1e-8 rel. "
          "residual")
UNIT = "DOF-updates/s"
# algorithmic HBM bytes per unknown
# (x, r in and out for an NE-GS sweep; the two NE-Jacobi
# halves 16 + 40; x, f in and r out for the residual; fine in plus coarse out
# per fine unknown for restriction; fine x in/out plus coarse in for
# prolongation)
BYTES = {"ne_gs": 32, "ne_jacobi": 56, "residual": 24, "restrict": 10,
         "prolong": 18}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("OCMG_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend)
    return ws, rank, local


def max_over_ranks(v, ws, device):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU oracle (reported baseline / reference arm)
# ---------------------------------------------------------------------------

def cpu_sweep_rate(level=10, sweeps=10, alpha=1e-6):
    """Oracle C port of kernels.lsgs_sweep (1 thread) on a seeded level."""
    import oracle as O
    osys = O.poisson_system(level, alpha)
    st = O.OracleSmoother(osys, "lsgs")
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, osys.n)
    r = osys.residual(x, rng.uniform(-1, 1, osys.n))
    st.lsgs(x, r, True)                      # warm caches
    t0 = time.perf_counter()
    for _ in range(sweeps):
        st.lsgs(x, r, True)
    dt = (time.perf_counter() - t0) / sweeps
    return osys.n / dt, dt, osys.n


def run_reference_arm(args, ws, rank):
    """The reference's CPU path on all host threads: the NE-GS sweep
    (kernels.lsgs_sweep) is sequential, so every thread sweeps its own
    replica of the system (the oracle's C port, same operation order; the
    ctypes call releases the GIL); value = all threads' DOF updates / s."""
    if rank != 0:
        return
    import threading
    level = args.cpu_level
    import oracle as O
    osys = O.poisson_system(level, args.alpha)
    st = O.OracleSmoother(osys, "lsgs")
    rng = np.random.default_rng(0)
    x0 = rng.uniform(-1, 1, osys.n)
    r0 = osys.residual(x0, rng.uniform(-1, 1, osys.n))
    try:
        nthreads = len(os.sched_getaffinity(0))
    except AttributeError:
        nthreads = os.cpu_count() or 1
    reps = [(x0.copy(), r0.copy()) for _ in range(nthreads)]
    go = threading.Barrier(nthreads + 1)
    done = threading.Barrier(nthreads + 1)

    def work(i):
        x, r = reps[i]
        for _ in range(args.warmup):
            st.lsgs(x, r, True)
        go.wait()
        for _ in range(args.steps):
            st.lsgs(x, r, True)
        done.wait()
    th = [threading.Thread(target=work, args=(i,)) for i in range(nthreads)]
    for t in th:
        t.start()
    go.wait()
    t0 = time.perf_counter()
    done.wait()
    dt = (time.perf_counter() - t0) / args.steps
    for t in th:
        t.join()
    v = nthreads * osys.n / dt
    sample = (f"forward NE-GS sweep of Poisson control L{level} ({osys.n} "
              f"unknowns) x {args.steps} per thread, oracle C port of "
              f"kernels.lsgs_sweep, {nthreads} threads each on its own replica "
              "(the sweep is sequential)")
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1])",
        "config": {"workload": f"poisson_control_L{args.level}_ne_gs_sweep",
                   "unknowns": osys.n, "alpha": args.alpha,
                   "sample": f"full forward NE-GS sweep of L{level} per thread "
                             "and step"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def time_events(fn, iters, stream):
    import torch
    fn()  # warm (first calls allocate scratch / build plans)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(iters):
        fn()
    stop.record(stream)
    stop.synchronize()
    return start.elapsed_time(stop) / iters / 1e3


def kernel_table(dsys, coarse_sys, transfer, x, r, f, stream, iters, hbm):
    """Each hot kernel of a cycle on the finest level, CUDA-event timed."""
    import paper_1502_03917_b200 as P
    n = dsys.n
    rows = {}
    gs = P.make_smoother(dsys, "lsgs", gs_mode="wavefront")
    mc = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    nj = P.make_smoother(dsys, "normal")
    res_out = r.clone()
    import torch
    rc = torch.empty(coarse_sys.n, dtype=torch.float64, device=x.device)

    def add(name, key, t, units):
        rows[name] = {"dof_per_s": units / t, "ms": t * 1e3,
                      "gbs": BYTES[key] * units / t / 1e9,
                      "frac_hbm": BYTES[key] * units / t / 1e9 / hbm}
    from paper_1502_03917_b200 import _lib
    add("residual", "residual", time_events(
        lambda: _lib.call("ocmg_residual", dsys.handle, _lib.dptr(x),
                          _lib.dptr(f), _lib.dptr(res_out),
                          _lib.stream_ptr()), iters, stream), n)
    add("ne_jacobi", "ne_jacobi",
        time_events(lambda: nj.sweep(x, r), iters, stream), n)
    add("ne_gs_wavefront", "ne_gs",
        time_events(lambda: gs.sweep(x, r), iters, stream), n)
    # the cycle driver's form: residual ping-pong, no copy back
    from paper_1502_03917_b200.smoothers import lsgs_sweep_into
    add("ne_gs_multicolour", "ne_gs",
        time_events(lambda: lsgs_sweep_into(mc, x, r, res_out), iters, stream), n)
    cg = P.make_smoother(dsys, "cgs", gs_mode="multicolour")
    add("cgs_multicolour", "ne_gs",
        time_events(lambda: cg.sweep(x, r), iters, stream), n)
    add("restrict", "restrict", time_events(
        lambda: transfer.restrict(r, rc), iters, stream), n)
    add("prolong_add", "prolong", time_events(
        lambda: transfer.prolong_add(rc, x), iters, stream), n)
    return rows


def solve_timing(level, alpha, cycle, coarsest, mode, sine, problem="poisson",
                 smoother="lsgs"):
    """Time to 1e-8 relative residual (BASELINE protocol), setup excluded."""
    import torch

    import paper_1502_03917_b200 as P
    t_setup = time.perf_counter()
    kind = (P.SmootherKind("normal", tau=0.4) if smoother == "normal"
            else P.SmootherKind(smoother))  # lsgs / cgs / vanka
    cfg = P.CycleConfig(smoother=kind, cycle=cycle,
                        coarsest_level=coarsest, gs_mode=mode)
    mg = P.build_solver(problem, level, alpha, cfg)
    f = P.baseline_rhs(mg.finest, 0 if problem == "poisson" else 1,
                       add_sine=sine)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    mg.solve_to_tolerance(f, tol=1e-8, max_cycles=2)      # graph capture
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=300)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    sm_name = ("NE-Jacobi(tau=0.4)" if smoother == "normal"
               else f"CGS[{mode}]" if smoother == "cgs"
               else "Vanka(tau=0.4)" if smoother == "vanka" else f"NE-GS[{mode}]")
    return {"config": f"{problem} L{level} alpha={alpha} {cycle.upper()}(2,2) "
                      f"{sm_name} coarsest L{coarsest}"
                      + (" y_D=U+sin*sin" if sine else ""),
            "cycles": len(hist), "final_rel_residual": hist[-1],
            "convergence_factor": float(hist[-1] ** (1.0 / len(hist))),
            "seconds": t, "setup_seconds": t_setup}


def stokes_l10_solves(level=10):
    """Config 5: Stokes control L10, alpha in {1e-2, 1e-6}, NE-GS (exact
    order and multicolour) and NE-Jacobi (tau 0.35, the reference's Stokes
    default), V(2,2) to 1e-8; one hierarchy per alpha, assembled once."""
    import torch

    import paper_1502_03917_b200 as P
    from paper_1502_03917_b200.multigrid import Multigrid, assemble_hierarchy
    out = []
    kern = {}
    for alpha in (1e-2, 1e-6):
        t_setup = time.perf_counter()
        systems, transfers = assemble_hierarchy("stokes", 1, level, alpha)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t_setup
        if alpha == 1e-2:
            kern = stokes_kernel_table(systems[-1])
        for smoother, mode in (("lsgs", "wavefront"), ("lsgs", "multicolour"),
                               ("normal", "wavefront")):
            kind = (P.SmootherKind("normal", tau=0.35) if smoother == "normal"
                    else P.SmootherKind("lsgs"))
            cfg = P.CycleConfig(smoother=kind, cycle="v", coarsest_level=1,
                                gs_mode=mode)
            mg = Multigrid(systems, transfers, cfg)
            f = P.baseline_rhs(mg.finest, 1)
            mg.solve_to_tolerance(f, tol=1e-8, max_cycles=2)   # graph capture
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=300)
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            name = ("NE-Jacobi(tau=0.35)" if smoother == "normal"
                    else f"NE-GS[{mode}]")
            out.append({"config": f"stokes L{level} alpha={alpha} V(2,2) {name} "
                                  f"coarsest L1",
                        "cycles": len(hist), "final_rel_residual": hist[-1],
                        "convergence_factor": float(hist[-1] ** (1.0 / len(hist))),
                        "seconds": t, "setup_seconds": t_setup})
            del mg
        del systems, transfers
        torch.cuda.empty_cache()
    return out, kern


def stokes_kernel_table(dsys, iters=3):
    """The generic (CSR) kernels on the finest Stokes level: DOF/s and the
    fraction of HBM at SURVEY §8(d)'s vector bytes per DOF, and at the bytes
    the CSR format also streams (values, int32 columns, and for NE-GS/Jacobi
    the row_scaled copy)."""
    import torch

    import paper_1502_03917_b200 as P
    from paper_1502_03917_b200 import _lib
    from paper_1502_03917_b200.smoothers import lsgs_sweep_into
    hbm, _ = peaks()
    n = dsys.n
    nnz = dsys.matrix.nnz
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    f = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    r = dsys.residual(x, f)
    r2 = torch.empty_like(r)
    stream = torch.cuda.current_stream()
    nj = P.make_smoother(dsys, "normal", tau=0.35)
    mc = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    rows = {}

    def add(name, t, vec_b, mat_b):
        rows[name] = {"ms": t * 1e3, "dof_per_s": n / t,
                      "frac_hbm_vector_bytes": vec_b * n / t / 1e9 / hbm,
                      "frac_hbm_with_matrix": (vec_b * n + mat_b) / t / 1e9 / hbm}
    add("residual", time_events(lambda: _lib.call(
        "ocmg_residual", dsys.handle, _lib.dptr(x), _lib.dptr(f), _lib.dptr(r2),
        _lib.stream_ptr()), iters, stream), BYTES["residual"], 12 * nnz)
    add("ne_jacobi", time_events(lambda: nj.sweep(x, r), iters, stream),
        BYTES["ne_jacobi"], 24 * nnz)
    add("ne_gs_multicolour", time_events(lambda: lsgs_sweep_into(mc, x, r, r2),
                                         iters, stream), BYTES["ne_gs"], 20 * nnz)
    return {"level": dsys.level, "unknowns": n, "nnz": int(nnz), "kernels": rows}


def run_strip_arm(args, ws, rank, local):
    """--partition strips (N > 1): ONE L12 system strip-partitioned over the
    ranks (strong scaling).  A step is the ghost exchange (torch.distributed
    P2P over NCCL) plus one multicolour strip sweep per rank
    (paper_1502_03917_b200.strips); time = max over ranks."""
    import torch

    import paper_1502_03917_b200 as P
    from paper_1502_03917_b200 import _lib
    from paper_1502_03917_b200.strips import (StripPartition, exchange_ghosts,
                                              strip_sweep)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    hbm, peak_kind = peaks()
    dsys = P.build_poisson_system(args.level, args.alpha)
    n, n1 = dsys.n, 2 ** args.level + 1
    part = StripPartition(n1, ws, rank)
    g = torch.Generator(device=device).manual_seed(1234)  # same on all ranks
    x = torch.rand(n, dtype=torch.float64, device=device, generator=g) * 2 - 1
    f = torch.rand(n, dtype=torch.float64, device=device, generator=g) * 2 - 1
    r = dsys.residual(x, f)
    xo = part.scatter(x)
    rs = [part.scatter(r), torch.empty((2, part.slab_rows, n1),
                                       dtype=torch.float64, device=device)]
    del x, f, r
    stream = torch.cuda.current_stream()

    def step(i):
        cur = rs[i % 2]
        exchange_ghosts(cur, part)
        strip_sweep(dsys, part, xo, cur, rs[(i + 1) % 2])

    for i in range(args.warmup + (args.warmup % 2)):
        step(i)
    torch.cuda.synchronize()
    barrier(ws)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        launches0 = _lib.launch_count()
        barrier(ws)
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            step(i)
        stop.record(stream)
        stop.synchronize()
        launches = _lib.launch_count() - launches0
        barrier(ws)
    t_step = max_over_ranks(start.elapsed_time(stop) / args.steps / 1e3, ws, device)
    value = n / t_step
    # end to end: each rank's strip from pinned host memory and back
    xh = xo.cpu().pin_memory()
    rh = rs[0].cpu().pin_memory()

    def e2e_step():
        xo.copy_(xh, non_blocking=True)
        rs[0].copy_(rh, non_blocking=True)
        step(0)
        xh.copy_(xo, non_blocking=True)
        rh.copy_(rs[1], non_blocking=True)
    t_e2e = max_over_ranks(time_events(e2e_step, max(1, args.steps), stream),
                           ws, device)
    # config 3 on the partition: W(2,2) multicolour cycle, coarsest L1 (the
    # reference default; the partition needs a gathered smoothed level)
    from paper_1502_03917_b200.strips import (DistComm, LoopbackComm,
                                              StripMultigrid)
    solve = None
    e2e_bytes = 8 * (xo.numel() + rs[0].numel())
    if not args.no_solve_l12:
        del rs, xo
        cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="w",
                            coarsest_level=1, gs_mode="multicolour")
        mg = P.build_solver("poisson", args.level, args.alpha, cfg)
        fs = P.baseline_rhs(mg.finest, 0, add_sine=True)
        sm = StripMultigrid(mg, ws, [rank], DistComm() if ws > 1 else LoopbackComm())
        sm.load(fs)
        torch.cuda.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        hist = sm.solve(tol=1e-8, max_cycles=300)
        torch.cuda.synchronize()
        t_solve = max_over_ranks(time.perf_counter() - t0, ws, device)
        solve = {"config": f"poisson L{args.level} alpha={args.alpha} W(2,2) "
                           "NE-GS[multicolour] coarsest L1 y_D=U+sin*sin, "
                           f"row strips x{ws} (levels >= "
                           f"{mg.systems[sm.first].level} partitioned)",
                 "cycles": len(hist), "final_rel_residual": hist[-1],
                 "seconds": t_solve}
    if rank == 0:
        achieved = BYTES["ne_gs"] * n / t_step / 1e9
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] iterate and rhs)",
            "config": {"workload": f"poisson_control_L{args.level}_ne_gs_sweep",
                       "unknowns": n, "alpha": args.alpha,
                       "gs_mode": "multicolour",
                       "step": "ghost exchange (15 rows/side, NCCL P2P) + "
                               "one multicolour strip sweep per rank",
                       "l2": "x+r larger than L2 at N<=2; strips of L12 at "
                             "N>=4 may be partly L2-resident",
                       "parallelism": f"row strips x{ws}"},
            "roofline": {"bound": "hbm", "achieved": achieved / ws, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / ws / hbm, "traffic": None,
                         "bytes_per_dof": BYTES["ne_gs"], "per": "GPU"},
            "e2e": {"value": n / t_e2e, "unit": UNIT,
                    "h2d_bytes_per_step": e2e_bytes,
                    "d2h_bytes_per_step": e2e_bytes},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "solve": [solve] if solve else [],
        }), flush=True)
    barrier(ws)


def run_gpu_arm(args, ws, rank, local):
    import torch

    import paper_1502_03917_b200 as P
    from paper_1502_03917_b200 import _lib
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    hbm, peak_kind = peaks()

    dsys = P.build_poisson_system(args.level, args.alpha)
    n = dsys.n
    g = torch.Generator(device=device).manual_seed(1234 + rank)
    x = torch.rand(n, dtype=torch.float64, device=device, generator=g) * 2 - 1
    f = torch.rand(n, dtype=torch.float64, device=device, generator=g) * 2 - 1
    r = dsys.residual(x, f)
    st = P.make_smoother(dsys, "lsgs", gs_mode=args.mode)
    stream = torch.cuda.current_stream()

    # the driver's form of a sweep: residual ping-pong between r and r2
    from paper_1502_03917_b200.smoothers import lsgs_sweep_into
    r2 = torch.empty_like(r)
    bufs = [r, r2]

    def step(i):
        lsgs_sweep_into(st, x, bufs[i % 2], bufs[(i + 1) % 2])

    for i in range(args.warmup + (args.warmup % 2)):
        step(i)
    torch.cuda.synchronize()
    barrier(ws)

    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        launches0 = _lib.launch_count()
        barrier(ws)
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            step(i)
        stop.record(stream)
        stop.synchronize()
        launches = _lib.launch_count() - launches0
        barrier(ws)
    t_step = start.elapsed_time(stop) / args.steps / 1e3
    if args.steps % 2:
        r.copy_(r2)  # the current residual back in r
    t_step = max_over_ranks(t_step, ws, device)
    value = ws * n / t_step

    # end to end through the public API with host buffers (pinned): every
    # step is an independent job (its own host inputs, copied in, swept,
    # copied out).  Jobs alternate between two streams, so one job's
    # device-to-host copy overlaps the next one's host-to-device copy (the
    # PCIe link is full duplex); all copies stay inside the timed region.
    slots = []
    for _ in range(2):
        slots.append({"xh": x.cpu().pin_memory(), "rh": r.cpu().pin_memory(),
                      "xd": torch.empty_like(x), "ri": torch.empty_like(r),
                      "ro": torch.empty_like(r), "s": torch.cuda.Stream()})

    # a level's device scratch (wavefront flags and rings, multicolour
    # barriers) belongs to one stream at a time (include/ocmg_b200.h), so the
    # sweeps themselves are ordered across the two streams by an event; only
    # the copies overlap
    swept = [None]

    def e2e_job(sl):
        with torch.cuda.stream(sl["s"]):
            sl["xd"].copy_(sl["xh"], non_blocking=True)
            sl["ri"].copy_(sl["rh"], non_blocking=True)
            if swept[0] is not None:
                sl["s"].wait_event(swept[0])
            lsgs_sweep_into(st, sl["xd"], sl["ri"], sl["ro"])
            ev = torch.cuda.Event()
            ev.record(sl["s"])
            swept[0] = ev
            sl["xh"].copy_(sl["xd"], non_blocking=True)
            sl["rh"].copy_(sl["ro"], non_blocking=True)

    def e2e_run(k):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        swept[0] = None
        for sl in slots:
            sl["s"].wait_event(ev0)
        for i in range(k):
            e2e_job(slots[i % 2])
        for sl in slots:
            stream.wait_stream(sl["s"])
        ev1.record(stream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1) / k / 1e3
    e2e_run(2)
    t_e2e = e2e_run(max(2, args.steps))
    t_e2e = max_over_ranks(t_e2e, ws, device)

    result = None
    if rank == 0:
        achieved = BYTES["ne_gs"] * n / t_step / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            tr = json.load(open(tp))
            traffic = tr.get(f"ne_gs_{args.mode}_L{args.level}")
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] iterate and rhs)",
            "config": {"workload": f"poisson_control_L{args.level}_ne_gs_sweep",
                       "unknowns": n, "alpha": args.alpha,
                       "gs_mode": args.mode,
                       "step": "one forward NE-GS sweep of the finest level "
                               "(ocmg_ne_gs_sweep_into: residual ping-pong "
                               "between two buffers, as in the cycle driver)",
                       "l2": "inputs larger than L2 (x+r 2x268 MB), no flush",
                       "parallelism": f"replicas x{ws}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "bytes_per_dof": BYTES["ne_gs"]},
            "e2e": {"value": ws * n / t_e2e, "unit": UNIT,
                    "h2d_bytes_per_step": 2 * 8 * n,
                    "d2h_bytes_per_step": 2 * 8 * n,
                    "api": "paper_1502_03917_b200.smoothers.lsgs_sweep_into on "
                           "pinned host x, r (one independent job per step, "
                           "two streams: copy-out of a job overlaps copy-in "
                           "of the next)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        # both NE-GS modes side by side: the exact (reference-order,
        # wavefront) sweep is the reference arm's own order
        other = "wavefront" if args.mode == "multicolour" else "multicolour"
        result["modes"] = {args.mode: {"dof_per_s": value, "ms": t_step * 1e3,
                                       "frac_hbm": achieved / hbm}}
        st_o = P.make_smoother(dsys, "lsgs", gs_mode=other)
        st_o.sweep(x, r)
        t_o = time_events(lambda: st_o.sweep(x, r), 5, stream)
        result["modes"][other] = {
            "dof_per_s": n / t_o, "ms": t_o * 1e3,
            "frac_hbm": BYTES["ne_gs"] * n / t_o / 1e9 / hbm}
        if not args.quick:
            from paper_1502_03917_b200.transfer import system_transfer
            coarse = P.build_poisson_system(args.level - 1, args.alpha)
            tr = system_transfer(coarse, dsys)
            result["kernels"] = kernel_table(dsys, coarse, tr, x, r, f,
                                             stream, args.kernel_iters, hbm)
            # config 2: L10, NE-GS (both modes) vs NE-Jacobi, three alphas
            result["solve"] = []
            for a in (1.0, 1e-4, 1e-8):
                result["solve"] += [solve_timing(10, a, "v", 2, m, False)
                                    for m in ("wavefront", "multicolour")]
                result["solve"].append(solve_timing(10, a, "v", 2, "wavefront",
                                                    False, smoother="normal"))
            # CGS collective smoother, config-2 shape
            result["solve"] += [solve_timing(10, 1e-4, "v", 2, m, False,
                                             smoother="cgs")
                                for m in ("reference", "multicolour")]
            # Stokes control (configs 4 and 5; generic CSR kernels)
            result["solve"] += [solve_timing(5, 1e-4, "v", 1, m, False, "stokes")
                                for m in ("wavefront", "multicolour")]
            # Vanka patch smoother, config-4 shape
            result["solve"].append(solve_timing(5, 1e-4, "v", 1, "wavefront", False,
                                                "stokes", smoother="vanka"))
            if not args.no_stokes_l10:
                sv, sk = stokes_l10_solves()
                result["solve"] += sv
                result["stokes_kernels"] = sk
            if not args.no_solve_l12:
                # config 3 at the reference's default coarsest level L1
                # (SURVEY §8(d)); the exact-order W-cycle is north_star's
                # target run (18 cycles, the reference's count; its
                # per-cycle iterates are pinned by tests/test_fullsize_gpu.py)
                modes = ["multicolour"] + ([] if args.no_solve_l12_wavefront
                                           else ["wavefront"])
                for m in modes:
                    result["solve"].append(solve_timing(
                        args.level, args.alpha, "w", 1, m, True))
                # and at coarsest L3 (round-1 runs used it)
                result["solve"].append(solve_timing(
                    args.level, args.alpha, "w", 3, "multicolour", True))
        if ws == 1 and not args.no_cpu:
            v, dt, ncpu = cpu_sweep_rate(args.cpu_level, args.cpu_sweeps,
                                         args.alpha)
            result["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"forward NE-GS sweep, Poisson control "
                          f"L{args.cpu_level} ({ncpu} unknowns) x "
                          f"{args.cpu_sweeps}, oracle C port of "
                          f"kernels.lsgs_sweep, 1 of {os.cpu_count()} host "
                          "threads"}
        print(json.dumps(result), flush=True)
    barrier(ws)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=12)
    ap.add_argument("--alpha", type=float, default=1e-6)
    ap.add_argument("--mode", default="multicolour",
                    choices=["wavefront", "reference", "multicolour"])
    ap.add_argument("--partition", default=None,
                    choices=["replicas", "strips"],
                    help="N>1: one L12 system in row strips with ghost "
                         "exchange (strong scaling, the default) or N "
                         "independent replicas (weak)")
    ap.add_argument("--quick", action="store_true",
                    help="headline only (no kernel table / solves)")
    ap.add_argument("--no-stokes-l10", action="store_true",
                    help="skip the config-5 Stokes L10 solve (~80 s incl. setup)")
    ap.add_argument("--no-solve-l12", action="store_true",
                    help="skip the config-3 W-cycle solves at L12")
    ap.add_argument("--no-solve-l12-wavefront", action="store_true",
                    help="skip the exact-order (wavefront) W-cycle at L12")
    ap.add_argument("--no-cpu", action="store_true")
    # the CPU arms sweep the headline level itself (same_config); --cpu-level
    # only for quick local runs
    ap.add_argument("--cpu-level", type=int, default=None)
    ap.add_argument("--cpu-sweeps", type=int, default=5)
    ap.add_argument("--kernel-iters", type=int, default=5)
    args = ap.parse_args()
    if args.cpu_level is None:
        args.cpu_level = args.level
    if args.partition is None:
        args.partition = "strips" if args.gpus > 1 else "replicas"
    if args.warmup < 3:
        print("warning: --warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
    elif args.partition == "strips":
        run_strip_arm(args, ws, rank, local)
    else:
        run_gpu_arm(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
