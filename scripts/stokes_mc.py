"""Stokes control multicolour V(2,2) solves at L9/L10 with the greedy
distance-2 colouring lifted to large levels (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, json, torch
import paper_1502_03917_b200 as P
from paper_1502_03917_b200 import assembly
from paper_1502_03917_b200.multigrid import Multigrid, assemble_hierarchy
assembly.COLOURING_MAX_ROWS = 30_000_000
for lev in (9, 10):
    t=time.perf_counter(); systems, transfers = assemble_hierarchy("stokes", 1, lev, 1e-2); torch.cuda.synchronize()
    print("setup L", lev, time.perf_counter()-t, flush=True)
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="v", coarsest_level=1, gs_mode="multicolour")
    mg = Multigrid(systems, transfers, cfg)
    f = P.baseline_rhs(mg.finest, 1)
    mg.solve_to_tolerance(f, tol=1e-8, max_cycles=2); torch.cuda.synchronize()
    t=time.perf_counter(); _, h = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=300); torch.cuda.synchronize()
    print(json.dumps({"level": lev, "cycles": len(h), "final": h[-1], "seconds": time.perf_counter()-t}), flush=True)
    del mg, systems, transfers; torch.cuda.empty_cache()
