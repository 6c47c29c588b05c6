"""Per-level cost of the cycle's pieces and whole-cycle times (dev tool).

python scripts/cycle_prof.py [--level 12] [--mode multicolour]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402
from paper_1502_03917_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=12)
ap.add_argument("--mode", default="multicolour")
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--no-levels", action="store_true")
ap.add_argument("--coarsest", default="1,3")
a = ap.parse_args()


def ev_time(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


print("level  n1   sweep_us  residual_us", flush=True)
for k in ([] if a.no_levels else range(2, a.level + 1)):
    sysk = P.build_poisson_system(k, 1e-6)
    x = torch.rand(sysk.n, dtype=torch.float64, device="cuda")
    r = torch.rand(sysk.n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(r)
    st = P.make_smoother(sysk, "lsgs", gs_mode=a.mode)
    ts = ev_time(lambda: st.sweep(x, r))
    tr = ev_time(lambda: _lib.call("ocmg_residual", sysk.handle, _lib.dptr(x),
                                   _lib.dptr(x), _lib.dptr(out), _lib.stream_ptr()))
    print(f"{k:5d} {2 ** k + 1:5d} {ts:10.1f} {tr:10.1f}", flush=True)

for cyc in ("v", "w"):
    for coarsest in [int(c) for c in a.coarsest.split(",")]:
        cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle=cyc,
                            coarsest_level=coarsest, gs_mode=a.mode)
        mg = P.build_solver("poisson", a.level, 1e-6, cfg)
        f = P.baseline_rhs(mg.finest, 0, add_sine=True)
        for use_stream in (False, True):
            s = torch.cuda.Stream() if use_stream else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                mg.solve_to_tolerance(f, tol=0.0, max_cycles=1)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                mg.solve_to_tolerance(f, tol=0.0, max_cycles=a.cycles)
                torch.cuda.synchronize()
                t = (time.perf_counter() - t0) / a.cycles
            print(f"{cyc.upper()}-cycle L{a.level} coarsest L{coarsest} "
                  f"{'side stream (graph)' if use_stream else 'default stream'}: "
                  f"{t * 1e3:8.2f} ms/cycle", flush=True)
