"""Run exactly one cycle (no graph) after setup -- for ncu launch lists."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=12)
ap.add_argument("--cycle", default="w")
ap.add_argument("--coarsest", type=int, default=3)
ap.add_argument("--mode", default="multicolour")
a = ap.parse_args()
cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle=a.cycle,
                    coarsest_level=a.coarsest, gs_mode=a.mode)
mg = P.build_solver("poisson", a.level, 1e-6, cfg)
f = P.baseline_rhs(mg.finest, 0, add_sine=True)
torch.cuda.synchronize()
mg.solve_to_tolerance(f, tol=0.0, max_cycles=1, use_graph=False)
torch.cuda.synchronize()
