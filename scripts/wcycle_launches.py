"""One L12 W(2,2) cycle (multicolour or wavefront), for an ncu launch list
(dev tool): python scripts/wcycle_launches.py [k] [v|w] [mode] [coarsest];
ncu --metrics gpu__time_duration.sum -s <warm-up launches> ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cyc = sys.argv[2] if len(sys.argv) > 2 else "w"
mode = sys.argv[3] if len(sys.argv) > 3 else "multicolour"
co = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle=cyc, coarsest_level=co,
                    gs_mode=mode)
mg = P.build_solver("poisson", k, 1e-6, cfg)
f = P.baseline_rhs(mg.finest, 0, add_sine=True)
mg.solve_to_tolerance(f, tol=0.0, max_cycles=1, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("cycle")
mg.solve_to_tolerance(f, tol=0.0, max_cycles=1, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
