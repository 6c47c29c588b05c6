"""Print the reference's iteration table, solved on the GPU.

python scripts/table.py [poisson|stokes] [k_lo k_hi] [--gs-mode M] [--fmt F]
e.g. python scripts/table.py poisson 5 10   (the reference stops at level 9)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03917_b200 import tables as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("problem", nargs="?", default="poisson")
ap.add_argument("levels", nargs="*", type=int)
ap.add_argument("--gs-mode", default="wavefront")
ap.add_argument("--fmt", default="markdown")
ap.add_argument("--cycle", default="w")
a = ap.parse_args()
spec = T.ExperimentSpec(problem=a.problem, levels=tuple(a.levels) or (),
                        gs_mode=a.gs_mode, fmt=a.fmt, cycle=a.cycle)
t0 = time.perf_counter()
res = T.run_table(spec)
print(T.render_table(res), end="")
print(f"({time.perf_counter() - t0:.1f} s on the GPU)", file=sys.stderr)
