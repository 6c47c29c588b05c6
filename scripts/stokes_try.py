"""Time Stokes solves at a given level (dev tool): python scripts/stokes_try.py L mode alpha"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

lv = int(sys.argv[1]) if len(sys.argv) > 1 else 5
mode = sys.argv[2] if len(sys.argv) > 2 else "multicolour"
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
t0 = time.time()
r = bench.solve_timing(lv, alpha, "v", 1, mode, False, problem="stokes")
print(r, "wall", time.time() - t0, flush=True)
