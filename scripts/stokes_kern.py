"""Stokes generic-level kernel timings at one level (dev tool):
python scripts/stokes_kern.py [level]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1502_03917_b200 import assembly
k = int(sys.argv[1]) if len(sys.argv) > 1 else 9
s = assembly.build_stokes_system(k, 1e-2)
print(json.dumps(bench.stokes_kernel_table(s, iters=5), indent=1))
