import sys, time, json, torch
sys.path.insert(0, '.')
import bench
for k in (5, 7, 8):
    t=time.perf_counter()
    r = bench.solve_timing(k, 1e-4, "v", 1, "wavefront", False, "stokes", smoother="vanka")
    print(json.dumps(r), "total", time.perf_counter()-t, flush=True)
