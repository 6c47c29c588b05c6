"""Config-3 solve timings (Poisson L12, W(2,2), U+sin*sin, alpha 1e-6) in both
NE-GS modes at coarsest L1 (the reference default) and L3.
python scripts/solve_c3.py [level] [coarsest ...]"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 12
coarsest = [int(a) for a in sys.argv[2:]] or [1, 3]
for c in coarsest:
    for mode in ("wavefront", "multicolour"):
        print(json.dumps(bench.solve_timing(level, 1e-6, "w", c, mode, True)), flush=True)
