"""Sweeps of one small level (dev tool, for ncu launch timing):
python scripts/small_sweep.py [k] [mode] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1502_03917_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "wavefront"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
s = P.build_poisson_system(k, 1e-6)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g)
r = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g)
st = P.make_smoother(s, "lsgs", gs_mode=mode)
for _ in range(reps):
    st.sweep(x, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    st.sweep(x, r)
e1.record()
e1.synchronize()
print(f"k={k} {mode}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per sweep (stream, incl. launch)")
