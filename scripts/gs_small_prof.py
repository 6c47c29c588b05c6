"""A few exact-order sweeps of a small Poisson level (dev tool; for ncu on
k_p1_gs_small): python scripts/gs_small_prof.py [k] [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 6
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
s = P.build_poisson_system(k, 1e-6)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - 0.5
f = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g)
r = s.residual(x, f)
st = P.make_smoother(s, "lsgs", gs_mode="reference")
for _ in range(5):
    st.sweep(x, r)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(sweeps):
    st.sweep(x, r)
b.record()
torch.cuda.synchronize()
print(f"L{k}: {1e3 * a.elapsed_time(b) / sweeps:.2f} us per sweep")
