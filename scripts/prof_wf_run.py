"""Run a few NE-GS wavefront sweeps at level k (profiling driver)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1502_03917_b200 as P

k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mode = sys.argv[2] if len(sys.argv) > 2 else "wavefront"
nsweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = P.build_poisson_system(k, 1e-6)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
r = s.residual(x, torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g))
st = P.make_smoother(s, "lsgs", gs_mode=mode)
for _ in range(nsweeps):
    st.sweep(x, r)
torch.cuda.synchronize()
print("ok")
