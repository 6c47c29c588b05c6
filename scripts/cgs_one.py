import sys
sys.path.insert(0, ".")
import torch
import paper_1502_03917_b200 as P
s = P.build_poisson_system(12, 1e-6)
x = torch.rand(s.n, dtype=torch.float64, device="cuda")
r = torch.rand(s.n, dtype=torch.float64, device="cuda")
st = P.make_smoother(s, "cgs", gs_mode="multicolour")
for _ in range(2):
    st.sweep(x, r)
torch.cuda.synchronize()
print("ok")
