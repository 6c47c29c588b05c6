"""Per-warp cycle split of k_p1_mc_roll (dev tool; needs a -DMC2_PROF build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1502_03917_b200 as P
from paper_1502_03917_b200 import _lib
k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
s = P.build_poisson_system(k, 1e-6)
x = torch.rand(s.n, dtype=torch.float64, device="cuda")
r = torch.rand(s.n, dtype=torch.float64, device="cuda")
st = P.make_smoother(s, "lsgs", gs_mode="multicolour")
for _ in range(3): st.sweep(x, r)
torch.cuda.synchronize()
n = 256 * 24 * 4
buf = (ctypes.c_ulonglong * n)()
fn = _lib.load().ocmg__debug_mc2_prof
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(fn(buf, n))
a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 24, 4).astype(np.float64)
live = a[:, 0, 3] > 0
a = a[live]
nst = 24
strip = np.arange(256)[live] % nst
print("CTAs", a.shape[0])
tot = a[:, 0, 3]
segs = np.arange(256)[live] // nst
print("total cycles by row segment (mean over strips):", [int(tot[segs == s].mean()) for s in range(segs.max() + 1)])
for s in range(segs.max() + 1):
    b = a[segs == s]
    print("  seg", s, "row warps wait %.0f compute %.0f duty %.0f | bw wait %.0f work %.0f arrive %.0f (totals / 1000)" % (
        b[:, :21, 0].mean() / 1e3, b[:, :21, 1].mean() / 1e3, b[:, :21, 2].mean() / 1e3,
        b[:, 21, 0].mean() / 1e3, b[:, 21, 1].mean() / 1e3, b[:, 21, 2].mean() / 1e3))
print("total cycles by strip (mean over segments):", [int(tot[strip == s].mean()) for s in range(nst)])
for name, sel in (("interior", (strip > 0) & (strip < nst - 1)), ("edge", (strip == 0) | (strip == nst - 1))):
    b = a[sel]
    if not len(b): continue
    print(name, "total cycles (max, mean):", b[:, :, 3].max(), b[:, :, 3].mean())
    print("  row warps: wait %.0f compute %.0f duty %.0f (mean per warp, cycles); per compute step: wait %.0f compute %.0f duty %.0f" % (
        b[:, :21, 0].mean(), b[:, :21, 1].mean(), b[:, :21, 2].mean(),
        b[:, :21, 0].mean() / 244, b[:, :21, 1].mean() / 244, b[:, :21, 2].mean() / 244))
    print("  boundary warp: wait %.0f work %.0f arrive %.0f" % (b[:, 21, 0].mean(), b[:, 21, 1].mean(), b[:, 21, 2].mean()))
    print("  per warp compute/step:", (b[:, :21, 1].mean(axis=0) / 244).round(0))
    print("  per warp duty/step:", (b[:, :21, 2].mean(axis=0) / 244).round(0))
