"""Per-op timing of the fused coarse block (dev tool)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402
from paper_1502_03917_b200 import _lib  # noqa: E402

cyc = sys.argv[1] if len(sys.argv) > 1 else "w"
co = int(sys.argv[2]) if len(sys.argv) > 2 else 3
top = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle=cyc, coarsest_level=co,
                    gs_mode="multicolour")
mg = P.build_solver("poisson", top, 1e-6, cfg)
h = mg.native().handle
n = mg.finest.n
x = torch.zeros(n, dtype=torch.float64, device="cuda")
f = torch.rand(n, dtype=torch.float64, device="cuda")
prof = torch.zeros(512, dtype=torch.int64, device="cuda")
nops = ctypes.c_int()
fn = _lib.load().ocmg__debug_subcycle_prof
fn.argtypes = [ctypes.c_void_p] * 4 + [ctypes.POINTER(ctypes.c_int)]
for rep in range(3):
    _lib.check(fn(h, _lib.dptr(x), _lib.dptr(f), _lib.dptr(prof), ctypes.byref(nops)))
t = prof[:nops.value].cpu().numpy()
d = (t[1:] - t[:-1]) / 1e3
names = ["resid", "sweepF", "sweepB", "restrict", "coarse", "prolong"]
print("nops", nops.value, "total us", (t[-1] - t[0]) / 1e3)
import collections
agg = collections.defaultdict(list)
# op codes are not exported: recompute the sequence as in sub_ops
ops = []
def sub_ops(j, w):
    if j == 0:
        ops.append(("coarse", 0)); return
    ops.append(("resid", j)); ops.extend([("sweepF", j)] * 2); ops.append(("restrict", j))
    for _ in range(2 if (w and j - 1 > 0) else 1):
        sub_ops(j - 1, w)
    ops.append(("prolong", j)); ops.append(("resid", j)); ops.extend([("sweepF", j)] * 2)
sub_ops(top - co, cyc == "w")
for (nm, j), dt in zip(ops, d):
    agg[(nm, j)].append(dt)
for k, v in sorted(agg.items()):
    print(k, len(v), "mean us %.2f" % (sum(v) / len(v)))
