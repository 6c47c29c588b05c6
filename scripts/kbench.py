"""Per-kernel timing of the HBM-bound level operations (dev tool).

python scripts/kbench.py [--level 12] [--iters 20] [--ops residual,ne_jacobi,...]
Prints one line per op: ms per call and GB/s against the algorithmic bytes
bench.py uses.  Run under ncu with --metrics gpu__time_duration.sum for the
per-kernel split.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402
from paper_1502_03917_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=12)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--ops", default="residual,ne_jacobi,multicolour,restrict,prolong")
a = ap.parse_args()

dev = torch.device("cuda:0")
sys_ = P.build_poisson_system(a.level, 1e-6)
coarse = P.build_poisson_system(a.level - 1, 1e-6)
from paper_1502_03917_b200.transfer import system_transfer  # noqa: E402
tr = system_transfer(coarse, sys_)
n = sys_.n
g = torch.Generator(device=dev).manual_seed(7)
x = torch.rand(n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
f = torch.rand(n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
r = sys_.residual(x, f)
out = torch.empty_like(r)
rc = torch.empty(coarse.n, dtype=torch.float64, device=dev)
nj = P.make_smoother(sys_, "normal")
mc = P.make_smoother(sys_, "lsgs", gs_mode="multicolour")
wfs = P.make_smoother(sys_, "lsgs", gs_mode="wavefront")
st = torch.cuda.current_stream()
BYTES = {"residual": 24, "ne_jacobi": 56, "multicolour": 32, "wavefront": 32,
         "restrict": 10, "prolong": 18}


def fn_for(op):
    if op == "residual":
        return lambda: _lib.call("ocmg_residual", sys_.handle, _lib.dptr(x),
                                 _lib.dptr(f), _lib.dptr(out), _lib.stream_ptr())
    if op == "ne_jacobi":
        return lambda: nj.sweep(x, r)
    if op == "multicolour":
        return lambda: mc.sweep(x, r)
    if op == "wavefront":
        return lambda: wfs.sweep(x, r)
    t = tr
    if op == "restrict":
        return lambda: t.restrict(r, rc)
    return lambda: t.prolong_add(rc, x)


for op in a.ops.split(","):
    fn = fn_for(op)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.iters):
        fn()
    e1.record(st)
    e1.synchronize()
    t = e0.elapsed_time(e1) / a.iters / 1e3
    print(f"{op:12s} {t * 1e3:8.4f} ms  {BYTES[op] * n / t / 1e9:8.1f} GB/s "
          f"(algorithmic {BYTES[op]} B/DOF)", flush=True)
