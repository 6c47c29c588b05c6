"""One-launch multicolour sweep vs its 7-pass form at one level (dev tool;
run under compute-sanitizer memcheck for new kernel variants)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402
from paper_1502_03917_b200 import _lib  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for forward in (True, False):
    dsys = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(11 + k)
    x = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    r = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    x2, r2 = x.clone(), r.clone()
    st = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    if forward:
        st.sweep(x, r)
    else:
        P.smoothers.lsgs_sweep(st, x, r, order="backward")
    fn = _lib.load().ocmg__debug_mc_passes
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.c_void_p]
    _lib.check(fn(dsys.handle, int(forward), _lib.dptr(x2), _lib.dptr(r2), _lib.stream_ptr()))
    torch.cuda.synchronize()
    dx = (x - x2).abs().max().item()
    dr = (r - r2).abs().max().item()
    print(f"k={k} forward={forward} max|dx|={dx:.3e} max|dr|={dr:.3e} equal={torch.equal(x, x2) and torch.equal(r, r2)}")
